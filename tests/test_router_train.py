"""Offline router training on the GPU (router.hpp:318-400) against the
reference's own acceptance test (test_router.cpp:180-224): same data (the
reference's Rng stream), same config, same pass criteria."""
import numpy as np
import pytest
import torch


def test_rng_port_matches_reference_stream(port):
    from paper_2605_08568_b200.train import Rng
    r = Rng(241)
    got = np.array([r.gaussian() for _ in range(64)])
    assert np.array_equal(got, port.gaussian(241, (64,)))
    r = Rng(7)
    assert [r.below(10) for _ in range(3)] == [r2 for r2 in _below_ref(7, 10, 3)]


def _below_ref(seed, n, count):
    from paper_2605_08568_b200.train import Rng
    r = Rng(seed)
    return [r.next_u64() % n for _ in range(count)]


@pytest.mark.gpu
def test_router_training_learns_input_dependent_selection():
    import paper_2605_08568_b200 as pg
    from paper_2605_08568_b200 import train
    sigma = [3.0, 2.5, 2.0, 1.5, 1.0, 0.5]
    A = np.diag(sigma)
    B = np.eye(6)
    rng = train.Rng(241)
    seqs, cluster = [], []
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for s in range(64):
        c = s % 2
        x = np.array([rng.gaussian() for _ in range(6 * 8)]).reshape(6, 8)
        x[0] += -3.0 if c else 3.0
        tgt = [2, 3] if c else [0, 1]
        y = A[:, tgt] @ (B[:, tgt].T @ x)
        seqs.append(train.precompute_router_stats(At, Bt, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
        cluster.append(c)
    cfg = train.RouterTrainConfig(learning_rate=5e-3, epochs=30, batch_size=16, warmup_frac=0.4, seed=7)
    res = train.train_router_matrix(A, B, 2, seqs, cfg)
    assert len(res.epoch_loss) == 30 and len(res.frozen_loss) == 30
    G = At.t() @ At
    routed = statict = 0.0
    correct = 0
    router = pg.RouterParams(res.theta, res.bias)
    for s, st in enumerate(seqs):
        # serve with the bit-exact device router (the reference's score + select_topk)
        sel = pg.route_select_pooled(router, st.h, 2)[0].long()
        routed += train._selection_loss(G, st, sel)
        statict += train._selection_loss(G, st, torch.tensor([0, 1], device="cuda"))
        correct += sel.tolist() == ([2, 3] if cluster[s] else [0, 1])
    routed /= 64
    statict /= 64
    assert routed <= statict + 1e-9
    assert routed < 0.25 * statict
    assert correct >= 58


@pytest.mark.gpu
def test_router_training_is_deterministic():
    from paper_2605_08568_b200 import train
    A = np.diag([2.0, 1.5, 1.0, 0.5])
    At = torch.from_numpy(A).cuda()
    rng = train.Rng(251)
    seqs = []
    for _ in range(12):
        x = np.array([rng.gaussian() for _ in range(4 * 5)]).reshape(4, 5)
        y = A[:, [0, 2]] @ x[[0, 2]]
        seqs.append(train.precompute_router_stats(At, torch.eye(4, dtype=torch.float64, device="cuda"),
                                                  torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
    cfg = train.RouterTrainConfig(learning_rate=1e-2, epochs=4, batch_size=5, seed=3)
    a = train.train_router_matrix(A, np.eye(4), 2, seqs, cfg)
    b = train.train_router_matrix(A, np.eye(4), 2, seqs, cfg)
    assert torch.equal(a.theta, b.theta) and torch.equal(a.bias, b.bias)
    assert a.epoch_loss == b.epoch_loss
    with pytest.raises(ValueError):
        train.train_router_matrix(A, np.eye(4), 2, [], cfg)
