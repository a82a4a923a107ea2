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


def _ref_train(A, B, K, xs, ys, cfg, tau=1.0):
    """router.hpp:318-400 itself, compiled from /root/reference (oracle/_ref)."""
    import ctypes as C
    import os
    from oracle import pyoracle
    path = os.path.join(os.path.dirname(pyoracle.__file__), "_ref", "libparse_ref.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(path)
    f = L.ref_train_router
    dp, sz = C.POINTER(C.c_double), C.c_size_t
    f.argtypes = [dp, dp, sz, sz, sz, sz, sz, C.POINTER(sz), dp, dp, C.c_double, sz, sz, C.c_double, C.c_double,
                  C.c_uint64, C.c_double, dp, dp, dp, dp]
    f.restype = C.c_int
    m, r = A.shape
    n = B.shape[0]
    T = (sz * len(xs))(*[x.shape[1] for x in xs])
    X = np.ascontiguousarray(np.concatenate([x.ravel() for x in xs]))
    Y = np.ascontiguousarray(np.concatenate([y.ravel() for y in ys]))
    th, bi = np.zeros((r, n)), np.zeros(r)
    el, fz = np.zeros(cfg.epochs), np.zeros(cfg.epochs)
    p = lambda a: np.ascontiguousarray(a).ctypes.data_as(dp)  # noqa: E731
    Ac, Bc = np.ascontiguousarray(A), np.ascontiguousarray(B)
    rc = f(p(Ac), p(Bc), m, n, r, K, len(xs), T, p(X), p(Y), cfg.learning_rate, cfg.epochs, cfg.batch_size,
           cfg.warmup_frac, cfg.weight_decay, cfg.seed, tau, th.ctypes.data_as(dp), bi.ctypes.data_as(dp),
           el.ctypes.data_as(dp), fz.ctypes.data_as(dp))
    assert rc == 0
    return th, bi, el, fz


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["acceptance", "random"])
def test_router_training_matches_reference(case, port):
    """train.py (torch f64 on the GPU) vs the reference's train_router_matrix
    compiled from /root/reference, on the same data and config: per-epoch
    update and frozen losses within f64 reassociation (1e-9 relative), and
    the returned routers select the same experts for every sequence."""
    from paper_2605_08568_b200 import train
    if case == "acceptance":  # test_router.cpp:180-224 data
        A, B = np.diag([3.0, 2.5, 2.0, 1.5, 1.0, 0.5]), np.eye(6)
        K, rng, xs, ys = 2, train.Rng(241), [], []
        for s in range(64):
            c = s % 2
            x = np.array([rng.gaussian() for _ in range(48)]).reshape(6, 8)
            x[0] += -3.0 if c else 3.0
            tgt = [2, 3] if c else [0, 1]
            xs.append(x)
            ys.append(A[:, tgt] @ (B[:, tgt].T @ x))
        cfg = train.RouterTrainConfig(learning_rate=5e-3, epochs=30, batch_size=16, warmup_frac=0.4, seed=7)
    else:  # a wider layer: r = 48 experts of a 40 x 32 matrix, K = 12, 96 sequences
        m, n, r, K = 40, 32, 48, 12
        A = port.gaussian(301, (m, r)) / np.sqrt(m)
        B = port.gaussian(302, (n, r)) / np.sqrt(n)
        xs = [port.gaussian(400 + s, (n, 6)) + (1.5 if s % 3 == 0 else -0.5) for s in range(96)]
        ys = [A[:, (s % 4) * 8:(s % 4) * 8 + K] @ (B[:, (s % 4) * 8:(s % 4) * 8 + K].T @ x) for s, x in enumerate(xs)]
        cfg = train.RouterTrainConfig(learning_rate=3e-3, epochs=12, batch_size=32, warmup_frac=0.25, seed=11)
    th, bi, el, fz = _ref_train(A, B, K, xs, ys, cfg)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    seqs = [train.precompute_router_stats(At, Bt, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
            for x, y in zip(xs, ys)]
    res = train.train_router_matrix(A, B, K, seqs, cfg)
    np.testing.assert_allclose(np.array(res.epoch_loss, dtype=np.float64), el, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.array(res.frozen_loss, dtype=np.float64), fz, rtol=1e-9, atol=1e-12)
    H = np.stack([x.mean(axis=1) for x in xs])
    got = train.select_topk(torch.from_numpy(H).cuda() @ res.theta.t() + res.bias, K).cpu().numpy()
    want = np.stack([np.sort(np.argsort(-(th @ h + bi), kind="stable")[:K]) for h in H])
    assert np.array_equal(np.sort(got, axis=1), want)
