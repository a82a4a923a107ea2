"""Serving-level parity on the GPU:

* PatternServer -- retrieve-or-route composition (pattern_cache.hpp:67-124,
  model.hpp:96-106): hit -> the entry's SelectionMap (packs reused across
  hits), miss -> bit-exact online routing of every tensor id + cache_insert
  (refused at capacity), each decision checked against the oracle's retrieve
  and select_topk(score(mean_pool(x))).
* ExecEngine / scattered_forward / ExecProvider (exec_engine.hpp:193-348): the
  reference's four-variant test (test_exec_engine.cpp:128-146) on the Python
  engine, f64 against the oracle's masked_forward (<= 1e-12), and the
  aggregated variants equal to each other bit for bit.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_08568_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def small_model(pg, port, dtype="f64", d=64, ff=96, blocks=1, ratio=0.5, seed=3):
    layers, routers, raw = {}, {}, {}
    shapes = {"q": (d, d), "k": (d, d), "v": (d, d), "o": (d, d), "up": (ff, d), "gate": (ff, d), "down": (d, ff)}
    for b in range(blocks):
        for j, (p, (m, n)) in enumerate(shapes.items()):
            tid = pg.tensor_id(b, p)
            K = pg.single_layer_k(m, n, ratio)
            r = pg.store_rank(K, min(m, n))
            A = port.gaussian(seed + 10 * j, (m, r)) / np.sqrt(m)
            B = port.gaussian(seed + 10 * j + 1, (n, r)) / np.sqrt(n)
            theta = port.gaussian(seed + 10 * j + 2, (r, n))
            layers[tid] = pg.FactorizedLayer(A, B, K, dtype=dtype, layer_id=tid)
            routers[tid] = pg.RouterParams(theta)
            raw[tid] = (A, B, theta, K)
    return pg.FactorizedModel(layers, routers, blocks), raw


def test_pattern_server_retrieve_or_route(pg, port):
    model, raw = small_model(pg, port)
    d = 64
    rng = np.random.default_rng(7)
    cache = pg.PatternCache(d, capacity=4, min_similarity=0.8)
    embs = rng.standard_normal((3, d))
    embs /= np.linalg.norm(embs, axis=1, keepdims=True)
    pats = [{tid: pg.RankSelection(np.sort(rng.choice(raw[tid][0].shape[1], raw[tid][3], replace=False)))
             for tid in raw} for _ in range(3)]
    cache.load([pg.CacheEntry(pg.PromptEmbedding(e), p) for e, p in zip(embs, pats)])
    server = pg.PatternServer(model, cache)

    def inputs_for(seed):
        g = np.random.default_rng(seed)
        xs = {tid: g.standard_normal((raw[tid][1].shape[0], 9)) for tid in raw}
        return xs, {tid: torch.from_numpy(x).cuda() for tid, x in xs.items()}

    # hit: near entry 1
    q = embs[1] + 0.05 * rng.standard_normal(d)
    q /= np.linalg.norm(q)
    e_ref, s_ref, h_ref = port.retrieve(embs, 0.8, q)
    xs, xd = inputs_for(1)
    s1 = server.select_for_prompt(pg.PromptEmbedding(q), xd)
    assert (s1.source, s1.entry, s1.similarity) == ("hit", e_ref, s_ref) and h_ref
    assert s1.pattern is cache.entries[1].pattern and not s1.inserted
    packs = server.layouts(s1)
    assert server.layouts(server.select_for_prompt(pg.PromptEmbedding(q), xd)) is packs  # second hit: no re-pack
    assert server.packs_built == 1

    # miss: far query -> every tensor id routed bit-exactly, then inserted
    far = rng.standard_normal(d)
    far /= np.linalg.norm(far)
    e_ref, s_ref, h_ref = port.retrieve(embs, 0.8, far)
    assert not h_ref
    xs, xd = inputs_for(2)
    s2 = server.select_for_prompt(pg.PromptEmbedding(far), xd)
    assert s2.source == "routed" and s2.inserted and s2.entry == 3 and len(cache.entries) == 4
    assert s2.similarity == pytest.approx(s_ref, abs=1e-12)
    for tid, (A, B, theta, K) in raw.items():
        want = port.select_topk(port.score(theta, np.zeros(theta.shape[0]), port.mean_pool(xs[tid])), K)
        assert np.array_equal(s2.pattern[tid].indices, want), tid
    # the routed prompt now hits its own entry
    s3 = server.select_for_prompt(pg.PromptEmbedding(far), xd)
    assert s3.source == "hit" and s3.entry == 3 and s3.pattern is s2.pattern

    # at capacity: a new miss is routed but refused by cache_insert
    far2 = rng.standard_normal(d)
    far2 /= np.linalg.norm(far2)
    s4 = server.select_for_prompt(pg.PromptEmbedding(far2), inputs_for(3)[1])
    assert s4.source == "routed" and not s4.inserted and s4.entry == -1 and len(cache.entries) == 4

    # serving with the frozen selection: prefill and decode through the provider
    prov = server.provider(s2)
    tid = pg.tensor_id(0, "up")
    A, B, _, _ = raw[tid]
    for T in (9, 1):
        x = rng.standard_normal((B.shape[0], T))
        y = prov.apply(0, "up", torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel(y, port.masked_forward(A, B, s2.pattern[tid].indices, x)) <= 1e-10


def test_exec_engine_four_variants(pg, port):
    """test_exec_engine.cpp:128-146 on the Python ExecEngine (f64)."""
    model, raw = small_model(pg, port, blocks=2)
    rng = np.random.default_rng(17)
    pats = []
    for _ in range(4):  # prefix-biased subsets so psi < 1 yields shared experts
        p = {}
        for tid, (A, B, _, K) in raw.items():
            pool = list(range(A.shape[1]))
            sel = []
            for _ in range(K):
                pick = 0 if rng.integers(2) else int(rng.integers(len(pool)))
                sel.append(pool.pop(pick))
            p[tid] = pg.RankSelection(np.sort(sel))
        pats.append(p)
    eng = pg.ExecEngine.build(model.layers, pats, 0.5)
    V = pg.ExecVariant
    worst = 0.0
    for tid, (A, B, _, _) in raw.items():
        x = rng.standard_normal((B.shape[0], 6))
        xd = torch.from_numpy(x).cuda()
        for pid in range(len(pats)):
            ref = port.masked_forward(A, B, pats[pid][tid].indices, x)
            outs = {v: eng.forward(tid, pid, xd, v).cpu().numpy() for v in V}
            for y in outs.values():
                worst = max(worst, rel(y, ref))
            assert np.array_equal(outs[V.aggregated_only], outs[V.aggregated_fused])
            assert np.array_equal(outs[V.scattered_unfused], outs[V.fused_only])
            assert np.array_equal(outs[V.scattered_unfused],
                                  pg.scattered_forward(model.layers[tid], pats[pid][tid], xd).cpu().numpy())
    assert worst <= 1e-12, worst
    with pytest.raises(IndexError):
        eng.forward(pg.tensor_id(0, "q"), 9, torch.zeros(64, 1, dtype=torch.float64, device="cuda"),
                    V.scattered_unfused)
    # ExecProvider: one launch descriptor per projection, same values as the engine
    prov = pg.ExecProvider(eng, 1, V.aggregated_fused)
    hn = torch.from_numpy(rng.standard_normal((64, 5))).cuda()
    q, k, v = prov.qkv(0, hn)
    assert prov.launches == 3
    assert torch.equal(q, eng.forward(pg.tensor_id(0, "q"), 1, hn, V.aggregated_fused))
    # storage overhead counts duplicated residual columns only
    same = pg.ExecEngine.build(model.layers, [pats[0]] * 3, 0.9)
    assert same.storage_overhead() == 0.0 and 0.0 < eng.storage_overhead() < 4.0
