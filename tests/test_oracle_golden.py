"""Pin the oracle (C restatement) to the reference.

1. Known-answer vectors from the reference's own doctest suites,
   run against the port AND the compiled reference.
2. Randomised bit-exact equivalence port == reference (oracle/_ref) on every
   hot-path routine.
3. The committed golden fixtures (tests/golden/, produced by
   tests/golden/make_golden.py from the compiled reference) reproduce exactly.
CPU only.
"""
import math
import os

import numpy as np
import pytest

from oracle import pyoracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(params=["port", "reference"])
def impl(request, port):
    if request.param == "port":
        return port
    return request.getfixturevalue("ref")


# ---------------- known-answer tests (reference tests, restated) ----------------

def test_select_topk_ties_lower_index(impl):
    # test_router.cpp:75-83
    logits = [1.0, 2.0, 2.0, 1.0, 2.0]
    assert impl.select_topk(logits, 2).tolist() == [1, 2]
    assert impl.select_topk(logits, 4).tolist() == [0, 1, 2, 4]
    with pytest.raises(ValueError):
        impl.select_topk(logits, 0)
    with pytest.raises(ValueError):
        impl.select_topk(logits, 6)


def test_select_topk_zero_router_is_static_prefix(impl):
    # router.hpp:34 zero init -> all logits equal -> prefix {0..K-1}
    assert impl.select_topk(np.zeros(37), 11).tolist() == list(range(11))


def test_cosine_frozen_values(impl):
    # test_pattern_cache.cpp:40-46
    assert impl.cosine([1, 0], [1, 1]) == pytest.approx(1 / math.sqrt(2), rel=1e-12)
    assert impl.cosine([2, 0, 0], [0, 3, 0]) == pytest.approx(0.0, abs=1e-12)
    assert impl.cosine([1, 2, 3], [2, 4, 6]) == pytest.approx(1.0, rel=1e-12)
    assert impl.cosine([1, 1], [-1, -1]) == pytest.approx(-1.0, rel=1e-12)


def test_retrieve_nearest_and_threshold(impl):
    # test_pattern_cache.cpp:80-112
    emb = np.array([[1.0, 0.0], [0.0, 1.0]])
    e, sim, hit = impl.retrieve(emb, 0.9, [0.995, 0.0998])
    assert hit and e == 0 and sim > 0.99
    e, sim, hit = impl.retrieve(emb, 0.9, [0.707, 0.707])
    assert not hit
    with pytest.raises(RuntimeError):
        impl.retrieve(np.zeros((0, 2)), 0.9, [1.0, 0.0])


def test_retrieve_duplicate_entries_first_max(impl):
    # strict '>' keeps the first maximum (pattern_cache.hpp:109)
    emb = np.array([[0.0, 1.0], [0.6, 0.8], [0.6, 0.8], [0.6, 0.8]])
    e, sim, hit = impl.retrieve(emb, 0.0, [0.6, 0.8])
    assert e == 1 and hit


def test_check_selection_errors(impl):
    # test_rank_experts.cpp:132-140
    with pytest.raises(ValueError):
        impl.check_selection([], 4)
    with pytest.raises(ValueError):
        impl.check_selection([2, 1], 4)
    with pytest.raises(ValueError):
        impl.check_selection([1, 1], 4)
    with pytest.raises(IndexError):
        impl.check_selection([0, 4], 4)
    impl.check_selection([0, 2, 3], 4)


def test_masked_forward_matches_naive(impl, port):
    # test_rank_experts.cpp:56-69 (masked vs explicit sum of a_e b_e^T) and :71-77
    A = port.gaussian(101, (6, 8)); B = port.gaussian(102, (8, 8)); x = port.gaussian(103, (8, 5))
    rng = np.random.default_rng(104)
    for _ in range(20):
        sel = np.flatnonzero(rng.random(8) < 0.5).astype(np.uint32)
        if sel.size == 0:
            sel = np.array([3], dtype=np.uint32)
        got = impl.masked_forward(A, B, sel, x)
        want = (A[:, sel] @ B[:, sel].T) @ x
        assert np.max(np.abs(got - want)) < 1e-11 * (1 + np.max(np.abs(want)))
    full = impl.masked_forward(A, B, np.arange(8, dtype=np.uint32), x)
    assert np.allclose(full, A @ B.T @ x, rtol=0, atol=1e-11 * (1 + np.abs(A @ B.T @ x).max()))


def test_aggregate_layout_frozen_split(impl, port):
    # test_exec_engine.cpp:89-116
    A = port.gaussian(1, (5, 4)); B = port.gaussian(2, (6, 4))
    pats = [[0, 1], [0, 1], [0, 2]]
    g = impl.aggregate_layout(A, B, pats, 0.9, elem=8)
    assert g.shared_ids.tolist() == [0]
    assert g.residual_ids(0).tolist() == [1]
    assert g.residual_ids(2).tolist() == [2]
    assert g.use_shared(0).tolist() == [1]
    assert [g.arena_offset(p) for p in range(3)] == [1, 2, 3]
    g2 = impl.aggregate_layout(A, B, pats, 0.5, elem=8)
    assert g2.shared_ids.tolist() == [0, 1]
    assert g2.use_shared(2).tolist() == [1, 0]
    for bad_psi in (0.0, 1.5):
        with pytest.raises(ValueError):
            impl.aggregate_layout(A, B, pats, bad_psi, elem=8)
    with pytest.raises(ValueError):
        impl.aggregate_layout(A, B, [], 0.9, elem=8)
    with pytest.raises(IndexError):
        impl.aggregate_layout(A, B, [[4]], 0.9, elem=8)
    # disjoint at psi=1 (:118-126)
    g3 = impl.aggregate_layout(A, B, [[0, 1], [2, 3]], 1.0, elem=8)
    assert g3.shared_ids.size == 0 and g3.residual_ids(0).size == 2


def test_aggregated_variants_match_masked(impl, port):
    # test_exec_engine.cpp:128-165: f64 bit-identical, f32 within 1e-5(1+|ref|)
    m, n, r = 12, 10, 8
    A = port.gaussian(5, (m, r)); B = port.gaussian(6, (n, r))
    pats = [p[0] for p in pyoracle.make_patterns(17, 4, [(r, 4)])]
    g64 = impl.aggregate_layout(A, B, pats, 0.5, elem=8)
    g32 = impl.aggregate_layout(A, B, pats, 0.5, elem=4)
    x = port.gaussian(19, (n, 6))
    for pid, sel in enumerate(pats):
        ref = impl.masked_forward(A, B, sel, x)
        assert np.array_equal(g64.forward(pid, x), ref)
        got32 = g32.forward(pid, x.astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(got32 - ref) < 1e-5 * (1 + np.abs(ref)))


def test_maximal_runs(impl):
    # test_exec_engine.cpp:76-87
    assert impl.maximal_runs([5, 0, 1, 2, 7, 6, 9]) == [(0, 3), (5, 3), (9, 1)]
    assert len(impl.maximal_runs([3, 3, 3])) == 1
    assert impl.maximal_runs([]) == []


def test_budget_shapes(impl):
    # SURVEY.md §8 derived-shapes table (factorize.hpp:86-89,135-195)
    for (m, n, rho, K, rs) in [(4096, 4096, 0.6, 819, 1638), (11008, 4096, 0.6, 1194, 2388),
                               (4096, 11008, 0.6, 1194, 2388), (5120, 5120, 0.4, 1536, 3072),
                               (13824, 5120, 0.4, 2241, 4482)]:
        assert impl.single_layer_k(m, n, rho) == K
        assert impl.store_rank(K, min(m, n), 2.0) == rs


# ---------------- port == reference, bit for bit ----------------

def test_port_equals_reference_router(port, ref):
    for seed, (r, n, T) in enumerate([(37, 19, 5), (300, 128, 16), (1638, 512, 3)]):
        theta = port.gaussian(1000 + seed, (r, n)); bias = port.gaussian(2000 + seed, (r,))
        x = port.gaussian(3000 + seed, (n, T))
        h1, h2 = port.mean_pool(x), ref.mean_pool(x)
        assert np.array_equal(h1, h2)
        z1, z2 = port.score(theta, bias, h1), ref.score(theta, bias, h2)
        assert np.array_equal(z1, z2)
        for k in (1, r // 2, r):
            assert np.array_equal(port.select_topk(z1, k), ref.select_topk(z2, k))


def test_port_equals_reference_cache(port, ref):
    emb = port.gaussian(11, (64, 48)); q = port.gaussian(12, (48,))
    assert port.retrieve(emb, 0.1, q) == ref.retrieve(emb, 0.1, q)
    for i in range(8):
        assert port.cosine(emb[i], q) == ref.cosine(emb[i], q)
    x = port.gaussian(13, (48, 7))
    assert np.array_equal(port.embed_normalize(x), ref.embed_normalize(x))


def test_port_equals_reference_values(port, ref):
    m, n, r = 40, 56, 30
    A = port.gaussian(21, (m, r)); B = port.gaussian(22, (n, r)); x = port.gaussian(23, (n, 3))
    pats = [p[0] for p in pyoracle.make_patterns(17171, 5, [(r, 15)])]
    for sel in pats:
        assert np.array_equal(port.masked_forward(A, B, sel, x), ref.masked_forward(A, B, sel, x))
        assert np.array_equal(port.scattered_forward_f32(A.astype(np.float32), B.astype(np.float32), sel,
                                                         x.astype(np.float32)),
                              ref.scattered_forward_f32(A.astype(np.float32), B.astype(np.float32), sel,
                                                        x.astype(np.float32)))
    for elem in (4, 8):
        g1 = port.aggregate_layout(A, B, pats, 0.9, elem)
        g2 = ref.aggregate_layout(A, B, pats, 0.9, elem)
        assert np.array_equal(g1.shared_ids, g2.shared_ids)
        for p in range(len(pats)):
            assert np.array_equal(g1.residual_ids(p), g2.residual_ids(p))
            assert g1.arena_offset(p) == g2.arena_offset(p)
            assert np.array_equal(g1.use_shared(p), g2.use_shared(p))
            xx = x.astype(np.float32) if elem == 4 else x
            assert np.array_equal(g1.forward(p, xx), g2.forward(p, xx))


def test_port_rng_equals_reference(port, ref):
    lib = ref.lib
    import ctypes as C
    f = lib.ref_fill_gaussian
    f.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.c_size_t]
    out = np.empty(1000)
    f(77, out.ctypes.data_as(C.POINTER(C.c_double)), 1000)
    assert np.array_equal(out, port.gaussian(77, (1000,)))


# ---------------- committed golden fixtures ----------------

def test_golden_fixtures_reproduce(port):
    path = os.path.join(GOLDEN, "route_cache_values.npz")
    if not os.path.exists(path):
        pytest.skip("golden fixtures not generated")
    g = np.load(path)
    x = port.gaussian(int(g["seed_x"]), tuple(g["x_shape"]))
    theta = port.gaussian(int(g["seed_theta"]), tuple(g["theta_shape"]))
    bias = np.zeros(theta.shape[0])
    h = port.mean_pool(x)
    assert np.array_equal(h, g["h"])
    z = port.score(theta, bias, h)
    assert np.array_equal(z, g["logits"])
    assert np.array_equal(port.select_topk(z, int(g["K"])), g["sel"])
    emb = port.gaussian(int(g["seed_emb"]), tuple(g["emb_shape"]))
    q = g["query"]
    e, sim, hit = port.retrieve(emb, float(g["min_sim"]), q)
    assert (e, sim, hit) == (int(g["entry"]), float(g["similarity"]), bool(g["hit"]))
    A = port.gaussian(int(g["seed_A"]), tuple(g["A_shape"]))
    B = port.gaussian(int(g["seed_B"]), tuple(g["B_shape"]))
    y = port.masked_forward(A, B, g["sel"], x[: B.shape[0]])
    assert np.array_equal(y, g["y_masked"])
