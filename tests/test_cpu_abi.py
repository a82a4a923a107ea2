"""CPU-side checks of the product boundary (no GPU needed):
the C-ABI library loads and exports every symbol include/parse_gpu.h declares,
argument validation that happens before any device work mirrors the reference's
exception classes/messages, and the host-side utilities (Rng, pattern generator,
plan, runs, shape rules) match the oracle / reference.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "parse_gpu.h")


@pytest.fixture(scope="module")
def pglib():
    from paper_2605_08568_b200 import _build, _lib
    _build.build()
    return _lib.lib()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(pglib):
    names = declared_functions()
    assert len(names) >= 35
    for nm in names:
        assert hasattr(pglib, nm), f"{nm} declared in parse_gpu.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2605_08568_b200", "lib",
                                                                     "libparse_gpu.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (pg_[a-z0-9_]+)", out))
    assert set(names) <= exported


def test_library_is_sm100a(pglib):
    so = os.path.join(ROOT, "paper_2605_08568_b200", "lib", "libparse_gpu.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_select_topk_validation_before_device_work(pglib):
    from paper_2605_08568_b200 import _lib
    with pytest.raises(ValueError, match="select_topk: K out of range"):
        _lib.call("pg_select_topk", None, 5, 1, 0, None, None)
    with pytest.raises(ValueError, match="select_topk: K out of range"):
        _lib.call("pg_select_topk", None, 5, 1, 6, None, None)


def test_rng_matches_reference(pglib, port):
    import paper_2605_08568_b200 as pg
    assert np.array_equal(pg.rng_gaussian(77, (4096,)), port.gaussian(77, (4096,)))


def test_pattern_generator_matches_reference_algorithm(pglib):
    import paper_2605_08568_b200 as pg
    from oracle import pyoracle
    layers = [(1638, 819), (2388, 1194), (37, 5)]
    a = pg.make_patterns(17171, 4, layers)
    b = pyoracle.make_patterns(17171, 4, layers)
    for ra, rb in zip(a, b):
        for sa, sb in zip(ra, rb):
            assert np.array_equal(sa.indices, sb)


def test_shape_rules(pglib, port):
    import paper_2605_08568_b200 as pg
    for (m, n, rho) in [(4096, 4096, 0.6), (11008, 4096, 0.6), (4096, 11008, 0.6), (5120, 5120, 0.4),
                        (13824, 5120, 0.4), (96, 96, 0.3), (24, 16, 0.3)]:
        k = pg.single_layer_k(m, n, rho)
        assert k == port.single_layer_k(m, n, rho)
        assert pg.store_rank(k, min(m, n)) == port.store_rank(k, min(m, n))


def test_build_plan_counts(pglib):
    import paper_2605_08568_b200 as pg
    # test_exec_engine.cpp:50-74 / acceptance criterion 7
    p1 = pg.build_plan(2, False)
    p2 = pg.build_plan(2, True)
    assert p1.launches_per_block == 8 and p2.launches_per_block == 9 and p1.unfused_per_block == 14
    for plan in (p1, p2):
        seen = {}
        for l in plan.launches:
            for tid in l.tensor_ids:
                seen[tid + "." + l.side] = seen.get(tid + "." + l.side, 0) + 1
        assert len(seen) == 14 * 2 and all(v == 1 for v in seen.values())
    assert p1.launches[0].kind == pg.LaunchKind.fused_B and len(p1.launches[0].tensor_ids) == 3
    assert len(p2.launches[1].tensor_ids) == 1 and len(p2.launches[2].tensor_ids) == 2


def test_maximal_runs_matches_oracle(pglib, port):
    import paper_2605_08568_b200 as pg
    rng = np.random.default_rng(5)
    for _ in range(20):
        cols = rng.integers(0, 40, size=rng.integers(0, 30))
        got = [(r.start, r.len) for r in pg.maximal_runs(cols)]
        assert got == port.maximal_runs(cols)


def test_product_does_not_import_oracle():
    """The product package must never route through the checker."""
    pkg = os.path.join(ROOT, "paper_2605_08568_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle_", "").lower() or f == "_build.py", f


def test_peer_buffer_sizing_and_validation(pglib):
    """Expert-sharded peer reduction: receive buffers hold 2 parities x npeer x m
    tagged 8-byte words; 1..8 ranks."""
    import ctypes as C
    from paper_2605_08568_b200 import _lib
    out = C.c_size_t()
    _lib.call("pg_peer_buffer_bytes", 4096, 4, C.byref(out))
    assert out.value == 2 * 4 * 4096 * 8
    with pytest.raises(ValueError, match="1..8 ranks"):
        _lib.call("pg_peer_buffer_bytes", 4096, 9, C.byref(out))
    with pytest.raises(ValueError, match="1..8 ranks"):
        _lib.call("pg_peer_buffer_bytes", 0, 2, C.byref(out))
    from paper_2605_08568_b200.dist import PeerReduceLinear
    with pytest.raises(ValueError, match="1..8 ranks"):
        PeerReduceLinear(np.zeros((4, 4)), np.zeros((4, 4)), 9, 0)
