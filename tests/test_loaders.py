"""Loader parity: checkpoints written by the reference's
own save_factorized / save_cache (tests/golden/make_ckpt.cpp, committed) load
onto the device and reproduce the reference's routed selections, values and
cache retrieval."""
import os

import numpy as np
import pytest
import torch

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ckpt")


def _expected():
    sel = {}
    with open(os.path.join(GOLD, "expected.txt")) as f:
        for line in f:
            parts = line.split()
            sel[parts[0]] = (int(parts[1]), np.array([int(v) for v in parts[2:]], dtype=np.uint32))
    return sel


def test_blob_errors_follow_the_reference(tmp_path):
    from paper_2605_08568_b200 import loaders
    p = tmp_path / "short.f64"
    np.arange(3.0).tofile(p)
    with pytest.raises(RuntimeError, match="short read"):
        loaders._blob(str(p), 4)
    with pytest.raises(RuntimeError, match="cannot read"):
        loaders._blob(str(tmp_path / "missing.f64"), 1)
    (tmp_path / "manifest.json").write_text('{"kind": "dense"}')
    with pytest.raises(RuntimeError, match="not a factorized checkpoint"):
        loaders.load_factorized(str(tmp_path))


def test_fixture_files_are_reference_layout():
    import json
    man = json.load(open(os.path.join(GOLD, "factorized", "manifest.json")))
    assert man["kind"] == "factorized" and man["format_version"] == 1
    for tid, tj in man["tensors"].items():
        a = os.path.getsize(os.path.join(GOLD, "factorized", f"{tid}.A.f64"))
        assert a == tj["m"] * tj["r_store"] * 8
    cj = json.load(open(os.path.join(GOLD, "cache", "cache.json")))
    assert cj["entry_count"] == 6 and cj["d_model"] == 32


@pytest.mark.gpu
def test_load_factorized_routes_and_forwards_like_the_reference():
    import paper_2605_08568_b200 as pg
    from paper_2605_08568_b200 import loaders
    model = loaders.load_factorized(os.path.join(GOLD, "factorized"), dtype="f64")
    exp = _expected()
    xs = np.fromfile(os.path.join(GOLD, "x.f64"))
    ys = np.fromfile(os.path.join(GOLD, "expected_y.f64"))
    xo = yo = 0
    assert sorted(model.layers) == sorted(exp)
    for tid in ["b0.q", "b0.k", "b0.v", "b0.o", "b0.up", "b0.gate", "b0.down"]:
        layer, router = model.layers[tid], model.routers[tid]
        K, want_sel = exp[tid]
        x = xs[xo: xo + layer.n * 5].reshape(layer.n, 5)
        y_ref = ys[yo: yo + layer.m * 5].reshape(layer.m, 5)
        xo += layer.n * 5
        yo += layer.m * 5
        got = pg.route_select(router, torch.from_numpy(x).cuda(), K)[0].cpu().numpy().astype(np.uint32)
        assert np.array_equal(got, want_sel), tid
        y = pg.masked_forward(layer, pg.RankSelection(got), torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.abs(y - y_ref).max() / np.abs(y_ref).max() <= 1e-10, tid
    assert model.core["embed"].shape == (8, 32) and model.n_blocks == 1


@pytest.mark.gpu
def test_load_cache_retrieves_like_the_reference():
    import paper_2605_08568_b200 as pg
    from paper_2605_08568_b200 import loaders
    cache = loaders.load_cache(os.path.join(GOLD, "cache"))
    assert len(cache.entries) == 6 and cache.min_similarity == 0.8
    entry, hit, sim = open(os.path.join(GOLD, "retrieve.txt")).read().split()
    q = np.fromfile(os.path.join(GOLD, "query.f64"))
    res = pg.retrieve(cache, q, exact_similarity=True)
    assert res.entry == int(entry) and res.hit == bool(int(hit))
    assert res.similarity == float(sim)
    assert res.pattern is cache.entries[int(entry)].pattern


@pytest.mark.gpu
def test_embed_prompt_on_device_matches_reference():
    """embed_prompt (pattern_cache.hpp:50-65): block-0 forward of the static-
    prefix model on device, pooled and normalised, vs the reference's own."""
    import paper_2605_08568_b200 as pg
    from paper_2605_08568_b200 import embed, loaders
    model = loaders.load_factorized(os.path.join(GOLD, "factorized"), dtype="f64")
    toks = [int(t) for t in open(os.path.join(GOLD, "embed_tokens.txt")).read().split()]
    want = np.fromfile(os.path.join(GOLD, "embed.f64"))
    got = embed.embed_prompt(model, toks, source="golden")
    assert got.source == "golden"
    assert np.abs(np.asarray(got.vec) - want).max() <= 1e-12
    cache = loaders.load_cache(os.path.join(GOLD, "cache"))
    a = pg.retrieve(cache, got.vec)
    b = pg.retrieve(cache, want)
    assert (a.entry, a.hit) == (b.entry, b.hit)
    with pytest.raises(ValueError):
        embed.embed_prompt(model, [])
