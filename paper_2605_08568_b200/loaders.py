"""Artifact loaders onto the device: the reference's
own checkpoint formats, so the GPU path serves reference-produced artefacts.

* ``load_factorized(dir)`` reads what ``save_factorized`` writes
  (checkpoint.hpp:135-202): ``manifest.json`` + ``<id>.A.f64`` (m x r_store) +
  ``<id>.B.f64`` (n x r_store) per tensor + ``router_<id>.f64`` = theta (r x n)
  followed by bias (r), all little-endian row-major f64.  Factors become
  device ``FactorizedLayer``s in the requested storage dtype (expert-major
  B^T, packed by the C-ABI), routers device ``RouterParams`` (f64, as the
  reference scores them).  The LM core blobs (embed / head / norms,
  checkpoint.hpp:69-97) are outside the hot path and are returned as host
  arrays.
* ``load_cache(dir)`` reads what ``save_cache`` writes
  (pattern_cache.hpp:267-327): ``cache.json`` + ``embeddings.f64`` +
  ``patterns.u32`` -> a device-resident ``PatternCache``.

Errors follow the reference: ``RuntimeError("not a factorized checkpoint")``,
``RuntimeError("cannot read <path>")`` / ``("short read: <path>")``.
"""
from __future__ import annotations

import json
import os

import numpy as np

from .api import CacheEntry, FactorizedLayer, FactorizedModel, PatternCache, PromptEmbedding, RankSelection, RouterParams


def _blob(path: str, count: int, dtype=np.float64) -> np.ndarray:
    """read_blob (checkpoint.hpp:27-35)."""
    if not os.path.exists(path):
        raise RuntimeError(f"cannot read {path}")
    a = np.fromfile(path, dtype=dtype, count=count)
    if a.size != count:
        raise RuntimeError(f"short read: {path}")
    return a


class LoadedModel(FactorizedModel):
    """FactorizedModel plus the manifest fields the reference keeps
    (lm_config, compression, seed) and the host LM-core blobs."""

    def __init__(self):
        super().__init__()
        self.lm_config: dict = {}
        self.compression: dict = {}
        self.seed: int = 0
        self.core: dict = {}
        self.sigma: dict = {}


def load_factorized(path: str, dtype: str = "bf16", routers: bool = True) -> LoadedModel:
    """load_factorized (checkpoint.hpp:165-202) onto the device."""
    mpath = os.path.join(path, "manifest.json")
    if not os.path.exists(mpath):
        raise RuntimeError(f"cannot read {mpath}")
    with open(mpath) as f:
        man = json.load(f)
    if man.get("kind") != "factorized":
        raise RuntimeError("not a factorized checkpoint")
    m = LoadedModel()
    m.lm_config = dict(man["lm_config"])
    m.compression = dict(man["compression"])
    m.seed = int(man["seed"])
    m.n_blocks = int(m.lm_config["n_blocks"])
    d, vocab = int(m.lm_config["d_model"]), int(m.lm_config["vocab"])
    m.core = {"embed": _blob(os.path.join(path, "embed.f64"), vocab * d).reshape(vocab, d),
              "head": _blob(os.path.join(path, "head.f64"), vocab * d).reshape(vocab, d),
              "norm_final": _blob(os.path.join(path, "norm_final.f64"), d)}
    for b in range(m.n_blocks):
        for nm in ("attn_norm", "mlp_norm"):
            m.core[f"b{b}.{nm}"] = _blob(os.path.join(path, f"b{b}.{nm}.f64"), d)
    for tid, tj in man["tensors"].items():
        rows, cols, K, r = int(tj["m"]), int(tj["n"]), int(tj["K"]), int(tj["r_store"])
        A = _blob(os.path.join(path, f"{tid}.A.f64"), rows * r).reshape(rows, r)
        B = _blob(os.path.join(path, f"{tid}.B.f64"), cols * r).reshape(cols, r)
        layer = FactorizedLayer(A, B, K, dtype=dtype, layer_id=tid, sigma=list(tj["sigma"]))
        layer.whitened = bool(tj.get("whitened", False))
        m.layers[tid] = layer
    if routers:
        for tid, rj in man.get("routers", {}).items():
            rr, nn = int(rj["r"]), int(rj["n"])
            blob = _blob(os.path.join(path, f"router_{tid}.f64"), rr * nn + rr)
            m.routers[tid] = RouterParams(blob[: rr * nn].reshape(rr, nn), blob[rr * nn:],
                                          tau=float(rj["tau"]), eps=float(rj["eps"]))
    return m


def load_cache(path: str) -> PatternCache:
    """load_cache (pattern_cache.hpp:294-327) into a device-resident cache."""
    jpath = os.path.join(path, "cache.json")
    if not os.path.exists(jpath):
        raise RuntimeError(f"cannot read {jpath}")
    with open(jpath) as f:
        j = json.load(f)
    d, n = int(j["d_model"]), int(j["entry_count"])
    emb = _blob(os.path.join(path, "embeddings.f64"), n * d).reshape(n, d)
    ppath = os.path.join(path, "patterns.u32")
    pats = np.fromfile(ppath, dtype=np.uint32) if os.path.exists(ppath) else np.zeros(0, np.uint32)
    cache = PatternCache(d, int(j["capacity"]), float(j["min_similarity"]))
    entries = []
    for ei, e in enumerate(j["entries"]):
        sel = {}
        for t in e["tensors"]:
            off, k = int(t["offset"]), int(t["K"])
            sel[t["id"]] = RankSelection(pats[off:off + k].copy())
        entries.append(CacheEntry(PromptEmbedding(emb[ei].copy(), e.get("source", "")), sel))
    cache.load(entries)
    return cache
