"""Prompt embedding on the device: embed_prompt
(pattern_cache.hpp:50-65) = the block-0 output of the static-prefix model
(FactorizedProvider without a map, pattern_cache.hpp:84 / model.hpp:55-63),
mean-pooled over the prompt and L2-normalised.  Drives pattern-cache
retrieval from tokens instead of from given embeddings.

Block 0 of forward_lm (toy_lm.hpp:219-258) in f64 on the GPU: the seven
projections run through the rank-expert kernels (masked_forward over the
prefix selection {0..K-1}); RMSNorm (toy_lm.hpp:116-132), RoPE (:134-150) and
causal attention (:165-194) are the block's glue around them, computed with
torch f64 ops in the reference's formulas (attention is outside the
north-star hot path).  The pooling + normalisation is the exact-order kernel
(``embed_pool``).  Values agree with the reference to rounding (sequential vs
tree summation in the projections); the committed fixture bounds it at 1e-12.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .api import PromptEmbedding, RankSelection, embed_pool, masked_forward, tensor_id

RMS_EPS = 1e-5      # toy_lm.hpp:38
ROPE_BASE = 10000.0  # toy_lm.hpp:39


def _rmsnorm(h: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """rmsnorm (toy_lm.hpp:116-132): per column x * g / sqrt(mean(x^2) + eps)."""
    r = torch.sqrt((h * h).sum(dim=0, keepdim=True) / h.shape[0] + RMS_EPS)
    return g[:, None] * h / r


def _rope(x: torch.Tensor, head_dim: int, pos0: int = 0) -> torch.Tensor:
    """rope_inplace (toy_lm.hpp:134-150): rotate adjacent pairs within each head."""
    d, T = x.shape
    j = torch.arange(0, head_dim - 1, 2, dtype=torch.float64, device=x.device)
    inv = torch.pow(torch.tensor(ROPE_BASE, dtype=torch.float64, device=x.device), -j / head_dim)
    p = torch.arange(pos0, pos0 + T, dtype=torch.float64, device=x.device)
    th = p[None, :] * inv[:, None]                       # [hd/2, T]
    c, s = torch.cos(th), torch.sin(th)
    xr = x.view(d // head_dim, head_dim // 2, 2, T)
    x0, x1 = xr[:, :, 0, :], xr[:, :, 1, :]
    out = torch.empty_like(xr)
    out[:, :, 0, :] = c * x0 - s * x1
    out[:, :, 1, :] = s * x0 + c * x1
    return out.view(d, T)


def _attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, n_heads: int, n_kv: int) -> torch.Tensor:
    """Causal attention of a prefill (toy_lm.hpp:165-194), heads grouped for GQA."""
    d, T = q.shape
    hd = d // n_heads
    group = n_heads // n_kv
    qh = q.view(n_heads, hd, T)
    kh = k.view(n_kv, hd, T).repeat_interleave(group, dim=0)
    vh = v.view(n_kv, hd, T).repeat_interleave(group, dim=0)
    sc = torch.einsum("hdt,hds->hts", qh, kh) * (1.0 / math.sqrt(hd))
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=q.device), diagonal=1)
    sc = sc.masked_fill(mask, float("-inf"))
    pr = torch.softmax(sc, dim=-1)
    return torch.einsum("hts,hds->hdt", pr, vh).reshape(d, T)


def block0_forward(model, tokens, selections: dict | None = None) -> torch.Tensor:
    """Block-0 output h (d x T, f64, device) of forward_lm over `tokens` with
    the static-prefix provider (or `selections`, a SelectionMap)."""
    cfg = model.lm_config
    d, nh, nkv = int(cfg["d_model"]), int(cfg["n_heads"]), int(cfg["n_kv_heads"])
    if len(tokens) == 0:
        raise ValueError("embed_prompt: empty prompt")
    dev = torch.device("cuda")
    emb = torch.from_numpy(np.asarray(model.core["embed"], dtype=np.float64)).to(dev)
    g_attn = torch.from_numpy(np.asarray(model.core["b0.attn_norm"], dtype=np.float64)).to(dev)
    g_mlp = torch.from_numpy(np.asarray(model.core["b0.mlp_norm"], dtype=np.float64)).to(dev)
    tok = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=dev)
    h = emb[tok].t().contiguous()  # d x T

    def proj(p, x):
        tid = tensor_id(0, p)
        layer = model.layers[tid]
        sel = (selections or {}).get(tid) or RankSelection(np.arange(layer.K, dtype=np.uint32))
        return masked_forward(layer, sel, x.contiguous(), out_dtype=torch.float64).double()

    hn = _rmsnorm(h, g_attn)
    q, k, v = proj("q", hn), proj("k", hn), proj("v", hn)
    hd = d // nh
    q, k = _rope(q, hd), _rope(k, hd)
    h = h + proj("o", _attention(q, k, v, nh, nkv))
    hn2 = _rmsnorm(h, g_mlp)
    up, gate = proj("up", hn2), proj("gate", hn2)
    act = up * gate / (1.0 + torch.exp(-gate))
    return h + proj("down", act)


def embed_prompt(model, tokens, source: str = "") -> PromptEmbedding:
    """embed_prompt (pattern_cache.hpp:50-65) on the device."""
    return embed_pool(block0_forward(model, tokens), layout="feature", source=source)
