"""Offline router training on the GPU: the
reference's ``train_router_matrix`` (router.hpp:318-400) on cached
per-sequence statistics (router.hpp:204-270), in f64 on the device.

Per sequence only Z = B^T X (r x T), P = A^T Y (r x T), the pooled input h and
||Y||^2 are kept; with the Gram matrix G = A^T A every loss and gate gradient
is a small product:
  selection_loss  = sum_t z_S^T G_SS z_S - 2 <P_S, Z_S> + ||Y||^2      (:224-236)
  hard gate grad  g_i = 2 (z_i . (G_{i,S} Z_S) - p_i . z_i)             (:239-253)
  soft gate grad  g_i = 2 (z_i . (G_{i,:} diag(w) Z) - p_i . z_i)       (:256-270)
chained through the soft mask (router.hpp:100-122), AdamW (:143-171) on a
cosine schedule with warmup (:174-179), deterministic Fisher-Yates over the
reference's splitmix64 stream, best-epoch checkpointing (zero init = the
static prefix, so the result is never worse than static on the training set).
Selections use the reference's top-K (ties to the lower index, ascending).
Offline, so the batched products go through torch (cuBLAS) rather than
hand-written kernels; the serving path is untouched.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

_M64 = (1 << 64) - 1


class Rng:
    """rng.hpp:10-41 (splitmix64): the reference's shuffle stream, bit-exact."""

    def __init__(self, seed: int = 0):
        self.state = seed & _M64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        return self.next_u64() % n

    def gaussian(self) -> float:
        u1, u2 = self.uniform(), self.uniform()
        while u1 <= 0:
            u1 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)


@dataclass
class RouterTrainConfig:
    """router.hpp:22-29."""
    learning_rate: float = 2e-4
    weight_decay: float = 1e-3
    warmup_frac: float = 0.1
    epochs: int = 5
    batch_size: int = 64
    seed: int = 0


@dataclass
class RouterSeqStats:
    """router.hpp:204-209 (device tensors)."""
    h: torch.Tensor   # [n]
    z: torch.Tensor   # [r, T]
    p: torch.Tensor   # [r, T]
    y_sq: float


@dataclass
class RouterTrainResult:
    theta: torch.Tensor
    bias: torch.Tensor
    epoch_loss: list = field(default_factory=list)
    frozen_loss: list = field(default_factory=list)


def precompute_router_stats(A: torch.Tensor, B: torch.Tensor, x: torch.Tensor, y: torch.Tensor) -> RouterSeqStats:
    """router.hpp:211-219: h = mean_pool(x) (reference order), Z = B^T x, P = A^T y."""
    from .api import mean_pool
    x = x.to(torch.float64)
    y = y.to(torch.float64)
    return RouterSeqStats(mean_pool(x, layout="feature"), B.t() @ x, A.t() @ y, float((y * y).sum()))


def select_topk(logits: torch.Tensor, k: int) -> torch.Tensor:
    """router.hpp:49-61 for a batch of logit rows [S, r]: K largest, ties to
    the lower index (stable descending sort), returned ascending."""
    order = torch.sort(logits, dim=-1, descending=True, stable=True).indices[..., :k]
    return torch.sort(order, dim=-1).values


def _soft_mask(logits, k, tau, eps):
    s = torch.sigmoid(logits / tau)
    return k * s / (s.sum(dim=-1, keepdim=True) + eps)


def _chain_soft_mask(logits, g_m, k, tau, eps):
    """router.hpp:100-122 (batched)."""
    s = torch.sigmoid(logits / tau)
    sp = s * (1.0 - s) / tau
    denom = s.sum(dim=-1, keepdim=True) + eps
    gs = (g_m * s).sum(dim=-1, keepdim=True)
    return k * sp / denom * (g_m - gs / denom)


def _selection_loss(G, st: RouterSeqStats, sel):
    zs = st.z[sel]
    return float((zs * (G[sel][:, sel] @ zs)).sum() - 2.0 * (st.p[sel] * zs).sum() + st.y_sq)


def train_router_matrix(A, B, K: int, seqs: list, cfg: RouterTrainConfig, tau: float = 1.0,
                        eps: float = 1e-8) -> RouterTrainResult:
    """router.hpp:318-400 on the device."""
    if not seqs:
        raise ValueError("train_router: empty corpus")
    A = torch.as_tensor(A, dtype=torch.float64, device="cuda")
    B = torch.as_tensor(B, dtype=torch.float64, device="cuda")
    r, n = A.shape[1], B.shape[0]
    G = A.t() @ A
    theta = torch.zeros(r, n, dtype=torch.float64, device="cuda")
    bias = torch.zeros(r, dtype=torch.float64, device="cuda")
    m_t, v_t = torch.zeros_like(theta), torch.zeros_like(theta)
    m_b, v_b = torch.zeros_like(bias), torch.zeros_like(bias)
    b1, b2, aeps = 0.9, 0.999, 1e-8
    H = torch.stack([s.h for s in seqs])  # [S, n]
    nb = (len(seqs) + cfg.batch_size - 1) // cfg.batch_size
    total = cfg.epochs * nb
    step = 0
    order = list(range(len(seqs)))
    rng = Rng(cfg.seed)

    def eval_pass(th, bb):
        sel = select_topk(H @ th.t() + bb, K)
        return sum(_selection_loss(G, st, sel[i]) for i, st in enumerate(seqs)) / len(seqs)

    best = (theta.clone(), bias.clone())
    best_loss = eval_pass(theta, bias)
    res = RouterTrainResult(theta, bias)
    for _ in range(cfg.epochs):
        for i in range(len(order), 1, -1):  # deterministic Fisher-Yates (rng.hpp stream)
            j = rng.below(i)
            order[i - 1], order[j] = order[j], order[i - 1]
        epoch_loss = 0.0
        for b0 in range(0, len(order), cfg.batch_size):
            idx = order[b0: b0 + cfg.batch_size]
            gt = torch.zeros_like(theta)
            gb = torch.zeros_like(bias)
            soft = step < cfg.warmup_frac * total
            for si in idx:
                st = seqs[si]
                logits = theta @ st.h + bias
                sel = select_topk(logits[None], K)[0]
                epoch_loss += _selection_loss(G, st, sel)
                pz = (st.p * st.z).sum(dim=1)
                if soft:  # residual at the soft reconstruction during warmup
                    w = _soft_mask(logits, K, tau, eps)
                    mz = (G * w[None, :]) @ st.z
                else:
                    mz = G[:, sel] @ st.z[sel]
                g_m = 2.0 * ((st.z * mz).sum(dim=1) - pz)
                gl = _chain_soft_mask(logits, g_m, K, tau, eps)
                gb += gl
                gt += gl[:, None] * st.h[None, :]
            inv = 1.0 / len(idx)
            gt *= inv
            gb *= inv
            warm = max(1.0, cfg.warmup_frac * total)
            if step < warm:
                lr = cfg.learning_rate * (step + 1) / warm
            else:
                prog = (step - warm) / max(1.0, total - warm)
                lr = cfg.learning_rate * 0.5 * (1.0 + math.cos(math.pi * min(1.0, prog)))
            step += 1  # AdamW (router.hpp:143-171): decoupled decay, none on the bias
            bc1, bc2 = 1.0 - b1 ** step, 1.0 - b2 ** step
            m_t.mul_(b1).add_((1 - b1) * gt)
            v_t.mul_(b2).add_((1 - b2) * gt * gt)
            theta -= lr * (m_t / bc1 / (torch.sqrt(v_t / bc2) + aeps) + cfg.weight_decay * theta)
            m_b.mul_(b1).add_((1 - b1) * gb)
            v_b.mul_(b2).add_((1 - b2) * gb * gb)
            bias -= lr * (m_b / bc1 / (torch.sqrt(v_b / bc2) + aeps))
        res.epoch_loss.append(epoch_loss / len(seqs))
        fl = eval_pass(theta, bias)
        res.frozen_loss.append(fl)
        if fl < best_loss:
            best_loss, best = fl, (theta.clone(), bias.clone())
    res.theta, res.bias = best
    return res
