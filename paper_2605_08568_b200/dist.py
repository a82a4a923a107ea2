"""Multi-GPU plumbing for the rank-expert path.

One process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU tests).

* Data parallel (configs 2-4): prompts are independent given replicated
  weights, routers and pattern cache, so each rank serves a disjoint subset of
  the prompt batch and no collective touches the data path.
  ``partition_prompts`` splits contiguously; ``partition_by_pattern`` keeps
  every prompt that shares a cache pattern on one rank (pattern affinity: that
  rank packs the pattern's experts once) while balancing prompt counts.
* Expert-sharded (config 5): expert e lives on rank e mod G.  Rank g computes
  the partial y_g = A_{S∩E_g} (B_{S∩E_g}^T x) over its share of the prompt's
  selection S and the partials are summed with one all-reduce per linear.
  Selection is unchanged (bit-exact); values differ from the single-GPU
  result only by the reduction order.  ``shard_layer`` keeps just the rank's
  expert columns (storage and HBM bytes / G).

The reference (single-process C++) has no multi-GPU path; this is the
north star's scale-out of its serving loop (model.hpp:96-106 per prompt).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


def partition_prompts(n_prompts: int, world: int, rank: int) -> range:
    """Contiguous, balanced prompt range of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("partition_prompts: bad rank / world")
    lo = n_prompts * rank // world
    hi = n_prompts * (rank + 1) // world
    return range(lo, hi)


def partition_by_pattern(pattern_ids, world: int) -> list[list[int]]:
    """Pattern affinity: prompts that share a cache pattern go to the same rank.
    Groups are placed largest-first on the currently lightest rank (ties to the
    lower rank), so the assignment is deterministic.  Returns, per rank, the
    prompt indices in ascending order."""
    if world < 1:
        raise ValueError("partition_by_pattern: bad world size")
    groups: dict[int, list[int]] = {}
    for i, p in enumerate(pattern_ids):
        groups.setdefault(int(p), []).append(i)
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for pid, idx in sorted(groups.items(), key=lambda kv: (-len(kv[1]), kv[0])):
        g = min(range(world), key=lambda r: (load[r], r))
        out[g].extend(idx)
        load[g] += len(idx)
    return [sorted(v) for v in out]


def expert_owner(expert: int, world: int) -> int:
    """Interleaved expert placement (e mod G) -- balanced for prefix-biased S."""
    return int(expert) % world


def shard_selection(sel, world: int, rank: int) -> np.ndarray:
    """S ∩ E_rank in ascending global ids."""
    s = np.asarray(sel.indices if hasattr(sel, "indices") else sel, dtype=np.int64)
    return s[s % world == rank].astype(np.uint32)


@dataclass
class ExpertShard:
    """Rank-local columns of a factorized layer: A[:, E_g], B[:, E_g] with the
    global -> local expert map (global e -> e // G on rank e mod G)."""
    A: object
    B: object
    world: int
    rank: int
    r_store: int

    def local_ids(self, global_ids) -> np.ndarray:
        g = np.asarray(global_ids, dtype=np.int64)
        if np.any(g % self.world != self.rank):
            raise ValueError("expert not owned by this rank")
        return (g // self.world).astype(np.uint32)


def shard_layer(A, B, world: int, rank: int) -> ExpertShard:
    """Keep only this rank's experts (columns e with e mod G == rank) of the
    absorbed factors A (m x r_store) and B (n x r_store) (factorize.hpp:28-37)."""
    r = A.shape[1]
    if B.shape[1] != r:
        raise ValueError("shard_layer: A and B disagree on r_store")
    cols = np.arange(rank, r, world)
    if isinstance(A, torch.Tensor):
        idx = torch.as_tensor(cols, device=A.device)
        return ExpertShard(A.index_select(1, idx).contiguous(), B.index_select(1, idx).contiguous(), world, rank, r)
    return ExpertShard(np.ascontiguousarray(A[:, cols]), np.ascontiguousarray(B[:, cols]), world, rank, r)


def sharded_forward(shard: ExpertShard, sel, x: torch.Tensor, forward, group=None) -> torch.Tensor:
    """Expert-sharded rank-expert linear: partial over S ∩ E_g, then an
    all-reduce (sum) across the group.  `forward(shard, local_ids, x)` computes
    A_loc[:, ids] (B_loc[:, ids]^T x) on this rank (the product passes the
    GPU path, e.g. a FactorizedLayer built from the shard + masked_forward);
    an empty local selection contributes zeros."""
    import torch.distributed as dist

    mine = shard_selection(sel, shard.world, shard.rank)
    y = forward(shard, shard.local_ids(mine), x) if mine.size else None
    if y is None:
        m = shard.A.shape[0]
        shape = (m,) if x.dim() == 1 else (m, x.shape[1])
        y = torch.zeros(shape, dtype=torch.float64 if x.dtype == torch.float64 else torch.float32, device=x.device)
    if shard.world > 1:
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
    return y


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing across the job (identity without a process group)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ShardedLinear:
    """Expert-sharded rank-expert linear on the GPU (config 5): this rank's
    expert columns as a device FactorizedLayer, the partial through the
    rank-expert kernels (masked_forward), the sum through one NCCL all-reduce.
    A, B: the full absorbed factors (host f64), sharded here."""

    def __init__(self, A, B, world: int, rank: int, dtype="bf16", group=None):
        from .api import FactorizedLayer
        self.shard = shard_layer(np.asarray(A, dtype=np.float64), np.asarray(B, dtype=np.float64), world, rank)
        self.world, self.rank, self.group = world, rank, group
        self.m, self.n = self.shard.A.shape[0], self.shard.B.shape[0]
        self.local = FactorizedLayer(self.shard.A, self.shard.B, None, dtype=dtype)

    def forward(self, sel, x: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
        from .api import RankSelection, masked_forward

        def fwd(_shard, local_ids, xt):
            return masked_forward(self.local, RankSelection(np.asarray(local_ids, dtype=np.uint32)), xt,
                                  out_dtype=out_dtype)

        return sharded_forward(self.shard, sel, x, fwd, group=self.group)
