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

import ctypes as C
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


class PeerReduceLinear:
    """Expert-sharded decode (config 5) with the all-reduce fused into the
    rank-expert kernel over peer memory (pg_agg_forward_peer): every rank
    computes its partial A_{S∩E_g}(B_{S∩E_g}^T x) in the decode chain, whose
    stage-2 epilogue pushes each output row's partial as a tagged word into all
    ranks' receive buffers (NVLink peer memory); each CTA then sums its rows
    over the ranks in rank order.  No NCCL call, no fence, and the result is
    bit-identical on every rank.  T = 1 tokens (decode); prefill chunks go
    through ShardedLinear.

    Receive buffers are exchanged as CUDA IPC handles over `group` (any
    torch.distributed backend), or passed in `peer_ptrs` when the ranks live in
    one process (tests: virtual ranks on one GPU, each on its own stream with a
    grid small enough that all ranks' kernels are co-resident)."""

    def __init__(self, A, B, world: int, rank: int, dtype="bf16", group=None, grid: int = 0, psi: float = 0.9):
        from .api import FactorizedLayer, call
        if not 1 <= world <= 8:
            raise ValueError("PeerReduceLinear: 1..8 ranks")
        self.shard = shard_layer(np.asarray(A, dtype=np.float64), np.asarray(B, dtype=np.float64), world, rank)
        self.world, self.rank, self.grid, self.psi = world, rank, grid, psi
        self.m, self.n = self.shard.A.shape[0], self.shard.B.shape[0]
        self.local = FactorizedLayer(self.shard.A, self.shard.B, None, dtype=dtype)
        nb = C.c_size_t()
        call("pg_peer_buffer_bytes", self.m, world, C.byref(nb))
        self.recv = torch.zeros(nb.value // 8, dtype=torch.int64, device="cuda")  # tags start at 1: zero = empty
        self.peer_ptrs = None
        self._opened = []
        self._aggs = {}
        self._last = None
        self._zero = None
        if group is not None and world > 1:
            self._exchange(group)

    def _exchange(self, group):
        import torch.distributed as dist
        from .api import call
        h = (C.c_char * 64)()
        call("pg_ipc_get_handle", C.c_void_p(self.recv.data_ptr()), h)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=group)
        ptrs = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                ptrs.append(self.recv.data_ptr())
                continue
            p = C.c_void_p()
            call("pg_ipc_open_handle", (C.c_char * 64).from_buffer_copy(hb), C.byref(p))
            self._opened.append(p)
            ptrs.append(p.value)
        self.peer_ptrs = ptrs

    @staticmethod
    def local_group(A, B, world: int, dtype="bf16", grid: int = 0) -> list:
        """All ranks in this process (virtual ranks sharing one device)."""
        ranks = [PeerReduceLinear(A, B, world, r, dtype=dtype, grid=grid) for r in range(world)]
        ptrs = [r.recv.data_ptr() for r in ranks]
        for r in ranks:
            r.peer_ptrs = ptrs
        return ranks

    def prepare(self, sel):
        """Pack this rank's share of the selection (reused across decode steps)."""
        return _prepare_shard(self, sel)

    def forward(self, sel, x: torch.Tensor, out_dtype=torch.float32, out=None, stream=None) -> torch.Tensor:
        from .api import _TORCH, _dtype_code, _ptr, call
        if self.peer_ptrs is None:
            raise RuntimeError("PeerReduceLinear: receive buffers not exchanged")
        agg = self.prepare(sel)
        x = x.reshape(-1)
        if x.numel() != self.n:
            raise ValueError("PeerReduceLinear: one token (x of n elements)")
        x = x.to(self.local.torch_dtype).contiguous()
        ydt = _dtype_code(out_dtype)
        y = out if out is not None else torch.empty(self.m, dtype=_TORCH[ydt], device=x.device)
        ptrs = (C.c_void_p * self.world)(*self.peer_ptrs)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        call("pg_agg_forward_peer", agg.handle, 0, _ptr(x), _ptr(y), ydt, self.rank, self.world, ptrs, self.grid, st)
        return y

    def close(self):
        from .api import call
        for p in self._opened:
            call("pg_ipc_close", p)
        self._opened = []


def _prepare_shard(h, sel):
    """Aggregated layout of this rank's share S ∩ E_rank of a selection (cached
    per selection; `h` carries shard / local / m / n / psi and the caches)."""
    from .api import FactorizedLayer, RankSelection, aggregate_layout
    if h._last is not None and h._last[0] is sel:  # decode steps reuse the same selection object
        return h._last[1]
    key = tuple(int(v) for v in np.asarray(sel.indices if hasattr(sel, "indices") else sel))
    if key not in h._aggs:
        mine = shard_selection(np.asarray(key, dtype=np.int64), h.world, h.rank)
        if mine.size == 0:
            # this rank owns none of the selected experts: it still launches
            # (the other ranks wait for its pushes) and pushes exact zeros,
            # through a one-expert all-zero layer of the same m x n
            if h._zero is None:
                h._zero = FactorizedLayer(np.zeros((h.m, 1)), np.zeros((h.n, 1)), 1, dtype=h.local.dtype)
            h._aggs[key] = aggregate_layout(h._zero, [RankSelection(np.zeros(1, dtype=np.uint32))], h.psi)
        else:
            h._aggs[key] = aggregate_layout(h.local, [RankSelection(h.shard.local_ids(mine))], h.psi)
    h._last = (sel, h._aggs[key])
    return h._aggs[key]


class _ShardHolder:
    """One linear's expert shard inside PeerReduceMLP (see _prepare_shard)."""

    def __init__(self, A, B, world, rank, dtype, psi):
        from .api import FactorizedLayer
        self.shard = shard_layer(np.asarray(A, dtype=np.float64), np.asarray(B, dtype=np.float64), world, rank)
        self.world, self.rank, self.psi = world, rank, psi
        self.m, self.n = self.shard.A.shape[0], self.shard.B.shape[0]
        self.local = FactorizedLayer(self.shard.A, self.shard.B, None, dtype=dtype)
        self._aggs, self._last, self._zero = {}, None, None


class PeerReduceMLP(PeerReduceLinear):
    """Expert-sharded MLP block (config 5 decode) in ONE decode-chain launch
    per rank (pg_mlp_forward_peer): up and gate partials are pushed to every
    rank's receive buffer and summed in rank order per act row, so every rank
    forms the whole act = silu(gate) * up (toy_lm.hpp:250-257) for its down
    shard; down's partials are then reduced the same way.  No NCCL call; the
    result is identical on every rank.  `up`, `gate`, `down` are (A, B) factor
    pairs (A m x r_store, B n x r_store); selections are global expert ids."""

    def __init__(self, up, gate, down, world: int, rank: int, dtype="bf16", group=None, grid: int = 0,
                 psi: float = 0.9):
        from .api import call
        if not 1 <= world <= 8:
            raise ValueError("PeerReduceMLP: 1..8 ranks")
        self.lins = [_ShardHolder(A, B, world, rank, dtype, psi) for A, B in (up, gate, down)]
        u, g, d = self.lins
        if u.m != g.m or u.n != g.n or d.n != u.m:
            raise ValueError("PeerReduceMLP: shape mismatch (up/gate m x n, down n x m)")
        self.world, self.rank, self.grid, self.psi = world, rank, grid, psi
        self.m, self.n, self.m_ff = d.m, u.n, u.m
        self.local = u.local
        nb = C.c_size_t()
        call("pg_peer_buffer_bytes", 2 * self.m_ff + self.m, world, C.byref(nb))
        self.recv = torch.zeros(nb.value // 8, dtype=torch.int64, device="cuda")  # tags start at 1: zero = empty
        self.peer_ptrs = None
        self._opened = []
        if group is not None and world > 1:
            self._exchange(group)

    @staticmethod
    def local_group(up, gate, down, world: int, dtype="bf16", grid: int = 0) -> list:
        """All ranks in this process (virtual ranks sharing one device)."""
        ranks = [PeerReduceMLP(up, gate, down, world, r, dtype=dtype, grid=grid) for r in range(world)]
        ptrs = [r.recv.data_ptr() for r in ranks]
        for r in ranks:
            r.peer_ptrs = ptrs
        return ranks

    def prepare(self, sels):
        """Pack this rank's share of the (up, gate, down) selections."""
        return [_prepare_shard(h, s) for h, s in zip(self.lins, sels)]

    def forward(self, sels, x: torch.Tensor, out_dtype=torch.float32, out=None, act=None,
                stream=None) -> torch.Tensor:
        from .api import _TORCH, _dtype_code, _ptr, call
        if self.peer_ptrs is None:
            raise RuntimeError("PeerReduceMLP: receive buffers not exchanged")
        aggs = self.prepare(sels)
        x = x.reshape(-1)
        if x.numel() != self.n:
            raise ValueError("PeerReduceMLP: one token (x of n elements)")
        x = x.to(self.local.torch_dtype).contiguous()
        ydt = _dtype_code(out_dtype)
        y = out if out is not None else torch.empty(self.m, dtype=_TORCH[ydt], device=x.device)
        if act is not None and (act.numel() != self.m_ff or act.dtype != self.local.torch_dtype):
            raise ValueError("PeerReduceMLP: act must hold m_ff elements of the weight dtype")
        ptrs = (C.c_void_p * self.world)(*self.peer_ptrs)
        pats = (C.c_size_t * 3)(0, 0, 0)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        call("pg_mlp_forward_peer", aggs[0].handle, aggs[1].handle, aggs[2].handle, pats, _ptr(x),
             _ptr(act) if act is not None else None, _ptr(y), ydt, self.rank, self.world, ptrs, self.grid, st)
        return y


class PeerBuffer:
    """A zeroed receive buffer for the fused peer reductions
    (pg_agg_forward_peer: words = m; pg_mlp_forward_peer: words = 2 m_ff + d)
    with every rank's buffer pointer, exchanged as CUDA IPC handles over
    `group` (one process per GPU).  `ptrs` is what the C-ABI takes."""

    def __init__(self, words: int, world: int, rank: int, group=None):
        from .api import call
        nb = C.c_size_t()
        call("pg_peer_buffer_bytes", words, world, C.byref(nb))
        self.world, self.rank = world, rank
        self.recv = torch.zeros(nb.value // 8, dtype=torch.int64, device="cuda")
        self._opened = []
        self.peer_ptrs = [self.recv.data_ptr()] if world == 1 else None
        if group is not None and world > 1:
            PeerReduceLinear._exchange(self, group)

    @property
    def ptrs(self):
        return (C.c_void_p * self.world)(*self.peer_ptrs)

    def close(self):
        PeerReduceLinear.close(self)
