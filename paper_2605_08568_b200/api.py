"""Python mirror of the reference's hot-path API over the sm_100a C-ABI.

Names, argument meaning and error classes follow /root/reference/proj/include/parse:
  router.hpp        RouterParams, mean_pool, score, select_topk          (:15-20,41-61,80-88)
  pattern_cache.hpp PatternCache, CacheEntry, PromptEmbedding, RetrieveResult,
                    cosine, retrieve, cache_insert, embed_prompt pooling  (:31-36,38-65,95-124)
  rank_experts.hpp  RankSelection, check_selection, masked_forward       (:13-37,52-72)
  factorize.hpp     FactorizedLayer, store_rank                           (:28-37,86-89)
  exec_engine.hpp   aggregate_layout, aggregated_forward, scattered_forward,
                    ExecEngine, ExecVariant, build_plan, maximal_runs, AccessTrace
  model.hpp         FactorizedModel, FactorizedProvider, RoutingProvider (:18-126)

Activations are torch CUDA tensors.  As in the reference, X is feature-major
(n x T) unless layout="token" (T x n).  Every compute call runs a kernel from
libparse_gpu.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import PG_BF16, PG_F32, PG_F64, PG_FEATURE_MAJOR, PG_TOKEN_MAJOR, call

_DT = {torch.float64: PG_F64, torch.float32: PG_F32, torch.bfloat16: PG_BF16}
_TORCH = {PG_F64: torch.float64, PG_F32: torch.float32, PG_BF16: torch.bfloat16}
_NAMES = {"f64": PG_F64, "f32": PG_F32, "bf16": PG_BF16, "float64": PG_F64, "float32": PG_F32,
          "bfloat16": PG_BF16}


def _dtype_code(dt) -> int:
    if isinstance(dt, int):
        return dt
    if isinstance(dt, torch.dtype):
        return _DT[dt]
    return _NAMES[str(dt)]


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _dev(x, dtype=None) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    x = torch.as_tensor(x)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.cuda().contiguous() if not x.is_cuda else x.contiguous()


def _layout(layout: str) -> int:
    if layout in ("feature", "feature_major", "nT"):
        return PG_FEATURE_MAJOR
    if layout in ("token", "token_major", "Tn"):
        return PG_TOKEN_MAJOR
    raise ValueError(f"unknown layout {layout!r}")


# ---------------------------------------------------------------- shapes
def store_rank(k: int, r_max: int, store_multiplier: float = 2.0) -> int:
    """factorize.hpp:86-89."""
    want = int(np.ceil(store_multiplier * float(k)))
    return min(r_max, max(k, want))


def single_layer_k(m: int, n: int, ratio: float) -> int:
    """allocate_budgets (factorize.hpp:135-195) for one layer: largest K with
    K*(m+n) <= (1-ratio)*m*n, K >= 1, K <= min(m, n)."""
    budget = (1.0 - ratio) * (float(m) * float(n))
    cost = float(m + n)
    k, used = 1, cost
    if used > budget:
        raise RuntimeError("ratio too aggressive for K≥1 floor")
    k = max(1, min(min(m, n), int(budget // cost)))
    while k > 1 and k * cost > budget:
        k -= 1
    while k < min(m, n) and (k + 1) * cost <= budget:
        k += 1
    return k


# ---------------------------------------------------------------- selections
@dataclass
class RankSelection:
    """rank_experts.hpp:13-28: strictly increasing expert ids."""
    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint32))

    def __post_init__(self):
        self.indices = np.ascontiguousarray(np.asarray(self.indices, dtype=np.uint32))

    def K(self) -> int:
        return int(self.indices.size)

    def contains(self, i: int) -> bool:
        j = np.searchsorted(self.indices, i)
        return bool(j < self.indices.size and self.indices[j] == i)

    @staticmethod
    def prefix(k: int) -> "RankSelection":
        return RankSelection(np.arange(k, dtype=np.uint32))

    def __eq__(self, other):
        return isinstance(other, RankSelection) and np.array_equal(self.indices, other.indices)


def check_selection(layer: "FactorizedLayer", sel: RankSelection) -> None:
    """rank_experts.hpp:30-37 (ValueError / IndexError as invalid_argument / out_of_range)."""
    s = np.ascontiguousarray(sel.indices, dtype=np.uint32)
    call("pg_check_selection", layer.handle, s.ctypes.data_as(C.POINTER(C.c_uint32)), s.size)


# ---------------------------------------------------------------- router
class RouterParams:
    """router.hpp:15-20 -- theta r x n (f64), bias r, on device."""

    def __init__(self, theta, bias=None, tau: float = 1.0, eps: float = 1e-8):
        if isinstance(theta, torch.Tensor) and theta.is_cuda:
            self.theta = theta.to(torch.float64).contiguous()
            r, n = self.theta.shape
            self.bias = (torch.zeros(r, dtype=torch.float64, device=theta.device) if bias is None
                         else _dev(bias, torch.float64))
        else:
            th = np.ascontiguousarray(theta, dtype=np.float64)
            r, n = th.shape
            self.theta = torch.from_numpy(th).cuda()
            self.bias = _dev(np.zeros(r) if bias is None else np.asarray(bias, dtype=np.float64), torch.float64)
        self.r, self.n = int(r), int(n)
        self.tau, self.eps = tau, eps
        h = C.c_void_p()
        call("pg_router_create_device", C.byref(h), self.r, self.n, self.theta.data_ptr(),
             self.bias.data_ptr(), 0)
        self.handle = h

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.lib().pg_router_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass


def make_router(r: int, n: int, tau: float = 1.0, eps: float = 1e-8) -> RouterParams:
    """router.hpp:31-39: zero init -> first selection is the static prefix."""
    return RouterParams(np.zeros((r, n)), np.zeros(r), tau, eps)


def mean_pool(x: torch.Tensor, layout: str = "feature", offsets=None) -> torch.Tensor:
    """router.hpp:80-88, bit-exact.  x: n x T (feature) or T x n (token).
    offsets (token-major batches): P+1 token offsets -> returns P x n."""
    lay = _layout(layout)
    x = _dev(x)
    if lay == PG_FEATURE_MAJOR:
        n, T = x.shape
    else:
        T, n = x.shape
    offs = np.asarray([0, T] if offsets is None else offsets, dtype=np.int64)
    P = offs.size - 1
    h = torch.empty((P, n), dtype=torch.float64, device=x.device)
    call("pg_mean_pool", _ptr(x), _dtype_code(x.dtype), lay, n, offs.ctypes.data_as(C.POINTER(C.c_int64)), P,
         _ptr(h), _stream())
    return h[0] if offsets is None else h


def score(router: RouterParams, h: torch.Tensor, exact: bool = True) -> torch.Tensor:
    """router.hpp:41-46.  exact=True: reference-order dot (bit-identical)."""
    h = _dev(h, torch.float64)
    if h.shape[-1] != router.n:
        raise ValueError("score: bad input length")
    P = 1 if h.dim() == 1 else h.shape[0]
    z = torch.empty((P, router.r), dtype=torch.float64, device=h.device)
    call("pg_score", router.handle, _ptr(h), P, _ptr(z), int(exact), _stream())
    return z[0] if h.dim() == 1 else z


def select_topk(logits, k: int) -> RankSelection:
    """router.hpp:49-61: K largest, ties toward the lower index, ascending."""
    z = _dev(logits, torch.float64)
    r = z.shape[-1]
    out = torch.empty(max(k, 1), dtype=torch.int32, device=z.device)
    call("pg_select_topk", _ptr(z), r, 1, k, _ptr(out), _stream())
    return RankSelection(out[:k].cpu().numpy().astype(np.uint32))


def route_select(router: RouterParams, x: torch.Tensor, k: int, layout: str = "feature", offsets=None,
                 return_logits: bool = False):
    """RoutingProvider's routing step (model.hpp:102) fused on device:
    select_topk(score(theta, mean_pool(x)), k), bit-identical to the reference.
    Returns a device int32 tensor [P, k] (ascending ids) (+ logits [P, r])."""
    lay = _layout(layout)
    x = _dev(x)
    T = x.shape[1] if lay == PG_FEATURE_MAJOR else x.shape[0]
    offs = np.asarray([0, T] if offsets is None else offsets, dtype=np.int64)
    P = offs.size - 1
    sel = torch.empty((P, max(k, 1)), dtype=torch.int32, device=x.device)
    lg = torch.empty((P, router.r), dtype=torch.float64, device=x.device) if return_logits else None
    call("pg_route_select", router.handle, _ptr(x), _dtype_code(x.dtype), lay,
         offs.ctypes.data_as(C.POINTER(C.c_int64)), P, k, _ptr(sel), _ptr(lg) if lg is not None else None,
         _stream())
    return (sel, lg) if return_logits else sel


def route_select_pooled(router: RouterParams, h: torch.Tensor, k: int, return_logits: bool = False):
    """route_select from already pooled inputs h (P x n f64 device, mean_pool's
    output): linears sharing an input (q/k/v, up/gate; toy_lm.hpp:220-249) pool
    once.  Bit-identical to route_select on the same x."""
    h = _dev(h, torch.float64)
    if h.dim() == 1:
        h = h.unsqueeze(0)
    if h.shape[-1] != router.n:
        raise ValueError("score: bad input length")
    P = h.shape[0]
    sel = torch.empty((P, max(k, 1)), dtype=torch.int32, device=h.device)
    lg = torch.empty((P, router.r), dtype=torch.float64, device=h.device) if return_logits else None
    call("pg_route_select_pooled", router.handle, _ptr(h), P, k, _ptr(sel), _ptr(lg) if lg is not None else None,
         _stream())
    return (sel, lg) if return_logits else sel


# ---------------------------------------------------------------- pattern cache
@dataclass
class PromptEmbedding:
    vec: np.ndarray
    source: str = ""


@dataclass
class CacheEntry:
    embedding: PromptEmbedding
    pattern: dict = field(default_factory=dict)  # SelectionMap: tensor id -> RankSelection


@dataclass
class RetrieveResult:
    """pattern_cache.hpp:95-100."""
    pattern: dict | None = None
    entry: int = 0
    similarity: float = -2.0
    hit: bool = False
    exact_similarity: bool = False


class PatternCache:
    """pattern_cache.hpp:31-36; embeddings live on device (N x d f64)."""

    def __init__(self, d_model: int, capacity: int = 0, min_similarity: float = 0.0):
        self.d_model, self.capacity, self.min_similarity = int(d_model), int(capacity), float(min_similarity)
        self.entries: list[CacheEntry] = []
        h = C.c_void_p()
        call("pg_cache_create", C.byref(h), self.d_model, self.capacity, self.min_similarity)
        self.handle = h

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.lib().pg_cache_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass

    def load(self, entries: list[CacheEntry]) -> None:
        """Bulk load (load_cache, pattern_cache.hpp:294-327)."""
        emb = np.ascontiguousarray(np.stack([np.asarray(e.embedding.vec, dtype=np.float64) for e in entries])
                                   if entries else np.zeros((0, self.d_model)))
        call("pg_cache_load", self.handle, emb.ctypes.data_as(C.POINTER(C.c_double)), len(entries))
        self.entries = list(entries)


def cosine(a, b) -> float:
    """pattern_cache.hpp:38-47, reference order (bit-exact)."""
    a = _dev(a, torch.float64)
    b = _dev(b, torch.float64)
    if a.numel() != b.numel():
        raise ValueError("cosine: length mismatch")
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    call("pg_cosine", _ptr(a), _ptr(b), a.numel(), _ptr(out), _stream())
    return float(out.item())


def cache_insert(cache: PatternCache, entry: CacheEntry) -> bool:
    """pattern_cache.hpp:120-124: refused once at capacity (no eviction)."""
    v = np.ascontiguousarray(entry.embedding.vec, dtype=np.float64)
    ins = C.c_int(0)
    call("pg_cache_insert", cache.handle, v.ctypes.data, 0, C.byref(ins), _stream())
    if ins.value:
        cache.entries.append(entry)
    return bool(ins.value)


def retrieve(cache: PatternCache, emb, exact_similarity: bool = False) -> RetrieveResult:
    """pattern_cache.hpp:104-117: first maximum, hit = sim >= min_similarity."""
    vec = emb.vec if isinstance(emb, PromptEmbedding) else emb
    q = _dev(vec, torch.float64)
    res = _lib.RetrieveResultC()
    call("pg_retrieve", cache.handle, _ptr(q), int(exact_similarity), C.byref(res), None, None, _stream())
    e = int(res.entry)
    pat = cache.entries[e].pattern if e < len(cache.entries) else None
    return RetrieveResult(pat, e, float(res.similarity), bool(res.hit), bool(res.exact_similarity))


def retrieve_device(cache: PatternCache, query: torch.Tensor):
    """Device-resident retrieve: returns (entry int32[1], hit int32[1]) tensors
    without synchronising, for pattern_dev-driven forwards."""
    q = _dev(query, torch.float64)
    entry = torch.empty(1, dtype=torch.int32, device=q.device)
    hit = torch.empty(1, dtype=torch.int32, device=q.device)
    call("pg_retrieve", cache.handle, _ptr(q), 0, None, _ptr(entry), _ptr(hit), _stream())
    return entry, hit


def embed_pool(block_out: torch.Tensor, layout: str = "feature", source: str = "") -> PromptEmbedding:
    """embed_prompt's pooling half (pattern_cache.hpp:60-64): mean_pool of the
    block-0 output then L2-normalise; RuntimeError('degenerate embedding')."""
    lay = _layout(layout)
    x = _dev(block_out)
    d, T = (x.shape if lay == PG_FEATURE_MAJOR else x.shape[::-1])
    if T == 0:
        raise ValueError("embed_prompt: empty prompt")
    out = torch.empty(d, dtype=torch.float64, device=x.device)
    call("pg_embed_normalize", _ptr(x), _dtype_code(x.dtype), lay, d, T, _ptr(out), _stream())
    return PromptEmbedding(out.cpu().numpy(), source)


# ---------------------------------------------------------------- layers
class FactorizedLayer:
    """factorize.hpp:28-37 on device: expert-major B^T [r_store, n] and A [m, r_store]."""

    def __init__(self, A=None, B=None, K: int | None = None, dtype="f32", layer_id: str = "layer",
                 sigma=None, _handle=None, _shape=None, _keep=None):
        self.layer_id = layer_id
        self.sigma = sigma
        self._keep = _keep
        if _handle is not None:
            self.handle = _handle
            self.m, self.n, self.r_store, self.K, self.dtype = _shape
            return
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        m, r = A.shape
        n, r2 = B.shape
        if r != r2:
            raise ValueError("FactorizedLayer: A and B disagree on r_store")
        self.m, self.n, self.r_store = int(m), int(n), int(r)
        self.K = int(r if K is None else K)
        self.dtype = _dtype_code(dtype)
        h = C.c_void_p()
        call("pg_layer_create", C.byref(h), m, n, r, self.K, A.ctypes.data_as(C.POINTER(C.c_double)),
             B.ctypes.data_as(C.POINTER(C.c_double)), self.dtype)
        self.handle = h

    @classmethod
    def from_device(cls, bt: torch.Tensor, a: torch.Tensor, K: int, layer_id: str = "layer", copy: bool = False):
        """bt: [r_store, n], a: [m, r_store] CUDA tensors (f64/f32/bf16)."""
        r, n = bt.shape
        m, r2 = a.shape
        if r != r2 or bt.dtype != a.dtype:
            raise ValueError("FactorizedLayer.from_device: shape/dtype mismatch")
        dt = _dtype_code(bt.dtype)
        h = C.c_void_p()
        call("pg_layer_create_device", C.byref(h), m, n, r, K, _ptr(bt), _ptr(a), dt, int(copy))
        return cls(layer_id=layer_id, _handle=h, _shape=(int(m), int(n), int(r), int(K), dt),
                   _keep=None if copy else (bt, a))

    @property
    def torch_dtype(self):
        return _TORCH[self.dtype]

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.lib().pg_layer_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass


def _out_dtype(wdt: int, out_dtype):
    if out_dtype is None:
        return PG_F64 if wdt == PG_F64 else PG_F32
    return _dtype_code(out_dtype)


def masked_forward(layer: FactorizedLayer, sel, x: torch.Tensor, layout: str = "feature",
                   out_dtype=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """rank_experts.hpp:52-72: y = sum_{e in S} a_e (b_e^T x).  sel is a
    RankSelection (host, validated) or a device int32 tensor (trusted)."""
    lay = _layout(layout)
    x = _dev(x, layer.torch_dtype)
    if lay == PG_FEATURE_MAJOR:
        if x.dim() == 1:
            x = x.view(-1, 1)
        n, T = x.shape
    else:
        T, n = x.shape
    if n != layer.n:
        raise ValueError("masked_forward: bad X shape")
    ydt = _out_dtype(layer.dtype, out_dtype)
    shape = (layer.m, T) if lay == PG_FEATURE_MAJOR else (T, layer.m)
    y = out if out is not None else torch.empty(shape, dtype=_TORCH[ydt], device=x.device)
    if isinstance(sel, torch.Tensor):
        s = sel.reshape(-1).to(torch.int32).contiguous()
        call("pg_masked_forward", layer.handle, _ptr(s), s.numel(), 1, _ptr(x), lay, T, _ptr(y), ydt, _stream())
    else:
        idx = np.ascontiguousarray(sel.indices if isinstance(sel, RankSelection) else sel, dtype=np.uint32)
        call("pg_masked_forward", layer.handle, idx.ctypes.data, idx.size, 0, _ptr(x), lay, T, _ptr(y), ydt,
             _stream())
    return y


class SelectionBatch:
    """P selections of one layer as device byte masks [P, stride]
    (pg_selection_masks); each selection is validated like check_selection
    (rank_experts.hpp:30-37)."""

    def __init__(self, layer: FactorizedLayer, selections):
        sels = [np.ascontiguousarray(s.indices if isinstance(s, RankSelection) else s, dtype=np.uint32)
                for s in selections]
        if not sels:
            raise ValueError("selection batch: no selections")
        stride = C.c_size_t()
        call("pg_selection_mask_stride", layer.handle, C.byref(stride))
        self.layer, self.P, self.stride = layer, len(sels), stride.value
        self.masks = torch.zeros(self.P * self.stride, dtype=torch.uint8, device="cuda")
        flat = np.ascontiguousarray(np.concatenate(sels))
        ks = (C.c_size_t * self.P)(*[s.size for s in sels])
        call("pg_selection_masks", layer.handle, flat.ctypes.data_as(C.POINTER(C.c_uint32)), ks, self.P,
             _ptr(self.masks), _stream())


def masked_forward_union(layer: FactorizedLayer, batch: SelectionBatch, token_patterns, x: torch.Tensor,
                         out_dtype=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """masked_forward (rank_experts.hpp:52-72) for every token of a heterogeneous
    token-major batch x [T, n]: token t uses selection token_patterns[t] of
    `batch`.  The weights are read once for the whole batch (config 4)."""
    if batch.layer is not layer:
        raise ValueError("masked_forward_union: selection batch built for another layer")
    x = _dev(x, torch.bfloat16)
    if x.dim() != 2 or x.shape[1] != layer.n:
        raise ValueError("masked_forward_union: bad X shape")
    T = x.shape[0]
    if isinstance(token_patterns, torch.Tensor) and token_patterns.is_cuda:
        tp = token_patterns.to(torch.int32).contiguous()  # device ids are trusted
    else:
        tpn = np.ascontiguousarray(token_patterns, dtype=np.int64)
        if tpn.size and (tpn.min() < 0 or tpn.max() >= batch.P):
            raise IndexError("masked_forward_union: unknown pattern")
        tp = torch.from_numpy(tpn.astype(np.int32)).cuda()
    if tp.numel() != T:
        raise ValueError("masked_forward_union: one pattern id per token")
    ydt = _out_dtype(layer.dtype, out_dtype)
    y = out if out is not None else torch.empty((T, layer.m), dtype=_TORCH[ydt], device=x.device)
    call("pg_masked_forward_union", layer.handle, _ptr(batch.masks), batch.P, _ptr(tp), T, _ptr(x), _ptr(y), ydt,
         _stream())
    return y


def module_forward_union(layers, batches, token_patterns, x: torch.Tensor, out_dtype=None, outs=None) -> list:
    """masked_forward_union for several linears sharing x (q/k/v or up/gate):
    one grouped launch per stage over all of them."""
    if len(layers) != len(batches) or not layers:
        raise ValueError("module_forward_union: one selection batch per layer")
    for L, b in zip(layers, batches):
        if b.layer is not L:
            raise ValueError("module_forward_union: selection batch built for another layer")
    x = _dev(x, torch.bfloat16)
    T = x.shape[0]
    if isinstance(token_patterns, torch.Tensor) and token_patterns.is_cuda:
        tp = token_patterns.to(torch.int32).contiguous()
    else:
        tpn = np.ascontiguousarray(token_patterns, dtype=np.int64)
        if tpn.size and (tpn.min() < 0 or tpn.max() >= min(b.P for b in batches)):
            raise IndexError("module_forward_union: unknown pattern")
        tp = torch.from_numpy(tpn.astype(np.int32)).cuda()
    if tp.numel() != T:
        raise ValueError("module_forward_union: one pattern id per token")
    ydt = _out_dtype(layers[0].dtype, out_dtype)
    ys = outs if outs is not None else [torch.empty((T, L.m), dtype=_TORCH[ydt], device=x.device) for L in layers]
    n = len(layers)
    hs = (C.c_void_p * n)(*[L.handle.value if hasattr(L.handle, "value") else L.handle for L in layers])
    ms = (C.c_void_p * n)(*[_ptr(b.masks) for b in batches])
    ps = (C.c_size_t * n)(*[b.P for b in batches])
    yp = (C.c_void_p * n)(*[_ptr(y) for y in ys])
    call("pg_module_forward_union", hs, ms, ps, n, _ptr(tp), T, _ptr(x), yp, ydt, _stream())
    return ys


class UnionProgram:
    """A whole heterogeneous decode step as ONE persistent launch
    (pg_union_prog_*, union_prog.cu): modules are recorded with
    add_module (the arguments of module_forward_union, minus the token
    patterns) and run() executes every stage of every module in one kernel,
    each stage's k-blocks waiting on device for the output tiles they read.
    Buffers are bound at add time; a module whose x is an earlier module's
    output consumes it tile by tile.  Outputs must be distinct buffers that
    no earlier module reads (e.g. per-layer activations).  The executed form
    of build_plan (exec_engine.hpp:19-68) for a stack of layers."""

    def __init__(self, T: int):
        self.T = int(T)
        h = C.c_void_p()
        call("pg_union_prog_create", C.byref(h), self.T)
        self.handle = h
        self._keep = []  # tensors whose addresses the program holds
        self._P = None

    def add_module(self, layers, batches, x: torch.Tensor, outs, tok_offset: int = 0,
                   weights_reused: bool = False) -> None:
        """tok_offset: x's T tokens are entries [tok_offset, tok_offset + T) of
        run()'s token patterns (independent token groups as separate dependency
        chains of one program, e.g. two halves of a batch interleaved so one
        half's split-K tail overlaps the other's streaming); weights_reused:
        another chain reads the same weights soon (L2 evict-normal)."""
        if len(layers) != len(batches) or not layers or len(outs) != len(layers):
            raise ValueError("union_program: one selection batch and one output per layer")
        for L, b in zip(layers, batches):
            if b.layer is not L:
                raise ValueError("union_program: selection batch built for another layer")
        if x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous() or tuple(x.shape) != (self.T, layers[0].n):
            raise ValueError("union_program: x must be a contiguous bf16 device tensor [T, n]")
        ydt = _out_dtype(layers[0].dtype, outs[0].dtype)
        for L, y in zip(layers, outs):
            if tuple(y.shape) != (self.T, L.m) or not y.is_contiguous() or _out_dtype(L.dtype, y.dtype) != ydt:
                raise ValueError("union_program: outputs must be contiguous [T, m] of one dtype")
        n = len(layers)
        hs = (C.c_void_p * n)(*[L.handle.value if hasattr(L.handle, "value") else L.handle for L in layers])
        ms = (C.c_void_p * n)(*[_ptr(b.masks) for b in batches])
        ps = (C.c_size_t * n)(*[b.P for b in batches])
        yp = (C.c_void_p * n)(*[_ptr(y) for y in outs])
        if tok_offset < 0 or tok_offset + self.T > 256:
            raise ValueError("union_program: token offset + T exceeds 256")
        call("pg_union_prog_add_module", self.handle, hs, ms, ps, n, _ptr(x), yp, ydt, int(tok_offset),
             int(bool(weights_reused)))
        self.ttab = max(getattr(self, "ttab", 0), int(tok_offset) + self.T)
        self._keep += [x, *outs, *batches, *layers]
        P = min(b.P for b in batches)
        self._P = P if self._P is None else min(self._P, P)

    def run(self, token_patterns) -> None:
        if isinstance(token_patterns, torch.Tensor) and token_patterns.is_cuda:
            tp = token_patterns
            if tp.dtype != torch.int32 or not tp.is_contiguous():
                raise ValueError("union_program: device token patterns must be contiguous int32")
        else:
            tpn = np.ascontiguousarray(token_patterns, dtype=np.int64)
            if tpn.size and (tpn.min() < 0 or tpn.max() >= (self._P or 0)):
                raise IndexError("union_program: unknown pattern")
            tp = torch.from_numpy(tpn.astype(np.int32)).cuda()
            self._tp = tp
        if tp.numel() != getattr(self, "ttab", self.T):
            raise ValueError("union_program: one pattern id per token of the program")
        call("pg_union_prog_run", self.handle, _ptr(tp), _stream())

    def info(self) -> tuple[int, int]:
        ph, gr = C.c_size_t(), C.c_size_t()
        call("pg_union_prog_info", self.handle, C.byref(ph), C.byref(gr))
        return ph.value, gr.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                call("pg_union_prog_destroy", h)
            except Exception:
                pass


@dataclass
class AccessTrace:
    """exec_engine.hpp:90-92."""
    a_cols: list = field(default_factory=list)
    b_cols: list = field(default_factory=list)


@dataclass
class ColRange:
    start: int = 0
    len: int = 0


def maximal_runs(cols) -> list[ColRange]:
    """exec_engine.hpp:77-88."""
    runs: list[ColRange] = []
    for c in sorted(set(int(v) for v in cols)):
        if runs and runs[-1].start + runs[-1].len == c:
            runs[-1].len += 1
        else:
            runs.append(ColRange(c, 1))
    return runs


class _Residual:
    def __init__(self, ids, use_shared, arena_offset):
        self.ids, self.use_shared, self.arena_offset = ids, use_shared, arena_offset


class AggregatedLayer:
    """exec_engine.hpp:97-110, arena gathered on device (expert gather, K3)."""

    def __init__(self, layer: FactorizedLayer, patterns, psi: float = 0.9):
        self.layer = layer
        self.m, self.n, self.r_store, self.psi = layer.m, layer.n, layer.r_store, psi
        pats = [np.ascontiguousarray(p.indices if isinstance(p, RankSelection) else p, dtype=np.uint32)
                for p in patterns]
        ks = np.array([p.size for p in pats], dtype=np.uintp)
        flat = np.ascontiguousarray(np.concatenate(pats) if pats else np.zeros(0, dtype=np.uint32), dtype=np.uint32)
        h = C.c_void_p()
        call("pg_aggregate_layout", C.byref(h), layer.handle, flat.ctypes.data_as(C.POINTER(C.c_uint32)),
             ks.ctypes.data_as(C.POINTER(C.c_size_t)), len(pats), float(psi), _stream())
        self.handle = h
        cnt = C.c_size_t()
        call("pg_agg_shared", h, C.byref(cnt), None)
        ids = np.zeros(max(cnt.value, 1), dtype=np.uint32)
        call("pg_agg_shared", h, C.byref(cnt), ids.ctypes.data_as(C.POINTER(C.c_uint32)))
        self.shared_ids = ids[: cnt.value]
        self.residuals = []
        s = self.shared_ids.size
        for p in range(len(pats)):
            rc, off = C.c_size_t(), C.c_size_t()
            call("pg_agg_residual", h, p, C.byref(rc), None, None, None)
            rid = np.zeros(max(rc.value, 1), dtype=np.uint32)
            us = np.zeros(max(s, 1), dtype=np.uint8)
            call("pg_agg_residual", h, p, C.byref(rc), rid.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(off),
                 us.ctypes.data_as(C.POINTER(C.c_uint8)))
            self.residuals.append(_Residual(rid[: rc.value], us[:s], int(off.value)))

    def nbytes(self) -> int:
        b = C.c_size_t()
        call("pg_agg_bytes", self.handle, C.byref(b))
        return int(b.value)

    def trace(self, pattern_id: int) -> AccessTrace:
        cnt = C.c_size_t()
        call("pg_agg_trace", self.handle, pattern_id, C.byref(cnt), None)
        cols = np.zeros(max(cnt.value, 1), dtype=np.uintp)
        call("pg_agg_trace", self.handle, pattern_id, C.byref(cnt), cols.ctypes.data_as(C.POINTER(C.c_size_t)))
        c = [int(v) for v in cols[: cnt.value]]
        return AccessTrace(list(c), list(c))

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.lib().pg_agg_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass


def aggregate_layout(layer: FactorizedLayer, patterns, psi: float = 0.9) -> AggregatedLayer:
    """exec_engine.hpp:112-164."""
    return AggregatedLayer(layer, patterns, psi)


def aggregated_forward(agg: AggregatedLayer, pattern_id, x: torch.Tensor, trace: AccessTrace | None = None,
                       layout: str = "feature", out_dtype=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """exec_engine.hpp:193-236.  pattern_id: int, or a device int32 tensor
    (e.g. retrieve_device's entry) consumed without a host round trip."""
    lay = _layout(layout)
    x = _dev(x, agg.layer.torch_dtype)
    if lay == PG_FEATURE_MAJOR:
        if x.dim() == 1:
            x = x.view(-1, 1)
        n, T = x.shape
    else:
        T, n = x.shape
    if n != agg.n:
        raise ValueError("aggregated_forward: bad X shape")
    ydt = _out_dtype(agg.layer.dtype, out_dtype)
    shape = (agg.m, T) if lay == PG_FEATURE_MAJOR else (T, agg.m)
    y = out if out is not None else torch.empty(shape, dtype=_TORCH[ydt], device=x.device)
    if isinstance(pattern_id, torch.Tensor):
        call("pg_aggregated_forward", agg.handle, 0, _ptr(pattern_id), _ptr(x), lay, T, _ptr(y), ydt, _stream())
    else:
        if trace is not None:
            tr = agg.trace(int(pattern_id))
            trace.a_cols += tr.a_cols
            trace.b_cols += tr.b_cols
        call("pg_aggregated_forward", agg.handle, int(pattern_id), None, _ptr(x), lay, T, _ptr(y), ydt, _stream())
    return y


def aggregated_forward_batched(agg: AggregatedLayer, pattern_ids, offsets, x: torch.Tensor, out_dtype=None,
                               out: torch.Tensor | None = None) -> torch.Tensor:
    """Heterogeneous token-major batch: prompt p (tokens offsets[p]:offsets[p+1])
    is served with pattern pattern_ids[p]."""
    x = _dev(x, agg.layer.torch_dtype)
    pats = np.ascontiguousarray(pattern_ids, dtype=np.int32)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    ydt = _out_dtype(agg.layer.dtype, out_dtype)
    y = out if out is not None else torch.empty((x.shape[0], agg.m), dtype=_TORCH[ydt], device=x.device)
    call("pg_aggregated_forward_batched", agg.handle, pats.ctypes.data_as(C.POINTER(C.c_int32)),
         offs.ctypes.data_as(C.POINTER(C.c_int64)), pats.size, _ptr(x), _ptr(y), ydt, _stream())
    return y


def prefill_batched(aggs: list, offsets, x: torch.Tensor, out_dtype=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Heterogeneous bf16 prefill (config 3): prompt p (tokens offsets[p]:offsets[p+1]
    of token-major x) is served by its own packed layout aggs[p]; all prompts run as
    grouped tcgen05 GEMM launches."""
    x = _dev(x, torch.bfloat16)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    ydt = _out_dtype(aggs[0].layer.dtype, out_dtype)
    y = out if out is not None else torch.empty((x.shape[0], aggs[0].m), dtype=_TORCH[ydt], device=x.device)
    hs = (C.c_void_p * len(aggs))(*[g.handle.value for g in aggs])
    call("pg_prefill_batched", hs, offs.ctypes.data_as(C.POINTER(C.c_int64)), len(aggs), _ptr(x), _ptr(y), ydt,
         _stream())
    return y


class PackedExperts:
    """Every prompt's selected experts packed on device (K3 for a routed batch,
    exec_engine.hpp:112-164 with one pattern per prompt): B^T rows [P, kp, ldb]
    and A columns [P, m, kp] in caller-owned (torch) buffers."""

    def __init__(self, layer: FactorizedLayer, k: int, n_prompts: int, bt: torch.Tensor | None, a: torch.Tensor,
                 sel: torch.Tensor | None = None):
        self.layer, self.k, self.P, self.bt, self.a = layer, k, n_prompts, bt, a
        self.sel = sel  # gathered packs (bt is None): the selection the prefill gathers B^T rows by

    @property
    def gathered(self) -> bool:
        return self.bt is None


def pack_selected(layer: FactorizedLayer, sel: torch.Tensor, into: PackedExperts | None = None,
                  gather: bool = False) -> PackedExperts:
    """Pack each prompt's selection sel [P, K] (device int32, ascending; the
    router's output) on the device -- no host round trip, no synchronisation.
    `into`: an earlier pack of the same layer and shape whose buffers are
    reused (serving loops: no allocation per batch).  gather=True packs the A
    columns only: prefill_packed then gathers the selected B^T rows straight
    from the layer inside the stage-1 GEMM (TMA gather4; `sel` must stay
    unchanged until that prefill has run; prompts of 0 or >= 256 tokens)."""
    if not (isinstance(sel, torch.Tensor) and sel.is_cuda):
        raise ValueError("pack_selected: device selection tensor [P, K] expected")
    if sel.dim() == 1:
        sel = sel.unsqueeze(0)
    sel = sel.to(torch.int32).contiguous()
    P, k = sel.shape
    bb, ab = C.c_size_t(), C.c_size_t()
    call("pg_pack_bytes", layer.handle, k, P, C.byref(bb), C.byref(ab))
    if into is not None:
        if (into.layer is not layer or into.gathered != gather or into.a.numel() != ab.value
                or (not gather and into.bt.numel() != bb.value)):
            raise ValueError("pack_selected: `into` packs another layer / shape / mode")
        bt, a = into.bt, into.a
    else:
        bt = None if gather else torch.empty(bb.value, dtype=torch.uint8, device=sel.device)
        a = torch.empty(ab.value, dtype=torch.uint8, device=sel.device)
    call("pg_pack_selected", layer.handle, _ptr(sel), k, P, None if bt is None else _ptr(bt), _ptr(a), _stream())
    return PackedExperts(layer, k, P, bt, a, sel if gather else None)


def prefill_packed(packed: PackedExperts, offsets, x: torch.Tensor, out_dtype=None,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """Routed heterogeneous prefill (config 3): prompt p (tokens
    offsets[p]:offsets[p+1] of token-major x [T, n]) through its packed experts,
    as grouped tcgen05 GEMMs."""
    L = packed.layer
    x = _dev(x, torch.bfloat16)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    if offs.size != packed.P + 1 or x.dim() != 2 or x.shape[1] != L.n or offs[-1] > x.shape[0]:
        raise ValueError("prefill_packed: bad X shape / offsets")
    ydt = _out_dtype(L.dtype, out_dtype)
    y = out if out is not None else torch.empty((x.shape[0], L.m), dtype=_TORCH[ydt], device=x.device)
    if packed.gathered:
        call("pg_prefill_gathered", L.handle, _ptr(packed.sel), _ptr(packed.a), packed.k,
             offs.ctypes.data_as(C.POINTER(C.c_int64)), packed.P, _ptr(x), _ptr(y), ydt, _stream())
    else:
        call("pg_prefill_packed", L.handle, _ptr(packed.bt), _ptr(packed.a), packed.k,
             offs.ctypes.data_as(C.POINTER(C.c_int64)), packed.P, _ptr(x), _ptr(y), ydt, _stream())
    return y


def scattered_forward(layer: FactorizedLayer, sel, x: torch.Tensor, trace: AccessTrace | None = None,
                      layout: str = "feature", out_dtype=None) -> torch.Tensor:
    """exec_engine.hpp:239-252: K strided column gathers in S order."""
    if trace is not None:
        ids = [int(v) for v in (sel.indices if isinstance(sel, RankSelection) else sel)]
        trace.a_cols += ids
        trace.b_cols += ids
    return masked_forward(layer, sel, x, layout=layout, out_dtype=out_dtype)


# ---------------------------------------------------------------- engine + providers
class ExecVariant(enum.Enum):
    scattered_unfused = "scattered-unfused"
    aggregated_only = "aggregated-only"
    fused_only = "fused-only"
    aggregated_fused = "aggregated+fused"


def variant_aggregated(v: ExecVariant) -> bool:
    return v in (ExecVariant.aggregated_only, ExecVariant.aggregated_fused)


def variant_fused(v: ExecVariant) -> bool:
    return v in (ExecVariant.fused_only, ExecVariant.aggregated_fused)


PROJ_NAMES = ("q", "k", "v", "o", "up", "gate", "down")


def tensor_id(block: int, proj: str) -> str:
    """toy_lm.hpp:62-64."""
    return f"b{block}.{proj}"


class LaunchKind(enum.Enum):
    fused_B = "fused_B"
    batched_A = "batched_A"
    single = "single"


@dataclass
class LaunchDesc:
    kind: LaunchKind
    tensor_ids: list
    side: str


@dataclass
class ExecPlan:
    launches: list = field(default_factory=list)
    launches_per_block: int = 0
    unfused_per_block: int = 14
    gqa: bool = False


def build_plan(n_blocks: int, gqa: bool) -> ExecPlan:
    """exec_engine.hpp:46-68: 8 (MHA) / 9 (GQA) descriptors per block vs 14."""
    plan = ExecPlan(gqa=gqa)
    for b in range(n_blocks):
        i = lambda p: tensor_id(b, p)  # noqa: E731
        plan.launches.append(LaunchDesc(LaunchKind.fused_B, [i("q"), i("k"), i("v")], "B"))
        if gqa:
            plan.launches.append(LaunchDesc(LaunchKind.batched_A, [i("q")], "A"))
            plan.launches.append(LaunchDesc(LaunchKind.batched_A, [i("k"), i("v")], "A"))
        else:
            plan.launches.append(LaunchDesc(LaunchKind.batched_A, [i("q"), i("k"), i("v")], "A"))
        plan.launches.append(LaunchDesc(LaunchKind.single, [i("o")], "B"))
        plan.launches.append(LaunchDesc(LaunchKind.single, [i("o")], "A"))
        plan.launches.append(LaunchDesc(LaunchKind.fused_B, [i("up"), i("gate")], "B"))
        plan.launches.append(LaunchDesc(LaunchKind.batched_A, [i("up"), i("gate")], "A"))
        plan.launches.append(LaunchDesc(LaunchKind.single, [i("down")], "B"))
        plan.launches.append(LaunchDesc(LaunchKind.single, [i("down")], "A"))
    plan.launches_per_block = len(plan.launches) // max(n_blocks, 1)
    return plan


class ExecEngine:
    """exec_engine.hpp:275-319: per tensor {layer, aggregated layout}."""

    def __init__(self):
        self.tensors: dict[str, tuple[FactorizedLayer, AggregatedLayer]] = {}
        self.patterns: list[dict] = []
        self.psi = 0.9

    @staticmethod
    def build(layers: dict, patterns: list, psi: float = 0.9) -> "ExecEngine":
        eng = ExecEngine()
        eng.psi = psi
        eng.patterns = list(patterns)
        for tid, layer in layers.items():
            sels = [p[tid] for p in eng.patterns]
            eng.tensors[tid] = (layer, aggregate_layout(layer, sels, psi))
        return eng

    def forward(self, tid: str, pattern_id: int, x, variant: ExecVariant = ExecVariant.aggregated_fused,
                trace: AccessTrace | None = None, **kw):
        layer, agg = self.tensors[tid]
        if variant_aggregated(variant):
            return aggregated_forward(agg, pattern_id, x, trace, **kw)
        if pattern_id >= len(self.patterns):
            raise IndexError("unknown pattern")
        return scattered_forward(layer, self.patterns[pattern_id][tid], x, trace, **kw)

    def storage_overhead(self) -> float:
        """duplicated residual columns beyond single-copy storage (:310-318)."""
        dup = base = 0.0
        for layer, agg in self.tensors.values():
            base += float(layer.r_store) * float(layer.m + layer.n)
            for r in agg.residuals:
                dup += float(r.ids.size) * float(layer.m + layer.n)
        return dup / base


@dataclass
class FactorizedModel:
    """model.hpp:18-47 (projection layers + routers; the LM core is out of scope)."""
    layers: dict = field(default_factory=dict)
    routers: dict = field(default_factory=dict)
    n_blocks: int = 0

    def layer_ids(self):
        return [tensor_id(b, p) for b in range(self.n_blocks) for p in PROJ_NAMES]

    def compute_params(self) -> float:
        return float(sum(l.K * (l.m + l.n) for l in self.layers.values()))

    def storage_params(self) -> float:
        return float(sum(l.r_store * (l.m + l.n) for l in self.layers.values()))


class ProjectionProvider:
    """toy_lm.hpp:68-75: the drop-in point (feature-major n x T activations)."""

    def apply(self, b: int, p: str, x):  # pragma: no cover - interface
        raise NotImplementedError

    def qkv(self, b, hn):
        return self.apply(b, "q", hn), self.apply(b, "k", hn), self.apply(b, "v", hn)

    def o_proj(self, b, x):
        return self.apply(b, "o", x)

    def upgate(self, b, hn):
        return self.apply(b, "up", hn), self.apply(b, "gate", hn)

    def down_proj(self, b, x):
        return self.apply(b, "down", x)


class FactorizedProvider(ProjectionProvider):
    """model.hpp:50-86: fixed SelectionMap, or the static prefix {0..K-1}
    (native SVD) when the map is absent or lacks the id."""

    def __init__(self, model: FactorizedModel, sel: dict | None = None, layout: str = "feature"):
        self.m, self.sel, self.layout = model, sel, layout
        self._prefix: dict[str, RankSelection] = {}

    def selection_for(self, tid: str) -> RankSelection:
        if self.sel is not None and tid in self.sel:
            return self.sel[tid]
        if tid not in self._prefix:
            self._prefix[tid] = RankSelection.prefix(self.m.layers[tid].K)
        return self._prefix[tid]

    def apply(self, b, p, x):
        tid = tensor_id(b, p)
        return masked_forward(self.m.layers[tid], self.selection_for(tid), x, layout=self.layout)


class RoutingProvider(ProjectionProvider):
    """model.hpp:90-126: route once per tensor id from the first call's input
    (prefill), reuse the frozen selection for every later call (decode)."""

    def __init__(self, model: FactorizedModel, layout: str = "feature"):
        if not model.routers:
            raise RuntimeError("model has no trained routers")
        self.m, self.layout = model, layout
        self._sel: dict[str, torch.Tensor] = {}

    def apply(self, b, p, x):
        tid = tensor_id(b, p)
        layer = self.m.layers[tid]
        if tid not in self._sel:
            self._sel[tid] = route_select(self.m.routers[tid], x, layer.K, layout=self.layout)[0]
        return masked_forward(layer, self._sel[tid], x, layout=self.layout)

    def selections(self) -> dict:
        return {k: RankSelection(v.cpu().numpy().astype(np.uint32)) for k, v in self._sel.items()}

    def reset(self):
        self._sel.clear()


class ExecProvider(ProjectionProvider):
    """exec_engine.hpp:322-348: plan-driven serving over an ExecEngine."""

    def __init__(self, eng: ExecEngine, pattern_id: int, variant: ExecVariant, layout: str = "feature"):
        self.eng, self.pattern, self.variant, self.layout = eng, pattern_id, variant, layout
        self.launches = 0

    def apply(self, b, p, x):
        self.launches += 1
        return self.eng.forward(tensor_id(b, p), self.pattern, x, self.variant, layout=self.layout)


# ---------------------------------------------------------------- serving composition
@dataclass
class PromptSelection:
    """The frozen per-tensor expert subsets a prompt is served with, and where
    they came from: "hit" (a cached entry's SelectionMap) or "routed" (online
    routing on the prompt's prefill inputs)."""
    pattern: dict
    source: str
    entry: int = -1           # cache entry serving / now holding the pattern (-1: not cached)
    similarity: float = -2.0  # retrieve's best cosine (-2 for an empty cache)
    inserted: bool = False    # miss path: cache_insert accepted the routed pattern


class PatternServer:
    """Retrieve-or-route serving (the north star's "S chosen by a linear router or
    by a pattern-cache lookup, then reused across decode steps"):

      retrieve(cache, embedding)                       pattern_cache.hpp:104-117
        hit  (sim >= min_similarity): the entry's SelectionMap
        miss: route every tensor id from the input it sees at prefill,
              select_topk(score(mean_pool(x)), K)      model.hpp:96-106 (route_prompt, pattern_cache.hpp:67-73)
              then cache_insert(cache, {embedding, S}) pattern_cache.hpp:120-124 (refused at capacity)

    The packed device layouts (aggregate_layout, exec_engine.hpp:112-164) are
    cached per cache entry, so repeated hits on an entry never re-pack; decode
    steps reuse the prompt's frozen selection (provider())."""

    def __init__(self, model: FactorizedModel, cache: PatternCache, psi: float = 0.9):
        self.model, self.cache, self.psi = model, cache, psi
        self._packs: dict[int, dict] = {}
        self.packs_built = 0

    def select_for_prompt(self, embedding, route_inputs, layout: str = "feature") -> PromptSelection:
        """embedding: PromptEmbedding (or its vector); route_inputs: {tensor id:
        x} or a callable tid -> x giving the input each routed linear sees at
        prefill (n x T feature-major, or T x n with layout="token")."""
        emb = embedding if isinstance(embedding, PromptEmbedding) else PromptEmbedding(np.asarray(embedding))
        sim = -2.0
        if self.cache.entries:
            res = retrieve(self.cache, emb, exact_similarity=True)  # the reference's RetrieveResult, bit for bit
            sim = res.similarity
            if res.hit:
                return PromptSelection(res.pattern, "hit", res.entry, res.similarity, False)
        get = route_inputs if callable(route_inputs) else route_inputs.__getitem__
        pattern = {}
        for tid, layer in self.model.layers.items():
            x = get(tid)
            sel = route_select(self.model.routers[tid], x, layer.K, layout=layout)[0]
            pattern[tid] = RankSelection(sel.cpu().numpy().astype(np.uint32))
        inserted = cache_insert(self.cache, CacheEntry(emb, pattern))
        return PromptSelection(pattern, "routed", len(self.cache.entries) - 1 if inserted else -1, sim, inserted)

    def layouts(self, sel: PromptSelection) -> dict:
        """Per tensor id, the prompt's packed layout (one pattern).  Cached per
        cache entry: a second hit on the same entry reuses the packs."""
        if sel.entry >= 0 and sel.entry in self._packs:
            return self._packs[sel.entry]
        packs = {tid: aggregate_layout(self.model.layers[tid], [s], self.psi) for tid, s in sel.pattern.items()}
        self.packs_built += 1
        if sel.entry >= 0:
            self._packs[sel.entry] = packs
        return packs

    def provider(self, sel: PromptSelection, layout: str = "feature") -> "FactorizedProvider":
        """Serve prefill and every decode step with the frozen selection."""
        return FactorizedProvider(self.model, sel.pattern, layout=layout)


def _pattern_args(pattern_ids, count):
    if isinstance(pattern_ids, torch.Tensor):
        return None, _ptr(pattern_ids)
    pats = [int(pattern_ids)] * count if np.isscalar(pattern_ids) else [int(p) for p in pattern_ids]
    arr = (C.c_size_t * count)(*pats)
    return arr, None


def module_forward(aggs: list, pattern_ids, x: torch.Tensor, out_dtype=None, outs=None) -> list:
    """K6 fused module (exec_engine.hpp:46-68 fused_B + batched_A), decode T=1:
    1..3 linears sharing x run as one kernel.  pattern_ids: int, list, or a
    device int32 tensor (retrieve_device's entry)."""
    x = _dev(x, aggs[0].layer.torch_dtype).reshape(-1)
    ydt = _out_dtype(aggs[0].layer.dtype, out_dtype)
    ys = outs if outs is not None else [torch.empty(g.m, dtype=_TORCH[ydt], device=x.device) for g in aggs]
    hs = (C.c_void_p * len(aggs))(*[g.handle.value for g in aggs])
    yp = (C.c_void_p * len(aggs))(*[_ptr(y) for y in ys])
    parr, pdev = _pattern_args(pattern_ids, len(aggs))
    call("pg_module_forward", hs, len(aggs), parr, pdev, _ptr(x), yp, ydt, _stream())
    return ys


def mlp_forward(up: "AggregatedLayer", gate: "AggregatedLayer", down: "AggregatedLayer", pattern_ids,
                x: torch.Tensor, out_dtype=None, out: torch.Tensor | None = None,
                act: torch.Tensor | None = None) -> torch.Tensor:
    """One decode token (T=1) through a rank-expert MLP block in ONE kernel:
    up/gate share x, act = silu(gate)*up (toy_lm.hpp:250-257), y = down(act).
    x and out may be pinned host tensors: the kernel then reads the token and
    writes the result over the host link itself (zero-copy step I/O)."""
    def io_ptr(t):
        if t.is_pinned() and t.is_contiguous():
            return t.data_ptr()
        return _ptr(t)
    if not (isinstance(x, torch.Tensor) and x.is_pinned() and x.dtype == up.layer.torch_dtype):
        x = _dev(x, up.layer.torch_dtype)
    x = x.reshape(-1)
    ydt = _out_dtype(up.layer.dtype, out_dtype)
    y = out if out is not None else torch.empty(down.m, dtype=_TORCH[ydt], device="cuda")
    parr, pdev = _pattern_args(pattern_ids, 3)
    call("pg_mlp_forward", up.handle, gate.handle, down.handle, parr, pdev, io_ptr(x),
         _ptr(act) if act is not None else None, io_ptr(y), ydt, _stream())
    return y


def mlp_forward_chain(blocks, x: torch.Tensor, pattern_ids=None, outs=None, acts=None) -> list:
    """A decode token through a chain of MLP blocks, block s+1 reading block
    s's output (x_{s+1} = y_s, every block as mlp_forward), up to 8 blocks per
    kernel launch (pg_mlp_forward_chain).  blocks: [(up, gate, down), ...]
    aggregated layers; pattern_ids: per block (up, gate, down) pattern ids
    (default 0).  Returns the blocks' outputs (weight dtype)."""
    S = len(blocks)
    if S < 1:
        raise ValueError("mlp_forward_chain: no blocks")
    dt = blocks[0][0].layer.torch_dtype
    x = _dev(x, dt).reshape(-1)
    ys = outs if outs is not None else [torch.empty(b[2].m, dtype=dt, device="cuda") for b in blocks]
    if len(ys) != S or any(y.dtype != dt or not y.is_contiguous() or y.numel() != b[2].m for y, b in zip(ys, blocks)):
        raise ValueError("mlp_forward_chain: one contiguous output of the weight dtype per block")
    pids = pattern_ids if pattern_ids is not None else [(0, 0, 0)] * S
    pat = (C.c_size_t * (3 * S))(*[int(v) for p in pids for v in p])
    hs = [(C.c_void_p * S)(*[b[i].handle.value for b in blocks]) for i in range(3)]
    ap = (C.c_void_p * S)(*[_ptr(a) for a in acts]) if acts is not None else None
    yp = (C.c_void_p * S)(*[_ptr(y) for y in ys])
    call("pg_mlp_forward_chain", hs[0], hs[1], hs[2], pat, S, _ptr(x), ap, yp, _dtype_code(dt), _stream())
    return ys


def copy_io(dst: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """Step I/O as a kernel on the current stream: dst <- src where either side
    may be pinned host memory (UVA-mapped).  Chains with the step's kernels
    (programmatic dependent launch) instead of a copy-engine node."""
    for t in (dst, src):
        if not (t.is_cuda or t.is_pinned()):
            raise ValueError("copy_io: buffers must be device or pinned host memory")
        if not t.is_contiguous():
            raise ValueError("copy_io: buffers must be contiguous")
    nb = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() != nb:
        raise ValueError("copy_io: size mismatch")
    call("pg_copy_io", C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), nb, _stream())
    return dst


def silu_mul(gate: torch.Tensor, up: torch.Tensor, out_dtype=torch.bfloat16, out=None) -> torch.Tensor:
    """MLP glue (toy_lm.hpp:250-257): silu(gate) * up on device."""
    if gate.shape != up.shape or gate.dtype != up.dtype:
        raise ValueError("silu_mul: shape mismatch")
    odt = _dtype_code(out_dtype)
    y = out if out is not None else torch.empty(gate.shape, dtype=_TORCH[odt], device=gate.device)
    call("pg_silu_mul", _ptr(gate), _ptr(up), _dtype_code(gate.dtype), gate.numel(), _ptr(y), odt, _stream())
    return y


# ---------------------------------------------------------------- generators
def rng_gaussian(seed: int, shape) -> np.ndarray:
    """Rng(seed).gaussian() stream (rng.hpp:10-41), identical bits to the reference."""
    count = int(np.prod(shape))
    out = np.empty(count, dtype=np.float64)
    _lib.lib().pg_rng_fill_gaussian(seed, out.ctypes.data_as(C.POINTER(C.c_double)), count)
    return out.reshape(shape)


def make_patterns(seed: int, n_patterns: int, layers: list[tuple[int, int]]) -> list[list[RankSelection]]:
    """The reference's prefix-biased generator (test_acceptance.cpp:412-425).
    layers: [(r_store, K), ...] -> pats[p][l]."""
    rs = np.array([l[0] for l in layers], dtype=np.uintp)
    ks = np.array([l[1] for l in layers], dtype=np.uintp)
    out = np.empty(n_patterns * int(ks.sum()), dtype=np.uint32)
    _lib.lib().pg_make_patterns(seed, n_patterns, rs.ctypes.data_as(C.POINTER(C.c_size_t)),
                                ks.ctypes.data_as(C.POINTER(C.c_size_t)), len(layers),
                                out.ctypes.data_as(C.POINTER(C.c_uint32)))
    res, w = [], 0
    for _ in range(n_patterns):
        row = []
        for k in ks:
            row.append(RankSelection(out[w:w + int(k)].copy()))
            w += int(k)
        res.append(row)
    return res
