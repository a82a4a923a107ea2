"""ctypes view of the parity checkers -- TEST INFRASTRUCTURE ONLY.

`Oracle("port")` loads oracle/liboracle.so (the C restatement, po_* symbols);
`Oracle("reference")` loads oracle/_ref/libparse_ref.so (the reference's own
headers compiled here, ref_* symbols).  Both expose the same numpy-level
methods so a test can run the same case through either and compare bits.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": (os.path.join(HERE, "liboracle.so"), "po_"),
    "reference": (os.path.join(HERE, "_ref", "libparse_ref.so"), "ref_"),
}

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_up = C.POINTER(C.c_uint32)
_sp = C.POINTER(C.c_size_t)
_bp = C.POINTER(C.c_uint8)
_sz = C.c_size_t


class RetrieveResultC(C.Structure):
    _fields_ = [("entry", C.c_size_t), ("similarity", C.c_double), ("hit", C.c_int)]


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind][0])


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _u(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a, t):
    return a.ctypes.data_as(t)


ERRORS = {1: ValueError, 2: IndexError, 3: RuntimeError}


def _raise(code: int, what: str):
    if code:
        raise ERRORS.get(code, RuntimeError)(f"{what}: error code {code}")


class Oracle:
    def __init__(self, kind: str = "port"):
        path, pre = PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `python oracle/build.py`")
        self.kind = kind
        self.lib = L = C.CDLL(path)
        self.p = pre
        g = lambda n: getattr(L, pre + n)  # noqa: E731
        self._fill = g("fill_gaussian"); self._fill.argtypes = [C.c_uint64, _dp, _sz]
        self._mean_pool = g("mean_pool"); self._mean_pool.argtypes = [_dp, _sz, _sz, _dp]
        self._score = g("score"); self._score.argtypes = [_dp, _dp, _sz, _sz, _dp, _dp]
        self._topk = g("select_topk"); self._topk.argtypes = [_dp, _sz, _sz, _up]; self._topk.restype = C.c_int
        self._cos = g("cosine"); self._cos.argtypes = [_dp, _dp, _sz]; self._cos.restype = C.c_double
        self._ret = g("retrieve")
        self._ret.argtypes = [_dp, _sz, _sz, C.c_double, _dp, C.POINTER(RetrieveResultC)]
        self._ret.restype = C.c_int
        self._emb = g("embed_normalize"); self._emb.argtypes = [_dp, _sz, _sz, _dp]; self._emb.restype = C.c_int
        self._chk = g("check_selection"); self._chk.argtypes = [_up, _sz, _sz]; self._chk.restype = C.c_int
        self._mf = g("masked_forward")
        self._mf.argtypes = [_dp, _dp, _sz, _sz, _sz, _up, _sz, _dp, _sz, _dp]
        self._mf.restype = C.c_int
        self._agg = g("aggregate_layout")
        self._agg.argtypes = [_dp, _dp, _sz, _sz, _sz, _up, _sp, _sz, C.c_double, C.c_int, C.POINTER(C.c_int)]
        self._agg.restype = C.c_void_p
        self._agg_free = g("agg_free"); self._agg_free.argtypes = [C.c_void_p]
        for nm in ("agg_shared_count",):
            f = g(nm); f.argtypes = [C.c_void_p]; f.restype = _sz; setattr(self, "_" + nm, f)
        f = g("agg_shared_ids"); f.argtypes = [C.c_void_p, _up]; self._agg_shared_ids = f
        f = g("agg_residual_count"); f.argtypes = [C.c_void_p, _sz]; f.restype = _sz; self._agg_res_count = f
        f = g("agg_residual_ids"); f.argtypes = [C.c_void_p, _sz, _up]; self._agg_res_ids = f
        f = g("agg_arena_offset"); f.argtypes = [C.c_void_p, _sz]; f.restype = _sz; self._agg_off = f
        f = g("agg_use_shared"); f.argtypes = [C.c_void_p, _sz, _bp]; self._agg_use = f
        f = g("aggregated_forward_f32"); f.argtypes = [C.c_void_p, _sz, _fp, _sz, _fp]; f.restype = C.c_int
        self._aggf32 = f
        f = g("aggregated_forward_f64"); f.argtypes = [C.c_void_p, _sz, _dp, _sz, _dp]; f.restype = C.c_int
        self._aggf64 = f
        f = g("scattered_forward_f32"); f.argtypes = [_fp, _fp, _sz, _sz, _sz, _up, _sz, _fp, _sz, _fp]
        self._scat = f
        f = g("maximal_runs"); f.argtypes = [_sp, _sz, _sp, _sp]; f.restype = _sz; self._runs = f
        f = g("store_rank"); f.argtypes = [_sz, _sz, C.c_double]; f.restype = _sz; self._store_rank = f
        f = g("single_layer_k"); f.argtypes = [_sz, _sz, C.c_double]; f.restype = _sz; self._slk = f

    # ---- rng / shapes ----
    def gaussian(self, seed: int, shape) -> np.ndarray:
        out = np.empty(int(np.prod(shape)), dtype=np.float64)
        self._fill(seed, _ptr(out, _dp), out.size)
        return out.reshape(shape)

    def store_rank(self, k, r_max, mult=2.0):
        return int(self._store_rank(k, r_max, mult))

    def single_layer_k(self, m, n, ratio):
        return int(self._slk(m, n, ratio))

    # ---- router ----
    def mean_pool(self, x):
        x = _d(x); n, T = x.shape
        h = np.empty(n); self._mean_pool(_ptr(x, _dp), n, T, _ptr(h, _dp)); return h

    def score(self, theta, bias, h):
        theta = _d(theta); bias = _d(bias); h = _d(h); r, n = theta.shape
        z = np.empty(r); self._score(_ptr(theta, _dp), _ptr(bias, _dp), r, n, _ptr(h, _dp), _ptr(z, _dp))
        return z

    def select_topk(self, logits, k):
        logits = _d(logits); out = np.empty(max(k, 1), dtype=np.uint32)
        _raise(self._topk(_ptr(logits, _dp), logits.size, k, _ptr(out, _up)), "select_topk")
        return out[:k]

    # ---- cache ----
    def cosine(self, a, b):
        a = _d(a); b = _d(b)
        if a.size != b.size:
            raise ValueError("cosine: length mismatch")
        return float(self._cos(_ptr(a, _dp), _ptr(b, _dp), a.size))

    def retrieve(self, emb, min_similarity, query):
        emb = _d(emb).reshape(-1, np.asarray(query).size) if np.asarray(emb).size else np.zeros((0, np.asarray(query).size))
        q = _d(query); res = RetrieveResultC()
        _raise(self._ret(_ptr(emb, _dp), emb.shape[0], q.size, min_similarity, _ptr(q, _dp), C.byref(res)), "retrieve")
        return int(res.entry), float(res.similarity), bool(res.hit)

    def embed_normalize(self, x):
        x = _d(x); d, T = x.shape; out = np.empty(d)
        _raise(self._emb(_ptr(x, _dp), d, T, _ptr(out, _dp)), "embed_normalize")
        return out

    # ---- rank experts ----
    def check_selection(self, sel, r_store):
        sel = _u(sel)
        _raise(self._chk(_ptr(sel, _up), sel.size, r_store), "check_selection")

    def masked_forward(self, A, B, sel, x):
        A = _d(A); B = _d(B); sel = _u(sel); x = _d(x)
        m, r = A.shape; n = B.shape[0]; T = x.shape[1]
        out = np.empty((m, T))
        _raise(self._mf(_ptr(A, _dp), _ptr(B, _dp), m, n, r, _ptr(sel, _up), sel.size, _ptr(x, _dp), T,
                        _ptr(out, _dp)), "masked_forward")
        return out

    def aggregate_layout(self, A, B, patterns, psi, elem=4):
        return _OracleAgg(self, A, B, patterns, psi, elem)

    def scattered_forward_f32(self, A32, B32, sel, x32):
        A32 = _f(A32); B32 = _f(B32); sel = _u(sel); x32 = _f(x32)
        m, r = A32.shape; n = B32.shape[0]; T = x32.shape[1]
        out = np.empty((m, T), dtype=np.float32)
        self._scat(_ptr(A32, _fp), _ptr(B32, _fp), m, n, r, _ptr(sel, _up), sel.size, _ptr(x32, _fp), T,
                   _ptr(out, _fp))
        return out

    def maximal_runs(self, cols):
        c = np.ascontiguousarray(cols, dtype=np.uint64).astype(np.uintp)
        starts = np.empty(max(c.size, 1), dtype=np.uintp); lens = np.empty_like(starts)
        nr = self._runs(c.ctypes.data_as(_sp), c.size, starts.ctypes.data_as(_sp), lens.ctypes.data_as(_sp))
        return [(int(starts[i]), int(lens[i])) for i in range(nr)]


class _OracleAgg:
    def __init__(self, o: Oracle, A, B, patterns, psi, elem):
        self.o = o
        A = _d(A); B = _d(B)
        self.m, r = A.shape; self.n = B.shape[0]; self.elem = elem
        ks = np.array([len(p) for p in patterns], dtype=np.uintp)
        flat = _u(np.concatenate([np.asarray(p, dtype=np.uint32) for p in patterns]) if len(patterns) else np.zeros(0))
        err = C.c_int(0)
        self.h = o._agg(_ptr(A, _dp), _ptr(B, _dp), self.m, self.n, r, _ptr(flat, _up), ks.ctypes.data_as(_sp),
                        len(patterns), psi, elem, C.byref(err))
        _raise(err.value, "aggregate_layout")
        self.P = len(patterns)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._agg_free(self.h)
            self.h = None

    @property
    def shared_ids(self):
        s = self.o._agg_shared_count(self.h); out = np.empty(max(s, 1), dtype=np.uint32)
        self.o._agg_shared_ids(self.h, _ptr(out, _up)); return out[:s]

    def residual_ids(self, p):
        c = self.o._agg_res_count(self.h, p); out = np.empty(max(c, 1), dtype=np.uint32)
        self.o._agg_res_ids(self.h, p, _ptr(out, _up)); return out[:c]

    def arena_offset(self, p):
        return int(self.o._agg_off(self.h, p))

    def use_shared(self, p):
        s = self.o._agg_shared_count(self.h); out = np.empty(max(s, 1), dtype=np.uint8)
        self.o._agg_use(self.h, p, _ptr(out, _bp)); return out[:s]

    def forward(self, pid, x):
        if self.elem == 4:
            x = _f(x); out = np.empty((self.m, x.shape[1]), dtype=np.float32)
            _raise(self.o._aggf32(self.h, pid, _ptr(x, _fp), x.shape[1], _ptr(out, _fp)), "aggregated_forward")
        else:
            x = _d(x); out = np.empty((self.m, x.shape[1]))
            _raise(self.o._aggf64(self.h, pid, _ptr(x, _dp), x.shape[1], _ptr(out, _dp)), "aggregated_forward")
        return out


def make_patterns(seed: int, n_patterns: int, layers: list[tuple[int, int]]) -> list[list[np.ndarray]]:
    """The reference's prefix-biased generator (test_acceptance.cpp:412-425) via the port.
    layers: [(r_store, K), ...]; returns pats[p][l] ascending uint32 arrays."""
    lib = C.CDLL(PATHS["port"][0])
    f = lib.po_make_patterns
    f.argtypes = [C.c_uint64, _sz, _sp, _sp, _sz, _up]
    rs = np.array([l[0] for l in layers], dtype=np.uintp)
    ks = np.array([l[1] for l in layers], dtype=np.uintp)
    out = np.empty(n_patterns * int(ks.sum()), dtype=np.uint32)
    f(seed, n_patterns, rs.ctypes.data_as(_sp), ks.ctypes.data_as(_sp), len(layers), _ptr(out, _up))
    res, w = [], 0
    for _ in range(n_patterns):
        row = []
        for k in ks:
            row.append(out[w:w + int(k)].copy()); w += int(k)
        res.append(row)
    return res
