"""ctypes binding of include/parse_gpu.h (libparse_gpu.so, sm_100a).

Fails loudly: if the shared library is missing or a call returns an error the
caller gets an exception -- there is no CPU fallback anywhere in the product.
Error classes mirror the reference's exceptions:
  PG_INVALID_ARGUMENT -> ValueError   (std::invalid_argument)
  PG_OUT_OF_RANGE     -> IndexError   (std::out_of_range)
  PG_RUNTIME_ERROR    -> RuntimeError (std::runtime_error)
  PG_CUDA_ERROR       -> CudaError
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libparse_gpu.so")
if os.environ.get("PG_LIB_VARIANT"):  # experiments only: lib/libparse_gpu_<variant>.so (tools/experiments)
    LIB_PATH = LIB_PATH[:-3] + "_" + os.environ["PG_LIB_VARIANT"] + ".so"

PG_F64, PG_F32, PG_BF16 = 0, 1, 2
PG_FEATURE_MAJOR, PG_TOKEN_MAJOR = 0, 1


class CudaError(RuntimeError):
    pass


_ERR = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: CudaError}


class RetrieveResultC(C.Structure):
    _fields_ = [("entry", C.c_size_t), ("similarity", C.c_double), ("hit", C.c_int),
                ("exact_similarity", C.c_int)]


_vp = C.c_void_p
_sz = C.c_size_t
_i = C.c_int
_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_uint32)
_sp = C.POINTER(C.c_size_t)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)

# name -> argtypes (all return int status unless listed in _RESTYPE)
_SIGS = {
    "pg_mean_pool": [_vp, _i, _i, _sz, _i64p, _sz, _vp, _vp],
    "pg_router_create": [C.POINTER(_vp), _sz, _sz, _dp, _dp],
    "pg_router_create_device": [C.POINTER(_vp), _sz, _sz, _vp, _vp, _i],
    "pg_router_destroy": [_vp],
    "pg_score": [_vp, _vp, _sz, _vp, _i, _vp],
    "pg_select_topk": [_vp, _sz, _sz, _sz, _vp, _vp],
    "pg_route_select": [_vp, _vp, _i, _i, _i64p, _sz, _sz, _vp, _vp, _vp],
    "pg_route_select_pooled": [_vp, _vp, _sz, _sz, _vp, _vp, _vp],
    "pg_cosine": [_vp, _vp, _sz, _vp, _vp],
    "pg_cache_create": [C.POINTER(_vp), _sz, _sz, C.c_double],
    "pg_cache_destroy": [_vp],
    "pg_cache_size": [_vp, _sp],
    "pg_cache_insert": [_vp, _vp, _i, C.POINTER(_i), _vp],
    "pg_cache_load": [_vp, _dp, _sz],
    "pg_retrieve": [_vp, _vp, _i, C.POINTER(RetrieveResultC), _vp, _vp, _vp],
    "pg_embed_normalize": [_vp, _i, _i, _sz, _sz, _vp, _vp],
    "pg_layer_create": [C.POINTER(_vp), _sz, _sz, _sz, _sz, _dp, _dp, _i],
    "pg_layer_create_device": [C.POINTER(_vp), _sz, _sz, _sz, _sz, _vp, _vp, _i, _i],
    "pg_layer_destroy": [_vp],
    "pg_layer_info": [_vp, _sp, _sp, _sp, _sp, C.POINTER(_i)],
    "pg_check_selection": [_vp, _up, _sz],
    "pg_masked_forward": [_vp, _vp, _sz, _i, _vp, _i, _sz, _vp, _i, _vp],
    "pg_aggregate_layout": [C.POINTER(_vp), _vp, _up, _sp, _sz, C.c_double, _vp],
    "pg_agg_destroy": [_vp],
    "pg_agg_patterns": [_vp, _sp],
    "pg_agg_shared": [_vp, _sp, _up],
    "pg_agg_residual": [_vp, _sz, _sp, _up, _sp, _u8p],
    "pg_agg_trace": [_vp, _sz, _sp, _sp],
    "pg_agg_bytes": [_vp, _sp],
    "pg_aggregated_forward": [_vp, _sz, _vp, _vp, _i, _sz, _vp, _i, _vp],
    "pg_aggregated_forward_batched": [_vp, _i32p, _i64p, _sz, _vp, _vp, _i, _vp],
    "pg_fill_normal_device": [_vp, _i, _sz, C.c_uint64, C.c_double, _vp],
    "pg_silu_mul": [_vp, _vp, _i, _sz, _vp, _i, _vp],
    "pg_copy_io": [_vp, _vp, _sz, _vp],
    "pg_peer_buffer_bytes": [_sz, _sz, _vp],
    "pg_agg_forward_peer": [_vp, _sz, _vp, _vp, _i, _i, _i, _vp, _i, _vp],
    "pg_mlp_forward_peer": [_vp, _vp, _vp, _sp, _vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp],
    "pg_ipc_get_handle": [_vp, _vp],
    "pg_ipc_open_handle": [_vp, _vp],
    "pg_ipc_close": [_vp],
    "pg_selection_mask_stride": [_vp, _vp],
    "pg_selection_masks": [_vp, _vp, _vp, _sz, _vp, _vp],
    "pg_masked_forward_union": [_vp, _vp, _sz, _vp, _sz, _vp, _vp, _i, _vp],
    "pg_module_forward_union": [_vp, _vp, _vp, _sz, _vp, _sz, _vp, _vp, _i, _vp],
    "pg_union_prog_create": [C.POINTER(_vp), _sz],
    "pg_union_prog_add_module": [_vp, _vp, _vp, _vp, _sz, _vp, _vp, _i, _sz, _i],
    "pg_union_prog_run": [_vp, _vp, _vp],
    "pg_union_prog_info": [_vp, C.POINTER(_sz), C.POINTER(_sz)],
    "pg_union_prog_destroy": [_vp],
    "pg_union_prog_debug": [_vp, _vp, _sz, C.POINTER(_i)],
    "pg_module_forward": [C.POINTER(_vp), _sz, _sp, _vp, _vp, C.POINTER(_vp), _i, _vp],
    "pg_prefill_batched": [C.POINTER(_vp), _i64p, _sz, _vp, _vp, _i, _vp],
    "pg_gemm_bf16": [_vp, C.c_int64, _vp, C.c_int64, _vp, C.c_int64, _sz, _sz, _sz, _i, _vp],
    "pg_chain_debug_dump": [C.POINTER(C.c_uint64), _sz],
    "pg_chain_workspace_release": [_vp],
    "pg_pack_bytes": [_vp, _sz, _sz, _sp, _sp],
    "pg_pack_selected": [_vp, _vp, _sz, _sz, _vp, _vp, _vp],
    "pg_prefill_packed": [_vp, _vp, _vp, _sz, _i64p, _sz, _vp, _vp, _i, _vp],
    "pg_prefill_gathered": [_vp, _vp, _vp, _sz, _i64p, _sz, _vp, _vp, _i, _vp],
    "pg_mlp_forward": [_vp, _vp, _vp, _sp, _vp, _vp, _vp, _vp, _i, _vp],
    "pg_mlp_forward_chain": [_vp, _vp, _vp, _sp, _sz, _vp, _vp, _vp, _i, _vp],
}
_VOID = {
    "pg_rng_fill_gaussian": [C.c_uint64, _dp, _sz],
    "pg_make_patterns": [C.c_uint64, _sz, _sp, _sp, _sz, _up],
}

_lib = None


def lib():
    """Load libparse_gpu.so once; raise if it is absent (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    for name, args in _VOID.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = None
    L.pg_last_error.restype = C.c_char_p
    L.pg_last_error.argtypes = []
    L.pg_launch_count.restype = C.c_uint64
    L.pg_launch_count.argtypes = []
    L.pg_abi_version.restype = C.c_int
    _lib = L
    return L


def check(code: int) -> None:
    if code:
        msg = lib().pg_last_error().decode(errors="replace")
        raise _ERR.get(code, RuntimeError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().pg_launch_count())
