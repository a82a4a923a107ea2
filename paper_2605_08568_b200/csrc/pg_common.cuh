// pg_common.cuh -- shared device/host helpers for the sm_100a rank-expert path.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "parse_gpu.h"

namespace pg {

// ---- error plumbing (C-ABI status + thread-local message) ----
struct Error {
    int code;
    std::string msg;
};
void set_error(int code, const std::string& msg);
inline Error invalid(const std::string& m) { return {PG_INVALID_ARGUMENT, m}; }
inline Error out_of_range(const std::string& m) { return {PG_OUT_OF_RANGE, m}; }
inline Error runtime(const std::string& m) { return {PG_RUNTIME_ERROR, m}; }

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define PG_CUDA_THROW(expr)                                                              \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            throw ::pg::Error{PG_CUDA_ERROR, std::string(#expr ": ") + cudaGetErrorString(_e)}; \
    } while (0)

#define PG_LAUNCH_CHECK()                                                                \
    do {                                                                                 \
        ::pg::count_launch();                                                            \
        cudaError_t _e = cudaGetLastError();                                             \
        if (_e != cudaSuccess)                                                           \
            throw ::pg::Error{PG_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(_e)}; \
    } while (0)

// ---- per-device host state (one process may drive several GPUs) ----
int current_device();
int device_sms();  // SM count of the current device (cached per device)
// Runs fn() once per device (under a lock; later callers on that device wait
// for it): kernel attributes, pool settings.  `tag` identifies the call site.
void once_per_device(const void* tag, void (*fn)());

inline cudaStream_t as_stream(pg_stream s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t dtype_size(pg_dtype d) { return d == PG_F64 ? 8 : d == PG_F32 ? 4 : 2; }

constexpr int kNumSMs = 148;
constexpr double kU = 1.1102230246251565e-16;  // 2^-53

// ---- dtype traits ----
template <typename W> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ double to_d(double v) { return v; }
__device__ __forceinline__ double to_d(float v) { return (double)v; }
__device__ __forceinline__ double to_d(__nv_bfloat16 v) { return (double)__bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_acc(float v);
template <> __device__ __forceinline__ float from_acc<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}
template <typename T> __device__ __forceinline__ T from_accd(double v);
template <> __device__ __forceinline__ double from_accd<double>(double v) { return v; }
template <> __device__ __forceinline__ float from_accd<float>(double v) { return (float)v; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// 128-bit streaming load that bypasses L1 allocation (weights are read once)
__device__ __forceinline__ int4 ld_stream(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---- launchers implemented per .cu (called from capi.cu) ----
struct SlotMap {
    // slot s -> storage column/row:
    //   idx != nullptr : idx[s] (gather; -1 = inactive)
    //   else           : s < run0_len ? s : run1_start + (s - run0_len)
    const int32_t* idx = nullptr;
    int run0_len = 0;
    int run1_start = 0;
    int run1_len = 0;
    const uint8_t* mask = nullptr;  // nullable; per slot in run0: 0 = inactive (z forced to 0)
    // device-resolved pattern (pg_aggregated_forward with pattern_dev): at kernel
    // start p = *dyn_pattern, run1 = dyn_table[2p..2p+1], mask = dyn_masks + p*stride
    const int32_t* dyn_pattern = nullptr;
    const int32_t* dyn_table = nullptr;
    const uint8_t* dyn_masks = nullptr;
    int dyn_mask_stride = 0;
    int cap = 0;  // host-side upper bound on nslots (smem / grid sizing when dyn_pattern is set)
    __host__ __device__ int nslots() const { return idx ? run0_len : run0_len + run1_len; }
};

__device__ __forceinline__ SlotMap resolve(SlotMap sm) {
    if (sm.dyn_pattern) {
        const int p = *sm.dyn_pattern;
        sm.run1_start = sm.dyn_table[2 * p];
        sm.run1_len = sm.dyn_table[2 * p + 1];
        sm.mask = sm.dyn_masks + (size_t)p * sm.dyn_mask_stride;
        sm.dyn_pattern = nullptr;
    }
    return sm;
}

}  // namespace pg
