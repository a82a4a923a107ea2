// block_utils.cuh -- block-wide scans, reductions and the exact (key, index)
// radix select used by the routing top-K and the cache arg-max.
#pragma once

#include "pg_common.cuh"

namespace pg {

// Orderable key for an f64: larger double -> larger key.  -0.0 is
// canonicalised to +0.0 because the reference's `logits[a] > logits[b]`
// treats them as equal (ties then fall to the lower index).
__device__ __forceinline__ uint64_t f64_key(double v) {
    if (v == 0.0) v = 0.0;
    uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(uint64_t k) {
    uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// Exclusive block scan of one int per thread; returns the prefix, writes the
// block total to *total.  scratch: >= 33 ints of shared memory.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < NT / 32 ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        scratch[lane] = s;  // inclusive
    }
    __syncthreads();
    int base = w ? scratch[w - 1] : 0;
    *total = scratch[NT / 32 - 1];
    __syncthreads();
    return base + x - v;
}

template <int NT>
__device__ __forceinline__ int block_sum_int(int v, int* scratch) {
    int total;
    block_excl_scan<NT>(v, scratch, &total);
    return total;
}

template <int NT>
__device__ __forceinline__ double block_max_f64(double v, double* scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_max(v);
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        double s = lane < NT / 32 ? scratch[lane] : -INFINITY;
        s = warp_max(s);
        if (lane == 0) scratch[32] = s;
    }
    __syncthreads();
    double r = scratch[32];
    __syncthreads();
    return r;
}

// K-th largest key among vals[0..r) by MSB-first 8-bit radix select.
// Returns the key; *need_eq = how many elements equal to it belong to the
// top-K (the rest of the top-K is strictly greater).  hist: 256 ints smem,
// sel: 2 ints smem.
template <int NT>
__device__ uint64_t radix_select_kth(const double* vals, int r, int K, int* hist, int* sel,
                                     int* need_eq) {
    uint64_t prefix = 0, maskbits = 0;
    int krem = K;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < r; i += NT) {
            uint64_t k = f64_key(vals[i]);
            if ((k & maskbits) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            // lane l owns digits [248-8l, 255-8l] (lane 0 the highest)
            int local = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) local += hist[255 - 8 * lane - b];
            int incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int before = incl - local;
            bool mine = before < krem && krem <= incl;
            unsigned ball = __ballot_sync(0xffffffffu, mine);
            int owner = __ffs(ball) - 1;
            if (lane == owner) {
                int cum = before;
                for (int b = 0; b < 8; ++b) {
                    int d = 255 - 8 * lane - b;
                    int h = hist[d];
                    if (cum + h >= krem) {
                        sel[0] = d;
                        sel[1] = krem - cum;
                        break;
                    }
                    cum += h;
                }
            }
        }
        __syncthreads();
        prefix |= (uint64_t)sel[0] << shift;
        maskbits |= (uint64_t)0xff << shift;
        krem = sel[1];
        __syncthreads();
    }
    *need_eq = krem;
    return prefix;
}

}  // namespace pg
