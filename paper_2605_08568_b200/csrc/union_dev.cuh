// union_dev.cuh -- device helpers shared by the weights-on-M union GEMMs:
// the per-GEMM launch (union_wm.cu) and the persistent multi-phase program
// (union_prog.cu).  Tiles: 128 weight rows per CTA (256 per CTA pair) x up to
// 256 tokens, 64-wide k-blocks in 128-byte-swizzled shared memory.
#pragma once

#include <cuda.h>

#include "tc_ptx.cuh"

namespace pg {

constexpr int WM_BM = 128;    // weight rows per CTA (256 per pair)
constexpr int WM_BK = 64;     // k-block (128 bytes of bf16: one SW128 row)
constexpr int WM_TMAX = 256;  // tokens per launch (UMMA N)
constexpr int WM_W_BYTES = WM_BM * WM_BK * 2;            // 16 KB
constexpr int WM_X_BYTES = (WM_TMAX / 2) * WM_BK * 2;    // 16 KB: this CTA's half of the tokens
constexpr int WM_PART_FLOATS = WM_TMAX * WM_BM;          // one CTA's partial tile [T][128] f32
__device__ __forceinline__ unsigned long long wm_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void wm_bar_epi() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// value -> output element (row `row` of the weights = output column)
template <class G_>
__device__ __forceinline__ void wm_put(const G_& G, int tok, int row, float v) {
    if (G.out_bf16)
        static_cast<__nv_bfloat16*>(G.out)[(long long)tok * G.ldo + row] = __float2bfloat16_rn(v);
    else
        static_cast<float*>(G.out)[(long long)tok * G.ldo + row] = v;
}

// Epilogue staging: each epilogue warp transposes 32 rows x 32 tokens through
// its own shared-memory tile ([token][row], 4 KB) so the global stores are
// 16-byte vectors of consecutive rows of one token (instead of 2-byte
// transposed scalars).
constexpr int WM_STG_BYTES = 32 * 32 * 4;

// whole tile: TMEM -> smem transpose -> (mask) -> Y[t, row0 .. row0 + 31]
template <class G_>
__device__ __forceinline__ void wm_epi_direct(int Tp, int T, const G_& G, uint32_t taddr, int row0,
                                              const int32_t* tps, float* stg, int lane, int c0 = 0, int cstep = 1) {
    const int nch = Tp / 32;
    void* const out = G.out;
    const long long ldo = G.ldo;
    const bool bf16 = G.out_bf16 != 0;
    const uint8_t* const mask = G.mask;
    const long long mask_ld = G.mask_ld;
    const int R = G.Rs;
    uint32_t ra[32];
    for (int c = c0; c < nch; c += cstep) {
        // this chunk's 4 selection-mask words, loaded before the TMEM read and
        // every store (loads issued after stores would serialise on aliasing)
        uint2 mw[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int sgi = it * 32 + lane, tok = c * 32 + (sgi >> 2);
            mw[it] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
            if (mask && tok < T)
                mw[it] = __ldg(reinterpret_cast<const uint2*>(mask + (long long)tps[tok] * mask_ld + row0 + (sgi & 3) * 8));
        }
        tmem_ld32(taddr + 32u * c, ra);
        tmem_wait_ld();
        __syncwarp();  // the previous chunk's reads of stg are done
#pragma unroll
        for (int j = 0; j < 32; ++j) stg[j * 32 + lane] = __uint_as_float(ra[j]);  // [token][row]
        __syncwarp();
        // 32 tokens x 32 rows: lane takes 8 rows (a 16-byte bf16 / 2 x 16-byte f32 segment) of one token
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int sgi = it * 32 + lane, tl = sgi >> 2, part = sgi & 3;
            const int tok = c * 32 + tl, row = row0 + part * 8;
            if (tok >= T) continue;
            float v[8];
            const float4 a0 = *reinterpret_cast<const float4*>(stg + tl * 32 + part * 8);
            const float4 a1 = *reinterpret_cast<const float4*>(stg + tl * 32 + part * 8 + 4);
            v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!(((e < 4 ? mw[it].x : mw[it].y) >> (8 * (e & 3))) & 0xFFu)) v[e] = 0.f;
            if (row + 8 <= R) {
                if (bf16) {
                    uint4 w;
                    uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
                        wp[e] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + tok * ldo + row) = w;
                } else {
                    float* o = static_cast<float*>(out) + tok * ldo + row;
                    *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
                    *reinterpret_cast<float4*>(o + 4) = make_float4(v[4], v[5], v[6], v[7]);
                }
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (row + e < R) {
                        if (bf16) static_cast<__nv_bfloat16*>(out)[tok * ldo + row + e] = __float2bfloat16_rn(v[e]);
                        else static_cast<float*>(out)[tok * ldo + row + e] = v[e];
                    }
            }
        }
    }
}

// split tile: TMEM -> smem transpose -> f32 partial [Tp][128] (16-byte stores)
__device__ __forceinline__ void wm_epi_partial(int Tp, uint32_t taddr, float* dst, int q, float* stg,
                                               int lane) {
    const int nch = Tp / 32;
    uint32_t ra[32];
    for (int c = 0; c < nch; ++c) {
        tmem_ld32(taddr + 32u * c, ra);
        tmem_wait_ld();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) stg[j * 32 + lane] = __uint_as_float(ra[j]);
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 8; ++it) {  // 32 tokens x 128 bytes: lane takes 16 bytes
            const int sgi = it * 32 + lane, tl = sgi >> 3, part = sgi & 7;
            const float4 v = *reinterpret_cast<const float4*>(stg + tl * 32 + part * 4);
            __stcg(reinterpret_cast<float4*>(dst + (size_t)(c * 32 + tl) * WM_BM + q * 32 + part * 4), v);
        }
    }
}

}  // namespace pg
