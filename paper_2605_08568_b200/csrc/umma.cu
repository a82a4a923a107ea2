// umma.cu -- K5: grouped bf16 GEMM on the 5th-gen tensor cores (tcgen05 + TMEM
// + TMA) for prefill, i.e. T > 8 tokens through a rank-expert layer:
//   stage 1  Z[T, Kp] = X[T, n]  . B_S^T[Kp, n]^T   (both operands K-major)
//   stage 2  Y[T, m]  = Z[T, Kp] . A_S [m, Kp]^T    (both operands K-major)
// (rank_experts.hpp:52-72 / exec_engine.hpp:193-236 at large T).  A "group" is
// one GEMM; heterogeneous prompts (each with its own S) are one launch.
//
// Persistent, warp-specialised, one CTA per SM (192 threads):
//   warp 0      TMA producer: 128x64 A box + BNx64 B box per k-block, 128B
//               swizzle, 4-stage smem ring (full/empty mbarriers);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (kind::f16, bf16 x bf16 -> f32, M=128, N=BN<=256, K=16),
//               double-buffered accumulators (2 x 256 TMEM columns);
//   warps 2-5   epilogue: tcgen05.ld 32x32b.x32 -> registers -> bf16/f32 ->
//               global (row/column masked), then release the accumulator.
// Roofline: tensor-pipe-bound, 2*M*N*K flops per group.
#include <cuda.h>

#include <cstdio>

#include <algorithm>
#include <memory>
#include <mutex>
#include <vector>

#include "tc_ptx.cuh"
#include "umma.cuh"

namespace pg {

constexpr int UM_BM = 128, UM_BK = 64, UM_BN_MAX = 256, UM_STAGES = 4;
constexpr int UM_THREADS = 192;
constexpr int UM_A_BYTES = UM_BM * UM_BK * 2;          // 16 KB
constexpr int UM_B_BYTES = UM_BN_MAX * UM_BK * 2;      // 32 KB (max)
constexpr int UM_STAGE_BYTES = UM_A_BYTES + UM_B_BYTES;
constexpr int UM_SMEM = UM_STAGES * UM_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

constexpr int UM_MAX_GROUPS = 32;


struct UmmaGroup {
    void* out;                 // [M, ldo] row-major
    long long ldo;
    int M, N, K;
    int bn;                    // tile N (multiple of 16, <= 256)
    int out_bf16;              // 1: bf16 out, 0: f32 out
    int tiles_m, tiles_n;
    int tile_base;             // prefix sum of tiles over groups
    const uint8_t* mask;       // nullable: per-row column mask (see UmmaSpec)
    long long mask_ld;
    const int32_t* row_pat;
    int direct_epi;
    int a_hint, b_hint;
    const int32_t* b_idx;  // gathered B rows (pair kernel), see UmmaSpec
    int b_idx_n, b_idx_rows;
};

// Passed as one __grid_constant__ parameter block (< 32 KB): TMA reads the
// tensor maps straight from parameter space, no staging copy.
struct __align__(64) UmmaParams {
    CUtensorMap maps[2 * UM_MAX_GROUPS];  // [2g] A [M rows, K] box {64,128}; [2g+1] B [N rows, K] box {64,BN}
    CUtensorMap omaps[UM_MAX_GROUPS];     // output [M rows, N] box {32, 32} (TMA-store epilogue of the pair kernel)
    UmmaGroup groups[UM_MAX_GROUPS];
    int ngroups;
    int total_tiles;
    int epi_deep;  // bf16 TMA-store epilogue: 4 x 2 KB staging slots per warp in flight (else 2)
    int gather;    // some group gathers its B rows: the pair kernel's producer runs as a whole warp
};

// ---- epilogue helpers: TMEM -> registers -> bf16 / f32 -> global, with the
// next chunk's tcgen05.ld in flight while the current chunk is stored
__device__ __forceinline__ void store_chunk(const UmmaGroup& G, int row, int n0, int c0, const uint32_t (&r)[32]) {
    if (row >= G.M) return;
    const int cb = n0 + c0;
    // columns of THIS tile only: the tile may be narrower than a 32-column chunk
    const int valid = min(32, min(G.bn - c0, G.N - cb));
    if (G.out_bf16) {
        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(G.out) + (long long)row * G.ldo + cb;
        if (valid == 32 && ((G.ldo & 7) == 0)) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                uint4 w;
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[v * 8 + 2 * e]),
                                                             __uint_as_float(r[v * 8 + 2 * e + 1]));
                    wp[e] = *reinterpret_cast<uint32_t*>(&h);
                }
                *reinterpret_cast<uint4*>(o + v * 8) = w;
            }
        } else {  // unrolled with a predicate: a dynamic index would put r in local memory
#pragma unroll
            for (int e = 0; e < 32; ++e)
                if (e < valid) o[e] = __float2bfloat16_rn(__uint_as_float(r[e]));
        }
    } else {
        float* o = static_cast<float*>(G.out) + (long long)row * G.ldo + cb;
        if (valid == 32 && ((G.ldo & 3) == 0)) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
                *reinterpret_cast<float4*>(o + v * 4) = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                                                    __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
        } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
                if (e < valid) o[e] = __uint_as_float(r[e]);
        }
    }
}
// union-masked batches: zero the columns this row's pattern does not select
// (32 mask bytes per chunk, two 16-byte loads; mask_ld >= N rounded up + 32)
__device__ __forceinline__ void mask_chunk(const UmmaGroup& G, int row, int col0, uint32_t (&r)[32]) {
    if (G.mask == nullptr) return;
    if (row >= G.M) return;
    const uint8_t* mr = G.mask + (long long)__ldg(G.row_pat + row) * G.mask_ld + col0;
    const uint4 m0 = __ldg(reinterpret_cast<const uint4*>(mr));
    const uint4 m1 = __ldg(reinterpret_cast<const uint4*>(mr + 16));
    const uint32_t w[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int e = 0; e < 32; ++e)
        if (((w[e >> 2] >> (8 * (e & 3))) & 0xFFu) == 0) r[e] = 0u;
}

// one accumulator tile: lanes of quadrant q, columns [0, bn) in 32-column chunks
__device__ __forceinline__ void epilogue_tile(const UmmaGroup& G, uint32_t tbase, int q, int row, int n0) {
    const int nch = (G.bn + 31) / 32;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
    uint32_t ra[32], rb[32];
    tmem_ld32(lane_base, ra);
    for (int c = 0; c < nch; c += 2) {
        tmem_wait_ld();
        if (c + 1 < nch) tmem_ld32(lane_base + (uint32_t)(32 * (c + 1)), rb);
        mask_chunk(G, row, n0 + 32 * c, ra);
        store_chunk(G, row, n0, 32 * c, ra);
        if (c + 1 >= nch) break;
        tmem_wait_ld();
        if (c + 2 < nch) tmem_ld32(lane_base + (uint32_t)(32 * (c + 2)), ra);
        mask_chunk(G, row, n0 + 32 * (c + 1), rb);
        store_chunk(G, row, n0, 32 * (c + 1), rb);
    }
}

__global__ void __launch_bounds__(UM_THREADS, 1) k_umma_grouped(const __grid_constant__ UmmaParams P) {
    extern __shared__ __align__(1024) unsigned char usmem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(usmem) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + UM_STAGES * UM_STAGE_BYTES);
    uint64_t* full = bars;                     // [STAGES]
    uint64_t* empty = bars + UM_STAGES;        // [STAGES]
    uint64_t* tfull = bars + 2 * UM_STAGES;    // [2]
    uint64_t* tempty = bars + 2 * UM_STAGES + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * UM_STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < UM_STAGES; ++s) {
            u_mbar_init(u_smem(&full[s]), 1);
            u_mbar_init(u_smem(&empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            u_mbar_init(u_smem(&tfull[a]), 1);
            u_mbar_init(u_smem(&tempty[a]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // allocate all 512 TMEM columns (2 accumulators x 256)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(u_smem(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    // programmatic dependent launch: the next grid may start its prologue now;
    // this grid reads its operands only after the previous grid completed
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            uint64_t pf, pl;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
                int g = 0;
                while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
                const UmmaGroup& G = P.groups[g];
                const int lt = t - G.tile_base;
                const int m0 = (lt % G.tiles_m) * UM_BM, n0 = (lt / G.tiles_m) * G.bn;
                const int kbs = (G.K + UM_BK - 1) / UM_BK;
                const uint32_t bytes = UM_A_BYTES + (uint32_t)G.bn * UM_BK * 2;
                for (int kb = 0; kb < kbs; ++kb) {
                    u_mbar_wait(u_smem(&empty[s]), ph ^ 1);
                    const uint32_t fb = u_smem(&full[s]);
                    u_mbar_arrive_tx(fb, bytes);
                    unsigned char* st = base + s * UM_STAGE_BYTES;
                    if (G.a_hint) u_tma_2d_h(u_smem(st), &P.maps[2 * g], kb * UM_BK, m0, fb, u_policy(G.a_hint, pf, pl));
                    else u_tma_2d(u_smem(st), &P.maps[2 * g], kb * UM_BK, m0, fb);
                    if (G.b_hint)
                        u_tma_2d_h(u_smem(st + UM_A_BYTES), &P.maps[2 * g + 1], kb * UM_BK, n0, fb,
                                   u_policy(G.b_hint, pf, pl));
                    else u_tma_2d(u_smem(st + UM_A_BYTES), &P.maps[2 * g + 1], kb * UM_BK, n0, fb);
                    if (++s == UM_STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
                int g = 0;
                while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
                const UmmaGroup& G = P.groups[g];
                const int kbs = (G.K + UM_BK - 1) / UM_BK;
                const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(G.bn >> 3) << 17) |
                                       ((uint32_t)(UM_BM >> 4) << 24);
                u_mbar_wait(u_smem(&tempty[acc]), aph ^ 1);  // epilogue drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(acc * UM_BN_MAX);
                for (int kb = 0; kb < kbs; ++kb) {
                    u_mbar_wait(u_smem(&full[s]), ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = u_smem(base + s * UM_STAGE_BYTES), sb = sa + UM_A_BYTES;
#pragma unroll
                    for (int k = 0; k < UM_BK / 16; ++k)
                        u_mma(d, u_desc(sa + k * 32), u_desc(sb + k * 32), idesc, (kb | k) != 0);
                    u_commit(u_smem(&empty[s]));  // frees the smem stage when these MMAs retire
                    if (++s == UM_STAGES) { s = 0; ph ^= 1; }
                }
                u_commit(u_smem(&tfull[acc]));  // accumulator ready for the epilogue
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2-5)
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        int acc = 0;
        uint32_t aph = 0;
        for (int t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
            int g = 0;
            while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
            const UmmaGroup& G = P.groups[g];
            const int lt = t - G.tile_base;
            const int m0 = (lt % G.tiles_m) * UM_BM, n0 = (lt / G.tiles_m) * G.bn;
            u_mbar_wait(u_smem(&tfull[acc]), aph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int row = m0 + q * 32 + lane;
            epilogue_tile(G, tmem + (uint32_t)(acc * UM_BN_MAX), q, row, n0);
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) u_mbar_arrive(u_smem(&tempty[acc]));
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}


// ---------------------------------------------------------------- 2-CTA variant
// CTA pair (cluster of 2, cta_group::2): 256 x BN tiles, each CTA of the pair
// loads its 128 rows of A and its BN/2 rows of B; the leader's single thread
// issues tcgen05.mma.cta_group::2 (M = 256) over both CTAs' shared memory and
// each CTA's TMEM receives its 128 rows.  Half the shared-memory bytes per
// MMA of the 1-CTA kernel, so the ring is 6 stages deep.
constexpr int U2_STAGES = 6;
constexpr int U2_A_BYTES = UM_BM * UM_BK * 2;                 // 16 KB (this CTA's 128 rows)
constexpr int U2_B_BYTES = (UM_BN_MAX / 2) * UM_BK * 2;       // 16 KB (this CTA's BN/2 rows)
constexpr int U2_STAGE_BYTES = U2_A_BYTES + U2_B_BYTES;
constexpr int U2_OUT_BYTES = 32 * 32 * 4;  // one 32 x 32 output chunk (f32 worst case)
// [align slack 1 KB][ring][barriers, 1 KB][per-warp output staging]
constexpr int U2_SMEM = U2_STAGES * U2_STAGE_BYTES + 1024 + 1024 + 4 * 2 * U2_OUT_BYTES;
// the CTA-pair kernel (k_umma_grouped2): U2_EPI_WARPS epilogue warps -- with 8,
// two per TMEM lane quadrant take alternate 32-column chunks (short-K tiles are
// drain-bound), and the ring gives up a stage for their staging
#ifndef U2_EPI_WARPS_CFG
#define U2_EPI_WARPS_CFG 4
#endif
constexpr int U2_EPI_WARPS = U2_EPI_WARPS_CFG;
constexpr int P2_THREADS = 64 + 32 * U2_EPI_WARPS;
constexpr int P2_STAGES = U2_EPI_WARPS == 8 ? 5 : U2_STAGES;
constexpr int P2_SMEM = P2_STAGES * U2_STAGE_BYTES + 1024 + 1024 + U2_EPI_WARPS * 2 * U2_OUT_BYTES;
static_assert(P2_SMEM <= 227 * 1024, "pair kernel shared memory");

// ---- k_umma_grouped4 (PG_UMMA_MC=1, off by default): clusters of two CTA
// pairs on consecutive M tiles of one N tile; each CTA loads a quarter of the
// B tile and multicasts it to its counterpart in the other pair, so per SM the
// B bytes per flop halve.  Measured: +9 % TFLOP/s per SM, but only 33 clusters
// of 4 fit (132 SMs) against 74 pairs (148 SMs), so whole-GPU throughput is
// equal or lower (profiles/r1_prefill_config3.txt).  Parity tests pass with it.
// B quarter tile multicast to the same-parity CTA of both pairs of a 4-CTA cluster
__device__ __forceinline__ void u_tma_2d_pair_mc(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                                 uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void u_commit2_mask(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"(mask)
                 : "memory");
}
// TMA-store epilogue: each warp stages its 32 rows x 32 columns in shared
// memory (double-buffered) and one lane stores the box with
// cp.async.bulk.tensor -- coalesced rows instead of one row per thread.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
                 "r"(y), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void epilogue_tile_tma(const UmmaGroup& G, const CUtensorMap* omap, uint32_t tbase, int q,
                                                  int lane, int row0, int n0, unsigned char* stage, int& nbuf,
                                                  int epi_deep, int c0 = 0, int cstep = 1) {
    const int nch = (G.bn + 31) / 32;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
    const int es = G.out_bf16 ? 2 : 4;
    // the warp's 8 KB of staging: 2 slots of a 32 x 32 f32 box, or (bf16) 4
    // slots of 2 KB -- stores in flight per warp bound the drain of short-K tiles
    const bool deep = epi_deep && G.out_bf16;
    const int slot_bytes = 32 * 32 * es;
    uint32_t ra[32], rb[32];
    auto emit = [&](int c, uint32_t (&r)[32]) {
        const int c0 = 32 * c;
        mask_chunk(G, row0 + lane, n0 + c0, r);
        if (c0 + 32 > G.bn) {  // partial chunk: the box would spill into the next tile
            store_chunk(G, row0 + lane, n0, c0, r);
            return;
        }
        unsigned char* buf = stage + (deep ? (nbuf & 3) * slot_bytes : (nbuf & 1) * U2_OUT_BYTES);
        if (lane == 0) {  // buf's previous store has read it
            if (deep) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncwarp();
        unsigned char* dst = buf + lane * 32 * es;
        if (G.out_bf16) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                uint4 w;
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[v * 8 + 2 * e]),
                                                             __uint_as_float(r[v * 8 + 2 * e + 1]));
                    wp[e] = *reinterpret_cast<uint32_t*>(&h);
                }
                *reinterpret_cast<uint4*>(dst + v * 16) = w;
            }
        } else {
#pragma unroll
            for (int v = 0; v < 8; ++v)
                *reinterpret_cast<uint4*>(dst + v * 16) = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(omap, u_smem(buf), n0 + c0, row0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++nbuf;
    };
    if (c0 >= nch) return;
    tmem_ld32(lane_base + (uint32_t)(32 * c0), ra);
    for (int c = c0; c < nch; c += 2 * cstep) {
        tmem_wait_ld();
        if (c + cstep < nch) tmem_ld32(lane_base + (uint32_t)(32 * (c + cstep)), rb);
        emit(c, ra);
        if (c + cstep >= nch) break;
        tmem_wait_ld();
        if (c + 2 * cstep < nch) tmem_ld32(lane_base + (uint32_t)(32 * (c + 2 * cstep)), ra);
        emit(c + cstep, rb);
    }
}

// GATHER: some group gathers its B rows (one gather4 per producer lane); a
// separate instantiation, so plain launches keep the lane-0 producer loop
template <bool GATHER>
__global__ void __launch_bounds__(P2_THREADS, 1) k_umma_grouped2(const __grid_constant__ UmmaParams P) {
    extern __shared__ __align__(1024) unsigned char usmem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(usmem) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + P2_STAGES * U2_STAGE_BYTES);
    uint64_t* full = bars;                        // [STAGES] (used in the leader)
    uint64_t* empty = bars + P2_STAGES;           // [STAGES] (each CTA)
    uint64_t* tfull = bars + 2 * P2_STAGES;       // [2] (each CTA)
    uint64_t* tempty = bars + 2 * P2_STAGES + 2;  // [2] (used in the leader: both CTAs' epilogues)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P2_STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < P2_STAGES; ++s) {
            u_mbar_init(u_smem(&full[s]), 1);
            u_mbar_init(u_smem(&empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            u_mbar_init(u_smem(&tfull[a]), 1);
            u_mbar_init(u_smem(&tempty[a]), 2 * U2_EPI_WARPS);  // epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // same warp in both CTAs: 2 accumulators x 256 columns
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(u_smem(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // see k_umma_grouped

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        // lane 0 drives the ring; with gathered B rows every lane issues one
        // gather4 (four rows) of this CTA's bn/2 rows per k-block (the whole-warp
        // loop costs ~2.5 % on plain launches, so only gathering launches run it)
        if (GATHER || lane == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        uint64_t pf, pl, pn;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pn));
        int s = 0;
        uint32_t ph = 0;
        for (int t = pair; t < P.total_tiles; t += npairs) {
            int g = 0;
            while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
            const UmmaGroup& G = P.groups[g];
            const int lt = t - G.tile_base;
            const int m0 = (lt % G.tiles_m) * 2 * UM_BM + (int)rank * UM_BM;
            const int n0 = (lt / G.tiles_m) * G.bn + (int)rank * (G.bn / 2);
            const int kbs = (G.K + UM_BK - 1) / UM_BK;
            const uint32_t bytes = 2 * (UM_A_BYTES + (uint32_t)(G.bn / 2) * UM_BK * 2);  // both CTAs
            const bool gat = GATHER && G.b_idx != nullptr, mine = gat && 4 * lane < G.bn / 2;
            int gr0 = 0, gr1 = 0, gr2 = 0, gr3 = 0;
            if (mine) {
                const int j = n0 + 4 * lane;
                gr0 = j < G.b_idx_n ? __ldg(G.b_idx + j) : G.b_idx_rows;
                gr1 = j + 1 < G.b_idx_n ? __ldg(G.b_idx + j + 1) : G.b_idx_rows;
                gr2 = j + 2 < G.b_idx_n ? __ldg(G.b_idx + j + 2) : G.b_idx_rows;
                gr3 = j + 3 < G.b_idx_n ? __ldg(G.b_idx + j + 3) : G.b_idx_rows;
            }
            const uint64_t bpol = G.b_hint ? u_policy(G.b_hint, pf, pl) : pn;
            for (int kb = 0; kb < kbs; ++kb) {
                if (lane == 0) u_mbar_wait(u_smem(&empty[s]), ph ^ 1);
                if (GATHER) __syncwarp();
                const uint32_t fb = leader_addr(u_smem(&full[s]));
                unsigned char* st = base + s * U2_STAGE_BYTES;
                if (lane == 0) {
                    if (leader) u_mbar_arrive_tx_cluster(fb, bytes);
                    if (G.a_hint)
                        u_tma_2d_pair_h(u_smem(st), &P.maps[2 * g], kb * UM_BK, m0, fb, u_policy(G.a_hint, pf, pl));
                    else u_tma_2d_pair(u_smem(st), &P.maps[2 * g], kb * UM_BK, m0, fb);
                    if (!gat) {
                        if (G.b_hint)
                            u_tma_2d_pair_h(u_smem(st + U2_A_BYTES), &P.maps[2 * g + 1], kb * UM_BK, n0, fb,
                                            u_policy(G.b_hint, pf, pl));
                        else u_tma_2d_pair(u_smem(st + U2_A_BYTES), &P.maps[2 * g + 1], kb * UM_BK, n0, fb);
                    }
                }
                if (mine)
                    u_tma_gather4_pair_h(u_smem(st + U2_A_BYTES) + (uint32_t)lane * 4 * UM_BK * 2, &P.maps[2 * g + 1],
                                         kb * UM_BK, gr0, gr1, gr2, gr3, fb, bpol);
                if (++s == P2_STAGES) { s = 0; ph ^= 1; }
            }
        }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (leader && lane == 0) {
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int t = pair; t < P.total_tiles; t += npairs) {
                int g = 0;
                while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
                const UmmaGroup& G = P.groups[g];
                const int kbs = (G.K + UM_BK - 1) / UM_BK;
                const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(G.bn >> 3) << 17) |
                                       ((uint32_t)((2 * UM_BM) >> 4) << 24);
                u_mbar_wait(u_smem(&tempty[acc]), aph ^ 1);  // both CTAs drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(acc * UM_BN_MAX);
                for (int kb = 0; kb < kbs; ++kb) {
                    u_mbar_wait(u_smem(&full[s]), ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = u_smem(base + s * U2_STAGE_BYTES), sb = sa + U2_A_BYTES;
#pragma unroll
                    for (int k = 0; k < UM_BK / 16; ++k)
                        u_mma2(d, u_desc(sa + k * 32), u_desc(sb + k * 32), idesc, (kb | k) != 0);
                    u_commit2(u_smem(&empty[s]));  // frees the stage in both CTAs
                    if (++s == P2_STAGES) { s = 0; ph ^= 1; }
                }
                u_commit2(u_smem(&tfull[acc]));  // accumulator ready in both CTAs
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2-5, both CTAs)
        const int q = warp & 3, h = (warp - 2) >> 2;  // TMEM lane quadrant; column-chunk half (8 warps)
        unsigned char* ostage = base + P2_STAGES * U2_STAGE_BYTES + 1024 + (warp - 2) * 2 * U2_OUT_BYTES;
        int nbuf = 0;
        int acc = 0;
        uint32_t aph = 0;
        for (int t = pair; t < P.total_tiles; t += npairs) {
            int g = 0;
            while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
            const UmmaGroup& G = P.groups[g];
            const int lt = t - G.tile_base;
            const int m0 = (lt % G.tiles_m) * 2 * UM_BM + (int)rank * UM_BM, n0 = (lt / G.tiles_m) * G.bn;
            u_mbar_wait(u_smem(&tfull[acc]), aph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int row = m0 + q * 32 + lane;
            if (G.direct_epi) {
                if (h == 0) epilogue_tile(G, tmem + (uint32_t)(acc * UM_BN_MAX), q, row, n0);
            }
            else epilogue_tile_tma(G, &P.omaps[g], tmem + (uint32_t)(acc * UM_BN_MAX), q, lane, m0 + q * 32, n0, ostage, nbuf,
                                   P.epi_deep, U2_EPI_WARPS == 8 ? h : 0, U2_EPI_WARPS / 4);
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) u_mbar_arrive_cluster(leader_addr(u_smem(&tempty[acc])));
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
    }
    if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores out of smem
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void __launch_bounds__(UM_THREADS, 1) k_umma_grouped4(const __grid_constant__ UmmaParams P) {
    extern __shared__ __align__(1024) unsigned char usmem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(usmem) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + U2_STAGES * U2_STAGE_BYTES);
    uint64_t* full = bars;                        // [STAGES] (used in the leader)
    uint64_t* empty = bars + U2_STAGES;           // [STAGES] (each CTA)
    uint64_t* tfull = bars + 2 * U2_STAGES;       // [2] (each CTA)
    uint64_t* tempty = bars + 2 * U2_STAGES + 2;  // [2] (used in the leader: both CTAs' epilogues)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * U2_STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // cluster of two CTA pairs: ranks {0,1} and {2,3}; both pairs work on the
    // same N tile (consecutive M tiles) and share its B tile: each CTA loads a
    // quarter of the B rows and multicasts it to its counterpart in the other pair
    const uint32_t crank = cluster_rank();
    const uint32_t rank = crank & 1u, pp = crank >> 1;
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 2, npairs = gridDim.x >> 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < U2_STAGES; ++s) {
            u_mbar_init(u_smem(&full[s]), 1);
            u_mbar_init(u_smem(&empty[s]), 2);  // both pairs' MMAs read this stage's B
        }
        for (int a = 0; a < 2; ++a) {
            u_mbar_init(u_smem(&tfull[a]), 1);
            u_mbar_init(u_smem(&tempty[a]), 8);  // 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // same warp in both CTAs: 2 accumulators x 256 columns
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(u_smem(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // see k_umma_grouped

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            uint64_t pf, pl;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
            int s = 0;
            uint32_t ph = 0;
            for (int t = pair; t < P.total_tiles; t += npairs) {
                int g = 0;
                while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
                const UmmaGroup& G = P.groups[g];
                const int lt = t - G.tile_base;
                const int m0 = (lt % G.tiles_m) * 4 * UM_BM + (int)pp * 2 * UM_BM + (int)rank * UM_BM;
                const int nq = (lt / G.tiles_m) * G.bn + (int)rank * (G.bn / 2) + (int)pp * (G.bn / 4);
                const uint16_t mc = (uint16_t)((1u << rank) | (1u << (rank + 2)));
                const int kbs = (G.K + UM_BK - 1) / UM_BK;
                const uint32_t bytes = 2 * (UM_A_BYTES + (uint32_t)(G.bn / 2) * UM_BK * 2);  // both CTAs
                for (int kb = 0; kb < kbs; ++kb) {
                    u_mbar_wait(u_smem(&empty[s]), ph ^ 1);
                    const uint32_t fb = leader_addr(u_smem(&full[s]));
                    if (leader) u_mbar_arrive_tx_cluster(fb, bytes);
                    unsigned char* st = base + s * U2_STAGE_BYTES;
                    if (G.a_hint)
                        u_tma_2d_pair_h(u_smem(st), &P.maps[2 * g], kb * UM_BK, m0, fb, u_policy(G.a_hint, pf, pl));
                    else u_tma_2d_pair(u_smem(st), &P.maps[2 * g], kb * UM_BK, m0, fb);
                    u_tma_2d_pair_mc(u_smem(st + U2_A_BYTES + pp * (G.bn / 4) * UM_BK * 2), &P.maps[2 * g + 1],
                                     kb * UM_BK, nq, fb, mc);
                    if (++s == U2_STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (leader && lane == 0) {
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int t = pair; t < P.total_tiles; t += npairs) {
                int g = 0;
                while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
                const UmmaGroup& G = P.groups[g];
                const int kbs = (G.K + UM_BK - 1) / UM_BK;
                const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(G.bn >> 3) << 17) |
                                       ((uint32_t)((2 * UM_BM) >> 4) << 24);
                u_mbar_wait(u_smem(&tempty[acc]), aph ^ 1);  // both CTAs drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(acc * UM_BN_MAX);
                for (int kb = 0; kb < kbs; ++kb) {
                    u_mbar_wait(u_smem(&full[s]), ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = u_smem(base + s * U2_STAGE_BYTES), sb = sa + U2_A_BYTES;
#pragma unroll
                    for (int k = 0; k < UM_BK / 16; ++k)
                        u_mma2(d, u_desc(sa + k * 32), u_desc(sb + k * 32), idesc, (kb | k) != 0);
                    u_commit2_mask(u_smem(&empty[s]), 0xF);  // this pair is done with the stage (all 4 CTAs)
                    if (++s == U2_STAGES) { s = 0; ph ^= 1; }
                }
                u_commit2_mask(u_smem(&tfull[acc]), (uint16_t)(3u << (2 * pp)));  // accumulator ready in this pair
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2-5, both CTAs)
        const int q = warp & 3;
        unsigned char* ostage = base + U2_STAGES * U2_STAGE_BYTES + 1024 + (q) * 2 * U2_OUT_BYTES;
        int nbuf = 0;
        int acc = 0;
        uint32_t aph = 0;
        for (int t = pair; t < P.total_tiles; t += npairs) {
            int g = 0;
            while (g + 1 < P.ngroups && P.groups[g + 1].tile_base <= t) ++g;
            const UmmaGroup& G = P.groups[g];
            const int lt = t - G.tile_base;
            const int m0 = (lt % G.tiles_m) * 4 * UM_BM + (int)pp * 2 * UM_BM + (int)rank * UM_BM,
                      n0 = (lt / G.tiles_m) * G.bn;
            u_mbar_wait(u_smem(&tfull[acc]), aph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int row = m0 + q * 32 + lane;
            if (G.direct_epi) epilogue_tile(G, tmem + (uint32_t)(acc * UM_BN_MAX), q, row, n0);
            else epilogue_tile_tma(G, &P.omaps[g], tmem + (uint32_t)(acc * UM_BN_MAX), q, lane, m0 + q * 32, n0, ostage, nbuf,
                                   P.epi_deep);
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) u_mbar_arrive_cluster(leader_addr(u_smem(&tempty[acc])));
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
    }
    if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores out of smem
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    if (!fn) throw Error{PG_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable"};
    return fn;
}

// 2-D bf16 K-major operand [rows, K] with row stride ld (elements), box {64, box_rows}
CUtensorMap make_map(const void* ptr, int rows, int K, long long ld, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {UM_BK, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error{PG_CUDA_ERROR, "cuTensorMapEncodeTiled failed"};
    return m;
}

CUtensorMap make_store_map(void* ptr, int rows, int cols, long long ld, bool bf16, int box_cols, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * (bf16 ? 2 : 4)};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = get_encode()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr,
                                    dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error{PG_CUDA_ERROR, "cuTensorMapEncodeTiled failed (store map)"};
    return m;
}

static CUtensorMap make_out_map(void* ptr, int rows, int cols, long long ld, bool bf16) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * (bf16 ? 2 : 4)};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = get_encode()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr,
                                    dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error{PG_CUDA_ERROR, "cuTensorMapEncodeTiled failed (output)"};
    return m;
}

static int pick_bn(int N) {
    const int tiles = (N + UM_BN_MAX - 1) / UM_BN_MAX;
    int bn = (N + tiles - 1) / tiles;
    bn = (bn + 15) / 16 * 16;
    return std::min(bn, UM_BN_MAX);
}

static int umma_pdl() {
    static const int v = [] {
        const char* e = getenv("PG_UMMA_PDL");
        return e ? atoi(e) : 1;
    }();
    return v;
}

static int umma_pairs_enabled() {
    static const int v = [] {
        const char* e = getenv("PG_UMMA_2CTA");
        return e ? atoi(e) : 1;
    }();
    return v;
}

void launch_umma(const std::vector<UmmaSpec>& specs, cudaStream_t st) {
    once_per_device(reinterpret_cast<const void*>(&k_umma_grouped), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_umma_grouped, cudaFuncAttributeMaxDynamicSharedMemorySize, UM_SMEM));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_umma_grouped2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_umma_grouped2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_umma_grouped4, cudaFuncAttributeMaxDynamicSharedMemorySize, U2_SMEM));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_umma_grouped4, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    });
    // CTA pairs for batches whose every GEMM has at least 256 rows
    bool pairs = umma_pairs_enabled() != 0;
    for (const UmmaSpec& sp : specs)  // (+ 16-byte aligned output rows for the TMA-store epilogue)
        pairs = pairs && sp.M >= 2 * UM_BM && (sp.ldo * (sp.out_bf16 ? 2 : 4)) % 16 == 0 &&
                reinterpret_cast<uintptr_t>(sp.out) % 16 == 0;
    const int sms = device_sms();
    for (size_t g0 = 0; g0 < specs.size(); g0 += UM_MAX_GROUPS) {
        const int ng = (int)std::min<size_t>(UM_MAX_GROUPS, specs.size() - g0);
        auto P = std::make_unique<UmmaParams>();
        int tiles = 0;
        static const int mc_env = [] {  // experiments: clusters of two CTA pairs sharing B by multicast
            const char* e = getenv("PG_UMMA_MC");
            return e ? atoi(e) : 0;
        }();
        const bool mc = pairs && mc_env != 0;
        // few tiles (small-batch decode through the tensor cores): one narrower
        // tile width for the whole launch until the SMs are covered, minimising
        // waves x tile width (time per tile ~ bn x K)
        int common_bn = 0;
        {
            const int rows = pairs ? 2 * UM_BM : UM_BM, slots = pairs ? sms / 2 : sms, step = pairs ? 32 : 16;
            auto tiles_at = [&](int cap) {
                long t = 0;
                for (int g = 0; g < ng; ++g) {
                    const UmmaSpec& s = specs[g0 + g];
                    int bn = pick_bn(s.N);
                    if (pairs) bn = std::min(UM_BN_MAX, (bn + 31) / 32 * 32);
                    if (cap > 0) bn = std::min(bn, cap);
                    t += (long)((s.M + rows - 1) / rows) * ((s.N + bn - 1) / bn);
                }
                return t;
            };
            bool autob = true;
            for (int g = 0; g < ng; ++g) autob = autob && specs[g0 + g].bn == 0;
            if (autob && tiles_at(0) < slots) {
                long best = -1;
                for (int bn = UM_BN_MAX; bn >= step; bn -= step) {
                    const long cost = ((tiles_at(bn) + slots - 1) / slots) * (long)bn;
                    if (best < 0 || cost < best) { best = cost; common_bn = bn; }
                }
            }
        }
        for (int g = 0; g < ng; ++g) {
            const UmmaSpec& s = specs[g0 + g];
            if ((s.lda * 2) % 16 || (s.ldb * 2) % 16 || s.K % 8)
                throw Error{PG_INVALID_ARGUMENT, "umma: operands need 16-byte aligned rows"};
            UmmaGroup& G = P->groups[g];
            G.bn = pick_bn(s.N);
            if (pairs) G.bn = (G.bn + 31) / 32 * 32;  // each CTA of a pair loads bn/2 rows (multiple of 16)
            if (G.bn > UM_BN_MAX) G.bn = UM_BN_MAX;
            if (s.bn > 0) G.bn = s.bn;
            else if (common_bn > 0) G.bn = std::min(G.bn, common_bn);
            P->maps[2 * g] = make_map(s.a, s.M, s.K, s.lda, UM_BM);
            if (s.b_idx) {  // gathered B rows: one-row boxes, four rows per TMA gather4
                if (!pairs || mc)
                    throw Error{PG_INVALID_ARGUMENT, "umma: gathered B rows need the CTA-pair kernel (M >= 256)"};
                P->maps[2 * g + 1] = make_map(s.b, s.b_idx_rows, s.K, s.ldb, 1);
            } else {
                P->maps[2 * g + 1] = make_map(s.b, s.b_rows > 0 ? std::min(s.b_rows, s.N) : s.N, s.K, s.ldb,
                                              mc ? G.bn / 4 : (pairs ? G.bn / 2 : G.bn));
            }
            G.b_idx = s.b_idx;
            if (s.b_idx) P->gather = 1;
            G.b_idx_n = s.b_idx_n;
            G.b_idx_rows = s.b_idx_rows;
            static const int hints_env = [] {
                const char* e = getenv("PG_UMMA_L2HINT");
                return e ? atoi(e) : 1;
            }();
            G.a_hint = hints_env ? s.a_hint : 0;
            G.b_hint = hints_env ? s.b_hint : 0;
            G.direct_epi = s.direct_epi;
            G.mask = s.mask;
            G.mask_ld = s.mask_ld;
            G.row_pat = s.row_pat;
            if (pairs) P->omaps[g] = make_out_map(s.out, s.M, s.N, s.ldo, s.out_bf16 != 0);
            G.out = s.out;
            G.ldo = s.ldo;
            G.M = s.M;
            G.N = s.N;
            G.K = s.K;
            G.out_bf16 = s.out_bf16;
            G.tiles_m = (s.M + (mc ? 4 * UM_BM : (pairs ? 2 * UM_BM : UM_BM)) - 1) / (mc ? 4 * UM_BM : (pairs ? 2 * UM_BM : UM_BM));
            G.tiles_n = (s.N + G.bn - 1) / G.bn;
            G.tile_base = tiles;
            tiles += G.tiles_m * G.tiles_n;
        }
        P->ngroups = ng;
        P->total_tiles = tiles;
        static const int epi_env = [] {
            const char* e = getenv("PG_UMMA_EPI_DEEP");
            return e ? atoi(e) : 1;
        }();
        P->epi_deep = epi_env;
        if (tiles == 0) continue;
        if (mc) {
            static int max_cl = [&] {
                cudaLaunchConfig_t q = {};
                q.gridDim = dim3((unsigned)(sms / 4 * 4));
                q.blockDim = dim3(UM_THREADS);
                q.dynamicSmemBytes = U2_SMEM;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeClusterDimension;
                a[0].val.clusterDim.x = 4;
                a[0].val.clusterDim.y = 1;
                a[0].val.clusterDim.z = 1;
                q.attrs = a;
                q.numAttrs = 1;
                int n = 0;
                if (cudaOccupancyMaxActiveClusters(&n, k_umma_grouped4, &q) != cudaSuccess || n <= 0) n = sms / 4;
                if (getenv("PG_UMMA_DEBUG")) fprintf(stderr, "umma4: max active clusters %d\n", n);
                return n;
            }();
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(4 * std::min(tiles, max_cl)));
            cfg.blockDim = dim3(UM_THREADS);
            cfg.dynamicSmemBytes = U2_SMEM;
            cfg.stream = st;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 4;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[1].val.programmaticStreamSerializationAllowed = umma_pdl();
            cfg.attrs = at;
            cfg.numAttrs = 2;
            PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_umma_grouped4, *P));
            count_launch();
        } else if (pairs) {
            // persistent: only as many pairs as can be co-resident (cluster
            // placement needs both SMs of a TPC free)
            static int max_pairs = [&] {
                cudaLaunchConfig_t q = {};
                q.gridDim = dim3((unsigned)(sms / 2 * 2));
                q.blockDim = dim3(P2_THREADS);
                q.dynamicSmemBytes = P2_SMEM;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeClusterDimension;
                a[0].val.clusterDim.x = 2;
                a[0].val.clusterDim.y = 1;
                a[0].val.clusterDim.z = 1;
                q.attrs = a;
                q.numAttrs = 1;
                int n = 0;
                if (cudaOccupancyMaxActiveClusters(&n, k_umma_grouped2<false>, &q) != cudaSuccess || n <= 0) n = sms / 2;
                if (getenv("PG_UMMA_DEBUG")) fprintf(stderr, "umma2: max active clusters %d (sms %d)\n", n, sms);
                return n;
            }();
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(2 * std::min(tiles, max_pairs)));
            cfg.blockDim = dim3(P2_THREADS);
            cfg.dynamicSmemBytes = P2_SMEM;
            cfg.stream = st;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[1].val.programmaticStreamSerializationAllowed = umma_pdl();
            cfg.attrs = at;
            cfg.numAttrs = 2;
            if (P->gather) PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_umma_grouped2<true>, *P));
            else PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_umma_grouped2<false>, *P));
            count_launch();
        } else {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)std::min(tiles, sms));
            cfg.blockDim = dim3(UM_THREADS);
            cfg.dynamicSmemBytes = UM_SMEM;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = umma_pdl();
            cfg.attrs = at;
            cfg.numAttrs = 1;
            PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_umma_grouped, *P));
            count_launch();
        }
    }
}

// ---------------------------------------------------------------- split-K
__global__ void k_splitk_reduce(const float* __restrict__ part, int S, int M, int N, const uint8_t* __restrict__ mask,
                                long long mask_ld, const int32_t* __restrict__ row_pat, void* out, long long ldo,
                                int out_bf16) {
    const long long slice = (long long)M * N, n4 = slice / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const long long e = 4 * i;
        const int row = (int)(e / N), col = (int)(e % N);
        float4 a = __ldcs(reinterpret_cast<const float4*>(part + e));
        for (int q = 1; q < S; ++q) {  // slice order: deterministic
            const float4 b = __ldcs(reinterpret_cast<const float4*>(part + q * slice + e));
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        if (mask) {
            const uint32_t mw = *reinterpret_cast<const uint32_t*>(mask + (long long)row_pat[row] * mask_ld + col);
            if (!(mw & 0xFFu)) a.x = 0.f;
            if (!(mw & 0xFF00u)) a.y = 0.f;
            if (!(mw & 0xFF0000u)) a.z = 0.f;
            if (!(mw & 0xFF000000u)) a.w = 0.f;
        }
        if (out_bf16) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
            uint2 w;
            w.x = *reinterpret_cast<uint32_t*>(&lo);
            w.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + row * ldo + col) = w;
        } else {
            *reinterpret_cast<float4*>(static_cast<float*>(out) + row * ldo + col) = a;
        }
    }
}

// S K-slices and the tile width: wide tiles (each A row block read by few N
// tiles), K split until the slices cover the SMs.  1 = do not split.
static int splitk_plan(const UmmaSpec& s, int* bn_out, int* kslice_out) {
    static const int env_max = [] {
        const char* e = getenv("PG_UMMA_SPLITK");  // max K slices (1 disables)
        return e ? std::max(1, atoi(e)) : UM_MAX_GROUPS;
    }();
    const int sms = device_sms();
    const bool pairs = umma_pairs_enabled() != 0 && s.M >= 2 * UM_BM;
    const int rows = pairs ? 2 * UM_BM : UM_BM, slots = pairs ? sms / 2 : sms;
    int bn = pick_bn(s.N);
    if (pairs) bn = std::min(UM_BN_MAX, (bn + 31) / 32 * 32);
    const long tiles = (long)((s.M + rows - 1) / rows) * ((s.N + bn - 1) / bn);
    static const int kmin = [] {  // measured: only the long-K GEMMs gain (down's stage 1, K = 11008)
        const char* e = getenv("PG_UMMA_SPLITK_KMIN");
        return e ? atoi(e) : 8192;
    }();
    if (s.N % 4 || s.ldo % 4 || tiles * 2 > (long)slots || s.K < kmin) return 1;
    int S = (int)(slots / tiles);
    S = std::min(S, std::max(1, s.K / 512));  // >= 8 k-blocks per slice
    S = std::min(S, std::min(UM_MAX_GROUPS, env_max));
    if (S <= 1) return 1;
    const int ks = (s.K + S - 1) / S;
    const int kslice = (ks + UM_BK - 1) / UM_BK * UM_BK;
    *bn_out = bn;
    *kslice_out = kslice;
    return (s.K + kslice - 1) / kslice;
}

size_t umma_splitk_bytes(const UmmaSpec& s) {
    int bn = 0, ks = 0;
    const int S = splitk_plan(s, &bn, &ks);
    return S > 1 ? (size_t)S * s.M * s.N * 4 : 0;
}

bool launch_umma_splitk(const UmmaSpec& s, void* ws, cudaStream_t st) {
    return launch_umma_splitk_multi({s}, ws, st);
}

bool launch_umma_splitk_multi(const std::vector<UmmaSpec>& specs, void* ws, cudaStream_t st) {
    std::vector<int> Ss, bns, kss;
    for (const UmmaSpec& s : specs) {
        int bn = 0, ks = 0;
        const int S = splitk_plan(s, &bn, &ks);
        if (S <= 1) return false;  // all or nothing: one grouped launch of every slice
        Ss.push_back(S);
        bns.push_back(bn);
        kss.push_back(ks);
    }
    if (ws == nullptr) return false;
    std::vector<UmmaSpec> parts;
    std::vector<float*> pws;
    float* w = static_cast<float*>(ws);
    for (size_t j = 0; j < specs.size(); ++j) {
        const UmmaSpec& s = specs[j];
        pws.push_back(w);
        for (int q = 0; q < Ss[j]; ++q) {
            const int k0 = q * kss[j];
            UmmaSpec p = s;
            p.a = static_cast<const __nv_bfloat16*>(s.a) + k0;
            p.b = static_cast<const __nv_bfloat16*>(s.b) + k0;
            p.K = std::min(kss[j], s.K - k0);
            p.out = w + (size_t)q * s.M * s.N;
            p.ldo = s.N;
            p.out_bf16 = 0;
            p.mask = nullptr;
            p.row_pat = nullptr;
            p.bn = bns[j];
            p.direct_epi = 1;
            parts.push_back(p);
        }
        w += (size_t)Ss[j] * s.M * s.N;
    }
    launch_umma(parts, st);
    const int sms = device_sms();
    for (size_t j = 0; j < specs.size(); ++j) {
        const UmmaSpec& s = specs[j];
        const long long n4 = (long long)s.M * s.N / 4;
        const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)sms * 8);
        k_splitk_reduce<<<blocks, 256, 0, st>>>(pws[j], Ss[j], s.M, s.N, s.mask, s.mask_ld, s.row_pat, s.out, s.ldo,
                                                s.out_bf16);
        PG_LAUNCH_CHECK();
    }
    return true;
}

}  // namespace pg
