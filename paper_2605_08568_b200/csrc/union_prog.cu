// union_prog.cu -- K5e: a whole heterogeneous decode step (BASELINE config 4:
// every linear of every layer, T <= 256 tokens from T prompts, each with its
// own expert subset per linear) as ONE persistent tcgen05 launch.
//
// A "program" is the sequence of GEMM phases of the step: per module (linears
// sharing an input: q/k/v, o, up/gate, down) stage 1 Z = mask(X . B^T) and
// stage 2 Y = Z . A^T (rank_experts.hpp:52-72 for every token, the union of
// the selections read once: union_wm.cu).  Each phase is cut exactly like a
// k_union_wm launch (CTA pair = 256 weight rows x all tokens; whole tiles
// round-robin, the remainder tiles K-split one piece per pair), but the
// phases are not separated by kernel boundaries: they are chained by data.
//
//   * ready counters, one per (phase, tile, 128-row half): the epilogue that
//     completes rows [h*128, h*128+128) of a phase's output for every token
//     adds 1 (release); a k-block of a later phase that reads those rows as
//     its X columns waits (acquire) until the counter reaches launch_tag x
//     the writers per launch (host table), then reads them with TMA;
//   * the weight tiles never depend on activations: a dedicated producer
//     warp streams them into the ring as soon as a slot is free, across
//     phase and layer boundaries, while the token producer waits for data;
//   * split tiles publish f32 partials (bulk stores from shared-memory
//     staging, tagged flags per phase) and their participants reduce one token
//     slice each, in pair order (deterministic); the partial buffers alternate
//     between two sets by phase parity and a writer waits until every reader of
//     the slot's previous use has counted itself out (consumed counters);
//   * the schedule (which pieces a pair runs, in order) is computed on the host
//     into one 128-byte record per piece, so no role walks phase metadata with
//     dependent global loads on the critical path.
// Everything waits only on earlier phases or on its own pipeline, and every
// CTA of the grid is co-resident (one CTA pair per TPC, grid = the occupancy
// bound), so the dataflow cannot deadlock.
//
// Warp roles (224 threads, one CTA per SM):
//   warp 0     weight producer (both CTAs; runs ahead of everything);
//   warp 1     TMEM allocator; leader CTA lane 0 issues tcgen05.mma.cta_group::2;
//   warp 2     token producer (both CTAs; waits on the ready counters);
//   warps 3-6  epilogue (TMEM -> mask -> bf16/f32 store, partials, reductions).
// Roofline: HBM, the stored experts of every linear read once per step
// (sum r_store (m + n) * 2 bytes); tensor 2 * T * r_store * (m + n) per linear.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <mutex>
#include <vector>

#include "umma.cuh"
#include "union_dev.cuh"
#include "union_prog.cuh"

namespace pg {

#ifndef UP_STAGES_CFG
#define UP_STAGES_CFG 6
#endif
constexpr int UP_STAGES = UP_STAGES_CFG;
constexpr int UP_STAGE_BYTES = WM_W_BYTES + WM_X_BYTES;  // 32 KB
#ifndef UP_EPI_WARPS_CFG
#define UP_EPI_WARPS_CFG 4
#endif
constexpr int UP_EPI_WARPS = UP_EPI_WARPS_CFG;  // 4 or 8: 1 or 2 warps per TMEM lane quadrant
constexpr int UP_EPI_T = 32 * UP_EPI_WARPS;
constexpr int UP_EPI_H = UP_EPI_WARPS / 4;      // epilogue halves (chunk interleave)
constexpr int UP_THREADS = 96 + UP_EPI_T;
constexpr int UP_MAXG = 4;
#ifndef UP_POLL_NS_CFG
#define UP_POLL_NS_CFG 100
#endif
constexpr int UP_POLL_NS = UP_POLL_NS_CFG;  // back-off between polls of a dependency counter
constexpr int UP_CSTRIDE = 32;   // ready counters one per 128-byte line
#ifndef UP_DRAIN_DIRECT
#define UP_DRAIN_DIRECT 0
#endif
#ifndef UP_RED_UNROLL_CFG
#define UP_RED_UNROLL_CFG 3
#endif
constexpr int UP_RED_UNROLL = UP_RED_UNROLL_CFG;  // LSU reduction: participants' loads in flight per batch
#ifndef UP_STG_BUFS_CFG
#define UP_STG_BUFS_CFG 2
#endif
constexpr int UP_STG_BUFS = UP_STG_BUFS_CFG;  // partial-drain bulk stores in flight (2 or 4)
constexpr int UP_STG_BYTES = UP_STG_BUFS * 32 * WM_BM * 4;  // epilogue staging: [32 tokens][128 rows] f32 buffers
static_assert(UP_STG_BYTES >= UP_EPI_WARPS * WM_STG_BYTES, "whole-tile staging must fit");
// [align slack][ring][barriers + slots, 1 KB][token -> pattern table, 1 KB][epilogue staging]
constexpr int UP_SMEM = 1024 + UP_STAGES * UP_STAGE_BYTES + 1024 + WM_TMAX * 4 + UP_STG_BYTES;

struct __align__(64) UpGroup {
    CUtensorMap wmap;  // weights [R, K], box {64, 128}
    CUtensorMap xmap;  // tokens [T, K], box {64, Tp / 2}
};

// one piece of one pair's work, in processing order (host-built)
struct __align__(128) UpRec {
    void* out;            // [T, ldo] token-major
    const uint8_t* mask;  // stage 1 selection mask [P, mask_ld] (or null)
    int ldo, mask_ld, Rs, out_bf16;
    int phase, g, row0;   // g: group (tensor maps); row0: first weight row of the pair's tile
    int k0, k1;           // k-block range
    int split, pf, n;     // split piece: participants [pf, pf + n)
    int src_ready;        // X k-block kb waits on ready[src_ready + kb / 2]; -1: external input
    int ready_idx;        // the tile's ready counter (rank 0 half; + rank)
    int flag_base;        // the phase's partial flags [pairs][2]
    int last_in_phase;    // last piece of this pair in its phase
    int tok_off;          // the GEMM's tokens in the launch's pattern table
    int w_hint;           // weight loads: 1 evict-first, 0 evict-normal (read again soon by another chain)
};

struct UpParams {
    const UpGroup* groups;
    const UpRec* recs;
    const int* pair_off;       // [pairs + 1] record ranges
    const unsigned* pair_tot;  // [pairs][2] partial-slot reads per launch, per parity set
    int T, Tp;
    int Ttab;                  // token -> pattern table entries (max tok_off + T over the GEMMs)
    const int32_t* tok_pat;
    unsigned* ready;
    const uint8_t* ready_exp;  // writers per launch of each ready counter
    unsigned* flags;
    unsigned* consumed;        // [2][pairs][2]
    float* partial;            // [2][pairs][2][WM_PART_FLOATS]
    unsigned long long* epoch;
    unsigned long long* dbg;
    int exp;  // PG_PROG_EXP (timing experiments only, wrong results): 1 no reduction loads, 2 no partial drain,
              // 4 no whole-tile stores, 8 half the tokens drained and reduced
};

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// poll with a short back-off: every CTA of a phase waits on the same few
// counters, and tight loads from 148 SMs would hammer their L2 lines.  The
// polls are relaxed (an acquire load invalidates the SM's L1 each time); one
// acquire load of the (monotonic) counter after the target is seen orders the
// caller's later reads.
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
    while ((int)(ld_relaxed(p) - target) < 0) __nanosleep(UP_POLL_NS);
    (void)ld_acquire(p);
}
__device__ __forceinline__ void up_bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(UP_EPI_T) : "memory"); }
__device__ __forceinline__ void up_bar_half(int h) { asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory"); }
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// PG_PROG_DBG=1: %globaltimer stamps [grid][64] for phases f < 8: [0] start,
// epilogue [1+f] first piece drained, [9+f] all pieces drained, [17+f] split
// partial flags seen, [25+f] phase done; X producer [33+f] first / [41+f] last
// X issued; W producer [49+f] first W issued
#define UP_STAMP(k)                                                       \
    do {                                                                  \
        if (P.dbg) P.dbg[blockIdx.x * 64 + (k)] = wm_gtimer();            \
    } while (0)

// split tile: TMEM -> [32 tokens][128 rows] f32 chunk in shared memory (4
// epilogue warps, one per TMEM lane quadrant, 16 KB) -> one 16 KB bulk store
// per chunk into the partial [Tp][128].  With 8 epilogue warps the two halves
// take alternate chunks, each with its own staging buffer and named barrier;
// with 4, one half double-buffers.  The stores are complete (and ordered
// before the caller's release) on return.
__device__ __forceinline__ void up_epi_partial_bulk(int Tp, uint32_t taddr, float* dst, int q, int h, float* buf,
                                                    int lane, int et) {
    const int nch = Tp / 32;
#if UP_DRAIN_DIRECT
    // direct: lane = row, one 4-byte store per token -> each warp store is one
    // full 128-byte line of the token-major partial; no staging, no bulk group
    if (h == 0) {
        uint32_t ra[32];
        for (int c = 0; c < nch; ++c) {
            tmem_ld32(taddr + 32u * c, ra);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcg(dst + (size_t)(c * 32 + j) * WM_BM + q * 32 + lane, __uint_as_float(ra[j]));
        }
    }
    return;
#endif
    const bool lead = (et & 127) == 0;
    uint32_t ra[32];
    for (int c = h; c < nch; c += UP_EPI_H) {
        const int bi = UP_EPI_H == 2 ? h : (c % UP_STG_BUFS);
        float* b = buf + bi * (32 * WM_BM);
        if (lead && c >= (UP_EPI_H == 2 ? 2 : UP_STG_BUFS)) {
            if (UP_EPI_H == 2) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else if (UP_STG_BUFS == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        up_bar_half(h);  // this half's buffer is free
        tmem_ld32(taddr + 32u * c, ra);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) b[j * WM_BM + q * 32 + lane] = __uint_as_float(ra[j]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        up_bar_half(h);  // chunk written
        if (lead) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (size_t)c * 32 * WM_BM),
                         "r"(u_smem(b)), "r"(32 * WM_BM * 4)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lead) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
}

constexpr int UP_RED_E = 32 * 32 / UP_EPI_T;  // float4s of a 32-token chunk per epilogue thread

struct F4xE {
    float4 v[UP_RED_E];
};

struct UpOut {  // epilogue view of a record (wm_epi_direct / wm_put)
    void* out;
    long long ldo;
    int out_bf16;
    const uint8_t* mask;
    long long mask_ld;
    int Rs;
};

__global__ void __launch_bounds__(UP_THREADS, 1) k_union_prog(const __grid_constant__ UpParams P) {
    extern __shared__ __align__(1024) unsigned char usmem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(usmem) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + UP_STAGES * UP_STAGE_BYTES);
    uint64_t* full = bars;                        // [STAGES] (leader's copy used; 2 arrivals: W and X producers)
    uint64_t* empty = bars + UP_STAGES;           // [STAGES] (each CTA)
    uint64_t* tfull = bars + 2 * UP_STAGES;       // [2] (each CTA)
    uint64_t* tempty = bars + 2 * UP_STAGES + 2;  // [2] (leader's copy: both CTAs' epilogues)
    uint32_t* slots = reinterpret_cast<uint32_t*>(bars + 2 * UP_STAGES + 4);  // [0] tmem base, [1] launch tag
    int32_t* tps = reinterpret_cast<int32_t*>(base + UP_STAGES * UP_STAGE_BYTES + 1024);
    unsigned char* stage = base + UP_STAGES * UP_STAGE_BYTES + 1024 + WM_TMAX * 4;  // epilogue staging

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, np = gridDim.x >> 1;
    const int r0 = P.pair_off[pair], r1 = P.pair_off[pair + 1];
    if (threadIdx.x == 0) {
        UP_STAMP(0);
        for (int s = 0; s < UP_STAGES; ++s) {
            u_mbar_init(u_smem(&full[s]), 2);
            u_mbar_init(u_smem(&empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            u_mbar_init(u_smem(&tfull[a]), 1);
            u_mbar_init(u_smem(&tempty[a]), 2 * UP_EPI_WARPS);  // epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // launch ticket before launch_dependents: every CTA of this launch holds
        // its ticket before a CTA of the next launch can start (old / grid = index)
        const unsigned long long old = atomicAdd(P.epoch, 1ull);
        slots[1] = (uint32_t)(old / gridDim.x) + 1u;
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(u_smem(slots)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slots[0];
    const uint32_t tag = slots[1];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ------------------------------------------------ weight producer (both CTAs)
        if (lane == 0) {
            uint64_t pfirst, pnorm;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pfirst));
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pnorm));
            int s = 0, issued = 0, lastf = -1;
            uint32_t ph = 0;
            for (int i = r0; i < r1; ++i) {
                const UpRec& R = P.recs[i];
                if (i + 1 < r1) prefetch_l1(&P.recs[i + 1]);
                const CUtensorMap* wm = &P.groups[R.g].wmap;
                const int row = R.row0 + (int)rank * WM_BM, k1 = R.k1, f = R.phase;
                for (int kb = R.k0; kb < k1; ++kb, ++issued) {
                    if (issued >= UP_STAGES) u_mbar_wait(u_smem(&empty[s]), ph ^ 1);
                    const uint32_t fb = leader_addr(u_smem(&full[s]));
                    if (leader) u_mbar_arrive_tx_cluster(fb, 2u * WM_W_BYTES);
                    u_tma_2d_pair_h(u_smem(base + s * UP_STAGE_BYTES), wm, kb * WM_BK, row, fb, R.w_hint ? pfirst : pnorm);
                    if (f != lastf && f < 8) UP_STAMP(49 + f);
                    lastf = f;
                    if (++s == UP_STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ token producer (both CTAs)
        if (lane == 0) {
            uint64_t plast;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(plast));
            const uint32_t xbytes = (uint32_t)(P.Tp / 2) * WM_BK * 2;
            const int xrow = (int)rank * (P.Tp / 2);
            asm volatile("griddepcontrol.wait;" ::: "memory");  // external inputs: the previous kernel's outputs
            int s = 0, issued = 0, seen = -1, lastf = -1;
            uint32_t ph = 0;
            for (int i = r0; i < r1; ++i) {
                const UpRec& R = P.recs[i];
                if (i + 1 < r1) prefetch_l1(&P.recs[i + 1]);
                const CUtensorMap* xm = &P.groups[R.g].xmap;
                const int src = R.src_ready, k1 = R.k1, f = R.phase;
                for (int kb = R.k0; kb < k1; ++kb, ++issued) {
                    if (issued >= UP_STAGES) u_mbar_wait(u_smem(&empty[s]), ph ^ 1);
                    if (src >= 0 && src + kb / 2 != seen) {
                        // X columns [kb*64, kb*64+64) = rows of the producing phase's
                        // output in its 128-row half kb / 2
                        seen = src + kb / 2;
                        wait_count(P.ready + (size_t)seen * UP_CSTRIDE, tag * (unsigned)P.ready_exp[seen]);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    const uint32_t fb = leader_addr(u_smem(&full[s]));
                    if (leader) u_mbar_arrive_tx_cluster(fb, 2u * xbytes);
                    u_tma_2d_pair_h(u_smem(base + s * UP_STAGE_BYTES + WM_W_BYTES), xm, kb * WM_BK, xrow, fb, plast);
                    if (f < 8) {
                        if (f != lastf) UP_STAMP(33 + f);
                        if (R.last_in_phase && kb == k1 - 1) UP_STAMP(41 + f);
                    }
                    lastf = f;
                    if (++s == UP_STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (leader && lane == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P.Tp >> 3) << 17) |
                                   ((uint32_t)((2 * WM_BM) >> 4) << 24);
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int i = r0; i < r1; ++i) {
                const int k0 = P.recs[i].k0, k1 = P.recs[i].k1;
                if (i + 1 < r1) prefetch_l1(&P.recs[i + 1]);
                u_mbar_wait(u_smem(&tempty[acc]), aph ^ 1);  // both CTAs drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(acc * WM_TMAX);
                for (int kb = k0; kb < k1; ++kb) {
                    u_mbar_wait(u_smem(&full[s]), ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = u_smem(base + s * UP_STAGE_BYTES), sb = sa + WM_W_BYTES;
#pragma unroll
                    for (int k = 0; k < WM_BK / 16; ++k)
                        u_mma2(d, u_desc(sa + k * 32), u_desc(sb + k * 32), idesc, (kb > k0 || k > 0) ? 1u : 0u);
                    u_commit2(u_smem(&empty[s]));
                    if (++s == UP_STAGES) { s = 0; ph ^= 1; }
                }
                u_commit2(u_smem(&tfull[acc]));
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 3-6, both CTAs)
        const int et = threadIdx.x - 96;  // 0 .. UP_EPI_T - 1
        const int q = warp & 3, h = (warp - 3) >> 2;  // TMEM lane quadrant; half (chunk interleave)
        float* stg = reinterpret_cast<float*>(stage) + (warp - 3) * (WM_STG_BYTES / 4);
        asm volatile("griddepcontrol.wait;" ::: "memory");  // outputs may still be read by the previous kernel
        for (int t = et; t < P.Ttab; t += UP_EPI_T) tps[t] = P.tok_pat ? __ldg(P.tok_pat + t) : 0;
        // reads of this pair's partial slots per launch, per parity set: a writer
        // waits for all readers of the slot's previous use before reusing it
        const unsigned tot0 = P.pair_tot[pair * 2], tot1 = P.pair_tot[pair * 2 + 1];
        unsigned used0 = 0u, used1 = 0u;  // scalars, not arrays indexed by the phase parity (no stack frame)
        up_bar_epi();
        int acc = 0, pi = 0, lastf = -1;
        uint32_t aph = 0;
        int red_rec = -1;  // this pair's split piece of the current phase
        for (int i = r0; i < r1; ++i) {
            const UpRec& R = P.recs[i];
            if (i + 1 < r1) prefetch_l1(&P.recs[i + 1]);
            const int f = R.phase, set = f & 1;
            pi = (f == lastf) ? pi + 1 : 0;
            lastf = f;
            if (R.split) {
                red_rec = i;
                if (et == 0)  // every reader of this slot's previous use is done
                    wait_count(P.consumed + (set * np + pair) * 2 + rank,
                               (tag - 1u) * (set ? tot1 : tot0) + (set ? used1 : used0));
            }
            u_mbar_wait(u_smem(&tfull[acc]), aph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (et == 0 && f < 7 && pi == 0) UP_STAMP(57 + f);  // accumulator of the phase's first piece ready
            if (R.split) up_bar_epi();  // the slot wait above
            const uint32_t taddr = tmem + (uint32_t)(acc * WM_TMAX) + ((uint32_t)(q * 32) << 16);
            if (P.exp & (R.split ? 2 : 4)) {
            } else if (!R.split) {
                const UpOut G{R.out, R.ldo, R.out_bf16, R.mask, R.mask_ld, R.Rs};
                wm_epi_direct(P.Tp, P.T, G, taddr, R.row0 + (int)rank * WM_BM + q * 32, tps + R.tok_off, stg, lane, h,
                              UP_EPI_H);
            } else {
                up_epi_partial_bulk((P.exp & 8) ? P.Tp / 2 : P.Tp, taddr, P.partial + ((size_t)(set * np + pair) * 2 + rank) * WM_PART_FLOATS, q,
                                    h, reinterpret_cast<float*>(stage), lane, et);
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) u_mbar_arrive_cluster(leader_addr(u_smem(&tempty[acc])));
            up_bar_epi();  // every epilogue thread's stores are issued (and the staging is free)
            if (et == 0) {  // the release is cumulative over the epilogue's stores (bar.sync above)
                if (R.split) {
                    st_release(P.flags + R.flag_base + pair * 2 + (int)rank, tag);
                    if (set) used1 += (unsigned)R.n;
                    else used0 += (unsigned)R.n;
                } else {
                    red_release_add(P.ready + (size_t)(R.ready_idx + (int)rank) * UP_CSTRIDE, 1u);
                }
                if (f < 8) {
                    if (pi == 0) UP_STAMP(1 + f);
                    if (R.last_in_phase) UP_STAMP(9 + f);
                }
            }
            if (++acc == 2) { acc = 0; aph ^= 1; }
            if (!R.last_in_phase) continue;
            if (red_rec >= 0) {
                // ---- this pair's token slice of its split tile: the n partials'
                // slices loaded (LSU, three participants in flight), summed in pair
                // order (deterministic), masked, stored
                const UpRec& S = P.recs[red_rec];
                const int pf = S.pf, n = S.n, me = pair - pf;
                void* const sout = S.out;
                const uint8_t* const smask = S.mask;
                const long long sldo = S.ldo, smask_ld = S.mask_ld;
                const int sRs = S.Rs, sbf16 = S.out_bf16, sflags = S.flag_base, sready = S.ready_idx, stok = S.tok_off;
                const int row0 = S.row0 + (int)rank * WM_BM;
                // token slice of this participant, 4-aligned (float4 along tokens)
                const int ta = me * (P.Tp / 4) / n * 4, tb = min(P.T, (me + 1) * (P.Tp / 4) / n * 4);
                const int cnt = (P.exp & 8) ? max(0, tb - ta) / 2 : max(0, tb - ta);  // (exp 8: half the tail bytes, timing only)
                // the slice's mask bytes (stage-1 outputs) into the idle staging
                // buffer while the participants finish: [cnt tokens][128 rows]
                uint8_t* const msk = stage;
                if (smask) {
                    for (int idx = et; idx < cnt * 8; idx += UP_EPI_T) {
                        const int tl = idx >> 3, part = idx & 7;
                        if (row0 + part * 16 < sRs)
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(u_smem(msk + tl * 128 + part * 16)),
                                         "l"(smask + (long long)tps[stok + ta + tl] * smask_ld + row0 + part * 16)
                                         : "memory");
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                }
                if (warp == 3)  // every participant's flag, one lane each
                    for (int pp = pf + lane; pp < pf + n; pp += 32) {
                        const unsigned* fl = P.flags + sflags + pp * 2 + (int)rank;
                        while (ld_relaxed(fl) != tag) __nanosleep(UP_POLL_NS);
                        (void)ld_acquire(fl);
                    }
                if (smask) asm volatile("cp.async.wait_all;" ::: "memory");
                up_bar_epi();
                if (et == 0 && f < 8) UP_STAMP(17 + f);
                const float* pbase = P.partial + ((size_t)(set * np) * 2 + rank) * WM_PART_FLOATS;
                auto store_chunk = [&](int ch, int ct, const F4xE& a) {
                    // chunk complete: masks first (read-only path, all 8 in flight), then
                    // the stores (plain loads after stores would serialise on aliasing)
                    uint32_t mw[UP_RED_E];
#pragma unroll
                    for (int j = 0; j < UP_RED_E; ++j) {
                        const int e = et + UP_EPI_T * j, tl = e >> 5, c4 = e & 31;
                        mw[j] = 0xFFFFFFFFu;
                        if (smask && tl < ct) mw[j] = *reinterpret_cast<const uint32_t*>(msk + (ch * 32 + tl) * 128 + 4 * c4);
                    }
#pragma unroll
                    for (int j = 0; j < UP_RED_E; ++j) {
                        const int e = et + UP_EPI_T * j, tl = e >> 5, c4 = e & 31;
                        if (tl >= ct) continue;
                        float4 v = a.v[j];
                        const int tok = ta + ch * 32 + tl, row = row0 + 4 * c4;
                        if (!(mw[j] & 0xFFu)) v.x = 0.f;
                        if (!(mw[j] & 0xFF00u)) v.y = 0.f;
                        if (!(mw[j] & 0xFF0000u)) v.z = 0.f;
                        if (!(mw[j] & 0xFF000000u)) v.w = 0.f;
                        if (row + 3 < sRs) {
                            if (sbf16) {
                                __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
                                uint2 w;
                                w.x = *reinterpret_cast<uint32_t*>(&lo);
                                w.y = *reinterpret_cast<uint32_t*>(&hi);
                                *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(sout) + (long long)tok * sldo + row) = w;
                            } else {
                                *reinterpret_cast<float4*>(static_cast<float*>(sout) + (long long)tok * sldo + row) = v;
                            }
                        } else {
                            const UpOut G{sout, sldo, sbf16, nullptr, 0, sRs};
                            if (row < sRs) wm_put(G, tok, row, v.x);
                            if (row + 1 < sRs) wm_put(G, tok, row + 1, v.y);
                            if (row + 2 < sRs) wm_put(G, tok, row + 2, v.z);
                        }
                    }
                };
                {
                    // LSU: per 32-token chunk, UP_RED_E float4 per thread per participant,
                    // three participants' loads in flight at a time, summed in pair order
                    for (int ch = 0; ch * 32 < cnt; ++ch) {
                        const int ct = min(32, cnt - ch * 32);
                        F4xE a;
                        for (int pp = 0; pp < n; pp += UP_RED_UNROLL) {
                            float4 v[UP_RED_UNROLL][UP_RED_E];
                            const float* s0 = pbase + (size_t)(pf + pp) * 2 * WM_PART_FLOATS + (size_t)(ta + ch * 32) * WM_BM;
#pragma unroll
                            for (int u = 0; u < UP_RED_UNROLL; ++u)
#pragma unroll
                                for (int j = 0; j < UP_RED_E; ++j) {
                                    v[u][j] = make_float4(0.f, 0.f, 0.f, 0.f);
                                    const int e = et + UP_EPI_T * j;
                                    if (pp + u < n && (e >> 5) < ct && !(P.exp & 1))
                                        v[u][j] = __ldcg(reinterpret_cast<const float4*>(s0 + (size_t)u * 2 * WM_PART_FLOATS) + e);
                                }
#pragma unroll
                            for (int u = 0; u < UP_RED_UNROLL; ++u)
#pragma unroll
                                for (int j = 0; j < UP_RED_E; ++j) {
                                    if (pp + u >= n) continue;
                                    if (pp + u == 0) a.v[j] = v[u][j];
                                    else { a.v[j].x += v[u][j].x; a.v[j].y += v[u][j].y; a.v[j].z += v[u][j].z; a.v[j].w += v[u][j].w; }
                                }
                        }
                        store_chunk(ch, ct, a);
                    }
                }
                up_bar_epi();  // slice stored
                if (et == 0) {  // cumulative release (bar.sync above)
                    red_release_add(P.ready + (size_t)(sready + (int)rank) * UP_CSTRIDE, 1u);
                }
                if (et < n) red_release_add(P.consumed + (set * np + pf + et) * 2 + rank, 1u);
                red_rec = -1;
            }
            if (et == 0 && f < 8) UP_STAMP(25 + f);
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- host side
namespace {
int up_max_pairs() {  // co-resident CTA pairs (per device); sets the smem attribute first
    static std::atomic<int> cache[128];
    const int dev = current_device();
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v) return v;
    once_per_device(reinterpret_cast<const void*>(&k_union_prog), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_union_prog, cudaFuncAttributeMaxDynamicSharedMemorySize, UP_SMEM));
    });
    const int sms = device_sms();
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3((unsigned)(sms / 2 * 2));
    q.blockDim = dim3(UP_THREADS);
    q.dynamicSmemBytes = UP_SMEM;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 2;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    q.attrs = a;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_union_prog, &q) != cudaSuccess || n <= 0) n = sms / 2;
    n = std::min(n, sms / 2);
    cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

struct HGroup {  // host metadata of one GEMM
    int R, K, kb, tiles, Rs, tile_base;
    void* out;
    long long ldo;
    int out_bf16;
    const uint8_t* mask;
    long long mask_ld;
    int src_ready;
    int tok_off, w_hint;
};
struct HPhase {
    int g0, ng, TT, full, rem, ready_base, flag_base;
};
}  // namespace

// Tensor maps read by TMA from global memory are cached by the TMA unit by
// address; a map written by the host into memory that once held another map
// could be served stale.  Map storage therefore comes from a process-wide bump
// pool that never hands out an address twice (chunks are never freed).
static UpGroup* alloc_maps(size_t n) {
    static std::mutex mu;
    static char* cur = nullptr;
    static size_t left = 0;
    std::lock_guard<std::mutex> lk(mu);
    const size_t bytes = (n * sizeof(UpGroup) + 255) / 256 * 256;
    if (bytes > left) {
        const size_t chunk = std::max<size_t>(bytes, (size_t)4 << 20);
        PG_CUDA_THROW(cudaMalloc(&cur, chunk));
        left = chunk;
    }
    UpGroup* p = reinterpret_cast<UpGroup*>(cur);
    cur += bytes;
    left -= bytes;
    return p;
}

struct UnionProgram::Impl {
    int T = 0, Tp = 0, pairs = 0, ttab = 0;
    int dev = 0;
    std::vector<UpGroup> groups;  // device tensor maps
    std::vector<HGroup> hg;
    std::vector<HPhase> phases;
    std::vector<uint8_t> exp;
    struct Region {
        const char* a;
        const char* b;
    };
    std::vector<std::vector<Region>> reads, writes;  // per phase
    bool finalized = false;
    char* ws = nullptr;  // [epoch 256 B | ready | exp | flags | consumed | pair_off | pair_tot | partials]
    UpParams P{};
    UpGroup* d_groups = nullptr;
    UpRec* d_recs = nullptr;
    unsigned long long* dbg = nullptr;
};

UnionProgram::UnionProgram(int T) : d(new Impl) {
    if (T < 1 || T > WM_TMAX) throw Error{PG_INVALID_ARGUMENT, "union_program: 1 <= T <= 256 tokens"};
    d->T = T;
    d->Tp = (T + 31) / 32 * 32;
    PG_CUDA_THROW(cudaGetDevice(&d->dev));
    d->pairs = up_max_pairs();
}

UnionProgram::~UnionProgram() {
    if (d->ws) cudaFree(d->ws);
    if (d->d_recs) cudaFree(d->d_recs);
    if (d->dbg) cudaFree(d->dbg);
}

static bool overlaps(const char* a0, const char* a1, const char* b0, const char* b1) { return a0 < b1 && b0 < a1; }

void UnionProgram::add_phase(const std::vector<WmSpec>& specs) {
    Impl& I = *d;
    if (I.finalized) throw Error{PG_RUNTIME_ERROR, "union_program: already finalized"};
    if (specs.empty() || (int)specs.size() > UP_MAXG) throw Error{PG_INVALID_ARGUMENT, "union_program: 1..4 GEMMs per phase"};
    HPhase ph{};
    ph.g0 = (int)I.hg.size();
    ph.ng = (int)specs.size();
    int TT = 0;
    std::vector<Impl::Region> rd, wr;
    std::vector<HGroup> gs;
    std::vector<UpGroup> maps;
    for (const WmSpec& s : specs) {
        if (s.R < 1 || s.K < 1 || (s.ldw * 2) % 16 || (s.ldx * 2) % 16 || s.ldo % 4 || s.ldx < s.K)
            throw Error{PG_INVALID_ARGUMENT, "union_program: bad GEMM shape / alignment"};
        if (reinterpret_cast<uintptr_t>(s.out) % 16 || (s.out_bf16 && s.ldo % 8) || (s.mask && s.mask_ld % 16) ||
            s.ldo > (1LL << 30) || s.mask_ld > (1LL << 30))
            throw Error{PG_INVALID_ARGUMENT, "union_program: bad output / mask alignment"};
        HGroup G{};
        G.R = s.R;
        G.K = s.K;
        G.kb = (s.K + WM_BK - 1) / WM_BK;
        G.tiles = (s.R + 2 * WM_BM - 1) / (2 * WM_BM);
        G.Rs = (int)std::min<long long>(s.ldo, (long long)G.tiles * 2 * WM_BM);
        G.tile_base = TT;
        TT += G.tiles;
        G.out = s.out;
        G.ldo = s.ldo;
        G.out_bf16 = s.out_bf16;
        G.mask = s.mask;
        G.mask_ld = s.mask_ld;
        if (s.tok_off < 0 || s.tok_off + I.T > WM_TMAX)
            throw Error{PG_INVALID_ARGUMENT, "union_program: token offset + T exceeds the 256-entry pattern table"};
        G.tok_off = s.tok_off;
        G.w_hint = s.w_hint;
        I.ttab = std::max(I.ttab, s.tok_off + I.T);
        UpGroup M{};
        M.wmap = make_map(s.w, s.R, s.K, s.ldw, WM_BM);
        M.xmap = make_map(s.x, I.T, s.K, s.ldx, I.Tp / 2);
        // X source: the latest earlier phase whose output is exactly this buffer
        G.src_ready = -1;
        for (int f = (int)I.phases.size() - 1; f >= 0 && G.src_ready < 0; --f)
            for (int g = 0; g < I.phases[f].ng; ++g) {
                const HGroup& S = I.hg[I.phases[f].g0 + g];
                if (S.out == s.x) {
                    if (S.ldo != s.ldx || !S.out_bf16 || S.Rs < s.K)
                        throw Error{PG_INVALID_ARGUMENT, "union_program: input is a mismatched earlier output"};
                    G.src_ready = I.phases[f].ready_base + 2 * S.tile_base;
                    break;
                }
            }
        const size_t esz = s.out_bf16 ? 2 : 4;
        const char* xo = static_cast<const char*>(s.x);
        rd.push_back({xo, xo + ((size_t)(I.T - 1) * s.ldx + s.K) * 2});
        const char* oo = static_cast<const char*>(s.out);
        wr.push_back({oo, oo + ((size_t)(I.T - 1) * s.ldo + G.Rs) * esz});
        gs.push_back(G);
        maps.push_back(M);
    }
    // a buffer is written once per program and never written after it is read
    // (the dataflow orders reads after writes, not writes after reads)
    for (const auto& w : wr) {
        for (size_t f = 0; f < I.phases.size(); ++f) {
            for (const auto& r : I.reads[f])
                if (overlaps(w.a, w.b, r.a, r.b))
                    throw Error{PG_INVALID_ARGUMENT, "union_program: an output overwrites an earlier phase's input"};
            for (const auto& r : I.writes[f])
                if (overlaps(w.a, w.b, r.a, r.b))
                    throw Error{PG_INVALID_ARGUMENT, "union_program: an output overwrites an earlier phase's output"};
        }
        for (const auto& r : rd)
            if (overlaps(w.a, w.b, r.a, r.b)) throw Error{PG_INVALID_ARGUMENT, "union_program: a phase writes its own input"};
    }
    for (size_t i = 0; i < wr.size(); ++i)
        for (size_t j = i + 1; j < wr.size(); ++j)
            if (overlaps(wr[i].a, wr[i].b, wr[j].a, wr[j].b))
                throw Error{PG_INVALID_ARGUMENT, "union_program: outputs of one phase overlap"};
    ph.TT = TT;
    ph.full = TT / I.pairs;
    ph.rem = TT % I.pairs;
    static const int split_env = [] {  // experiments: 0 = whole tiles only (no K split)
        const char* e = getenv("PG_PROG_SPLIT");
        return e ? atoi(e) : 1;
    }();
    if (!split_env && ph.rem > 0) {
        ph.full = (TT + I.pairs - 1) / I.pairs;  // the last round leaves pairs idle
        ph.rem = 0;
    }
    ph.ready_base = (int)I.exp.size();
    ph.flag_base = (int)I.phases.size() * I.pairs * 2;
    I.hg.insert(I.hg.end(), gs.begin(), gs.end());
    I.groups.insert(I.groups.end(), maps.begin(), maps.end());
    // writers per launch of each (tile, half): 1 for a whole tile, n for a split tile
    I.exp.resize(I.exp.size() + 2 * (size_t)TT, 1);
    for (int r = 0; r < ph.rem; ++r) {
        const int np = I.pairs, pf = r * np / ph.rem, nr = (r + 1) * np / ph.rem - pf;
        const int Ti = ph.full * np + r;
        int g = ph.g0;
        while (g + 1 < ph.g0 + ph.ng && I.hg[g + 1].tile_base <= Ti) ++g;
        const int n = std::min(nr, I.hg[g].kb);
        I.exp[ph.ready_base + 2 * Ti] = I.exp[ph.ready_base + 2 * Ti + 1] = (uint8_t)n;
    }
    I.phases.push_back(ph);
    I.reads.push_back(rd);
    I.writes.push_back(wr);
}

void UnionProgram::finalize(cudaStream_t st) {
    Impl& I = *d;
    if (I.finalized) return;
    if (I.phases.empty()) throw Error{PG_INVALID_ARGUMENT, "union_program: no phases"};
    const int np = I.pairs;
    // ---- per-pair piece records: per phase, the pair's remainder piece first
    // (its partial is published early), then its whole tiles (tile p + i * np)
    std::vector<UpRec> recs;
    std::vector<int> off(np + 1, 0);
    std::vector<unsigned> tot((size_t)np * 2, 0u);
    auto tile_of = [&](const HPhase& ph, int Ti, int& g, int& t) {
        g = ph.g0;
        while (g + 1 < ph.g0 + ph.ng && I.hg[g + 1].tile_base <= Ti) ++g;
        t = Ti - I.hg[g].tile_base;
    };
    auto make = [&](int f, int g, int t, int k0, int k1) {
        const HGroup& G = I.hg[g];
        const HPhase& ph = I.phases[f];
        UpRec R{};
        R.out = G.out;
        R.mask = G.mask;
        R.ldo = (int)G.ldo;
        R.mask_ld = (int)G.mask_ld;
        R.Rs = G.Rs;
        R.out_bf16 = G.out_bf16;
        R.phase = f;
        R.g = g;
        R.row0 = t * 2 * WM_BM;
        R.k0 = k0;
        R.k1 = k1;
        R.src_ready = G.src_ready;
        R.ready_idx = ph.ready_base + 2 * (G.tile_base + t);
        R.flag_base = ph.flag_base;
        R.tok_off = G.tok_off;
        R.w_hint = G.w_hint;
        return R;
    };
    for (int pair = 0; pair < np; ++pair) {
        off[pair] = (int)recs.size();
        for (int f = 0; f < (int)I.phases.size(); ++f) {
            const HPhase& ph = I.phases[f];
            const size_t first = recs.size();
            if (ph.rem > 0) {
                int r = (int)((long long)pair * ph.rem / np);
                while (r + 1 < ph.rem && (r + 1) * np / ph.rem <= pair) ++r;
                while (r > 0 && r * np / ph.rem > pair) --r;
                const int pf = r * np / ph.rem, nr = (r + 1) * np / ph.rem - pf, j = pair - pf;
                int g, t;
                tile_of(ph, ph.full * np + r, g, t);
                const int kb = I.hg[g].kb, n = std::min(nr, kb);
                if (j < n) {
                    UpRec R = make(f, g, t, j * kb / n, (j + 1) * kb / n);
                    R.split = n > 1;
                    R.pf = pf;
                    R.n = n;
                    if (R.split) tot[(size_t)pair * 2 + (f & 1)] += (unsigned)n;
                    recs.push_back(R);
                }
            }
            for (int i = 0; i < ph.full; ++i) {
                if (i * np + pair >= ph.TT) break;  // whole-tile phases: the last round is partial
                int g, t;
                tile_of(ph, i * np + pair, g, t);
                recs.push_back(make(f, g, t, 0, I.hg[g].kb));
            }
            if (recs.size() > first) recs.back().last_in_phase = 1;
        }
    }
    off[np] = (int)recs.size();
    if (recs.empty()) throw Error{PG_INVALID_ARGUMENT, "union_program: no work"};

    const size_t nready = I.exp.size();
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t o_ready = 256, o_exp = o_ready + up(nready * 4 * UP_CSTRIDE), o_flags = o_exp + up(nready);
    const size_t nflags = I.phases.size() * np * 2;
    const size_t o_cons = o_flags + up(nflags * 4), o_off = o_cons + up((size_t)2 * np * 2 * 4);
    const size_t o_tot = o_off + up((size_t)(np + 1) * 4), o_part = o_tot + up((size_t)np * 2 * 4);
    const size_t bytes = o_part + (size_t)2 * np * 2 * WM_PART_FLOATS * 4;
    PG_CUDA_THROW(cudaMalloc(&I.ws, bytes));
    PG_CUDA_THROW(cudaMemsetAsync(I.ws, 0, o_off, st));
    PG_CUDA_THROW(cudaMemcpyAsync(I.ws + o_exp, I.exp.data(), nready, cudaMemcpyHostToDevice, st));
    PG_CUDA_THROW(cudaMemcpyAsync(I.ws + o_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st));
    PG_CUDA_THROW(cudaMemcpyAsync(I.ws + o_tot, tot.data(), tot.size() * 4, cudaMemcpyHostToDevice, st));
    I.d_groups = alloc_maps(I.groups.size());
    PG_CUDA_THROW(cudaMalloc(&I.d_recs, recs.size() * sizeof(UpRec)));
    PG_CUDA_THROW(cudaMemcpyAsync(I.d_groups, I.groups.data(), I.groups.size() * sizeof(UpGroup),
                                  cudaMemcpyHostToDevice, st));
    PG_CUDA_THROW(cudaMemcpyAsync(I.d_recs, recs.data(), recs.size() * sizeof(UpRec), cudaMemcpyHostToDevice, st));
    PG_CUDA_THROW(cudaStreamSynchronize(st));
    const char* e = getenv("PG_PROG_DBG");
    if (e && atoi(e)) {
        PG_CUDA_THROW(cudaMalloc(&I.dbg, (size_t)2 * np * 64 * 8));
        PG_CUDA_THROW(cudaMemset(I.dbg, 0, (size_t)2 * np * 64 * 8));
    }
    UpParams& P = I.P;
    const char* ex = getenv("PG_PROG_EXP");
    P.exp = ex ? atoi(ex) : 0;
    P.groups = I.d_groups;
    P.recs = I.d_recs;
    P.pair_off = reinterpret_cast<const int*>(I.ws + o_off);
    P.pair_tot = reinterpret_cast<const unsigned*>(I.ws + o_tot);
    P.T = I.T;
    P.Tp = I.Tp;
    P.Ttab = I.ttab;
    P.epoch = reinterpret_cast<unsigned long long*>(I.ws);
    P.ready = reinterpret_cast<unsigned*>(I.ws + o_ready);
    P.ready_exp = reinterpret_cast<const uint8_t*>(I.ws + o_exp);
    P.flags = reinterpret_cast<unsigned*>(I.ws + o_flags);
    P.consumed = reinterpret_cast<unsigned*>(I.ws + o_cons);
    P.partial = reinterpret_cast<float*>(I.ws + o_part);
    P.dbg = I.dbg;
    I.finalized = true;
}

void UnionProgram::run(const int32_t* tok_pat, cudaStream_t st) {
    Impl& I = *d;
    int dev = 0;
    PG_CUDA_THROW(cudaGetDevice(&dev));
    if (dev != I.dev) throw Error{PG_INVALID_ARGUMENT, "union_program: run on another device"};
    if (!I.finalized) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        PG_CUDA_THROW(cudaStreamIsCapturing(st, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            throw Error{PG_RUNTIME_ERROR, "union_program: run once before graph capture (workspace allocation)"};
        finalize(st);
    }
    UpParams P = I.P;
    P.tok_pat = tok_pat;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * I.pairs));
    cfg.blockDim = dim3(UP_THREADS);
    cfg.dynamicSmemBytes = UP_SMEM;
    cfg.stream = st;
    // cooperative: the CTAs wait on each other's output tiles, so the launch must
    // guarantee that the whole grid is co-resident (it fails instead of hanging)
    static const int coop = [] {
        const char* e = getenv("PG_PROG_COOP");
        return e ? atoi(e) : 1;
    }();
    cudaLaunchAttribute at[3];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    at[2].id = cudaLaunchAttributeCooperative;
    at[2].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = coop ? 3 : 2;
    PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_union_prog, P));
    count_launch();
}

int UnionProgram::phases() const { return (int)d->phases.size(); }
int UnionProgram::grid() const { return 2 * d->pairs; }

int UnionProgram::debug_dump(unsigned long long* out, size_t n) const {
    if (!d->dbg) return 0;
    PG_CUDA_THROW(cudaMemcpy(out, d->dbg, std::min<size_t>(n, (size_t)2 * d->pairs * 64) * 8, cudaMemcpyDeviceToHost));
    return 1;
}

}  // namespace pg
