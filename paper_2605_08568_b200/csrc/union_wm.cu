// union_wm.cu -- K5d: the heterogeneous decode batch of BASELINE config 4
// (T <= 256 tokens from T prompts, each with its own expert subset S_p) as
// weights-on-M tcgen05 GEMMs with a balanced whole-tile + split-K schedule.
//
// Per linear, masked_forward (rank_experts.hpp:52-72) for every token reads the
// union of the batch's selections -- all r_store experts once a GPU serves more
// than a handful of patterns -- once for the whole batch:
//   stage 1  Z[t, e] = mask_{S_p(t)}(e) * sum_j B^T[e, j] x[t, j]
//   stage 2  Y[t, i] = sum_e A[i, e] Z[t, e]
// Both stages are D^T = W . X^T with the WEIGHTS on the UMMA M side (CTA pair,
// cta_group::2, 256 weight rows per pair) and the whole token batch as N (<= 256
// columns of one TMEM accumulator).  Per 64-wide k-block a CTA loads 16 KB of
// weights and 16 KB of tokens, so the L2->SMEM bytes are 2x the weight bytes,
// against (N tiles x token tile) for tokens on M (the round-1 kernel: the
// 128-token tile re-read for every narrow expert tile).
//
// Work split: tiles of 256 weight rows x all tokens.  Whole tiles go round-
// robin to the pairs (tile p + i * pairs to pair p); the TT mod pairs remaining
// tiles are each cut along K over ~pairs / remainder pairs, ONE piece per pair,
// so every SM streams the same weight bytes whatever the tile count (7 tiles
// of 256 rows for a 1638-expert stage, 86 for up+gate's 22016 rows).  A pair
// runs its split piece first: it stores the f32 partial ([tokens][128 rows]
// per CTA) and raises a tagged flag early; after its whole tiles, each
// participant of a split tile pulls the same token slice of every partial into
// shared memory with bulk copies and sums them in pair order (deterministic:
// the split depends only on the shapes), masks, converts and stores its slice.
// (A contiguous stream-K split was measured first: up to two split pieces per
// pair doubled the partial traffic and serialised two reductions -- 2x slower.)
//
// Warp roles (192 threads, one CTA per SM, persistent pair per TPC):
//   warp 0     TMA producer; the first ring's weight tiles are issued BEFORE
//              griddepcontrol.wait (weights never depend on the previous kernel),
//              the token tiles after it;
//   warp 1     TMEM allocator; the leader CTA's lane 0 issues tcgen05.mma.cta_group::2
//              (M = 256, N = padded T, K = 16) into double-buffered accumulators;
//   warps 2-5  epilogue: tcgen05.ld 32x32b (lane = weight row, columns = tokens),
//              stage-1 selection mask, transposed store Y[t, row] (a warp writes
//              32 consecutive rows of one token per store), or the f32 partial.
// Roofline: HBM, sum_l R_l K_l * 2 bytes of weights per launch; tensor work
// 2 * T * R * K flops (the masked union: 2x the useful flops at K = r_store / 2).
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "tc_ptx.cuh"
#include "umma.cuh"
#include "union_dev.cuh"
#include "union_wm.cuh"

namespace pg {

constexpr int WM_STAGES = 6;
constexpr int WM_STAGE_BYTES = WM_W_BYTES + WM_X_BYTES;  // 32 KB
constexpr int WM_THREADS = 192;
constexpr int WM_MAXG = 4;
// [align slack][ring][barriers + slots, 1 KB][token -> pattern table, 1 KB][epilogue staging 4 x 4 KB]
constexpr int WM_SMEM = 1024 + WM_STAGES * WM_STAGE_BYTES + 1024 + WM_TMAX * 4 + 4 * 32 * 32 * 4;

struct WmGroup {
    int R, K, kb, tiles;
    int Rs;          // rows stored: min(ldo, 256 * tiles) >= R; rows [R, Rs) are exact zeros (zero-filled
                     // weights), so a padded Z (ldo = r rounded to 8) is fully written for the next GEMM
    int tile_base;   // first launch-wide tile index of this GEMM
    void* out;       // [T, ldo] token-major
    long long ldo;
    int out_bf16;
    const uint8_t* mask;  // stage 1: Z[t, e] = 0 unless mask[tok_pat[t] * mask_ld + e]
    long long mask_ld;
};

struct __align__(64) WmParams {
    CUtensorMap wmap[WM_MAXG];  // weights [R, K], box {64, 128}
    CUtensorMap xmap[WM_MAXG];  // tokens [T, K], box {64, Tp / 2}
    WmGroup g[WM_MAXG];
    int ng, T, Tp;
    int full;     // whole-tile rounds: tiles [0, full * pairs) go whole, tile p + i * pairs to pair p
    int rem;      // remaining tiles [full * pairs, full * pairs + rem), each K-split over ~pairs / rem pairs
    const int32_t* tok_pat;
    float* partial;              // [pairs][2 CTAs][WM_PART_FLOATS]
    unsigned* flags;             // [pairs][2 CTAs]: launch tag once the partial is stored
    unsigned long long* epoch;   // launch ticket counter (one add per CTA per launch)
    unsigned long long* dbg;     // optional %globaltimer stamps [grid][8] (PG_WM_DBG=1)
};

#define WM_STAMP(k) \
    do {            \
        if (P.dbg) P.dbg[blockIdx.x * 16 + (k)] = wm_gtimer(); \
    } while (0)

struct WmPiece {
    int g, t, k0, k1;
    int split;  // 1: part of a remainder tile cut across pairs (f32 partial + end-of-launch reduction)
};

__device__ __forceinline__ void wm_tile(const WmParams& P, int Ti, int& g, int& t) {
    g = 0;
    while (g + 1 < P.ng && P.g[g + 1].tile_base <= Ti) ++g;
    t = Ti - P.g[g].tile_base;
}

// This pair's share of the remainder tiles: remainder tile r is cut along K
// over pairs [r * np / rem, (r + 1) * np / rem) (at most kb of them), one piece
// per pair.  Returns false when the pair has no remainder piece.
__device__ __forceinline__ bool wm_rem_piece(const WmParams& P, int np, int pair, WmPiece& pc, int& pf, int& n) {
    if (P.rem == 0) return false;
    int r = (int)((long long)pair * P.rem / np);
    while (r + 1 < P.rem && (r + 1) * np / P.rem <= pair) ++r;
    while (r > 0 && r * np / P.rem > pair) --r;
    pf = r * np / P.rem;
    const int nr = (r + 1) * np / P.rem - pf, j = pair - pf;
    int g, t;
    wm_tile(P, P.full * np + r, g, t);
    const int kb = P.g[g].kb;
    n = min(nr, kb);
    if (j >= n) return false;
    pc.g = g;
    pc.t = t;
    pc.k0 = j * kb / n;
    pc.k1 = (j + 1) * kb / n;
    pc.split = n > 1;
    return true;
}

// pieces of a pair, in processing order: its remainder piece first (a split
// piece's partial is then published early, so the end-of-launch reduction does
// not wait on it), then its whole tiles
struct WmSched {
    int npieces, has_rem, pf, n;
    WmPiece rem;
};
__device__ __forceinline__ WmSched wm_sched(const WmParams& P, int np, int pair) {
    WmSched S;
    S.has_rem = wm_rem_piece(P, np, pair, S.rem, S.pf, S.n) ? 1 : 0;
    S.npieces = P.full + S.has_rem;
    return S;
}
__device__ __forceinline__ WmPiece wm_get(const WmParams& P, const WmSched& S, int np, int pair, int idx) {
    if (S.has_rem) {
        if (idx == 0) return S.rem;
        --idx;
    }
    WmPiece pc;
    wm_tile(P, idx * np + pair, pc.g, pc.t);
    pc.k0 = 0;
    pc.k1 = P.g[pc.g].kb;
    pc.split = 0;
    return pc;
}

__global__ void __launch_bounds__(WM_THREADS, 1) k_union_wm(const __grid_constant__ WmParams P) {
    extern __shared__ __align__(1024) unsigned char wsmem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(wsmem) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + WM_STAGES * WM_STAGE_BYTES);
    uint64_t* full = bars;                       // [STAGES] (leader's copy used)
    uint64_t* empty = bars + WM_STAGES;          // [STAGES] (each CTA)
    uint64_t* tfull = bars + 2 * WM_STAGES;      // [2] (each CTA)
    uint64_t* tempty = bars + 2 * WM_STAGES + 2; // [2] (leader's copy: both CTAs' epilogues)
    uint64_t* rbar = bars + 2 * WM_STAGES + 4;   // reduction bulk loads (each CTA)
    uint32_t* slots = reinterpret_cast<uint32_t*>(bars + 2 * WM_STAGES + 5);  // [0] tmem base, [1] launch tag
    int32_t* tps = reinterpret_cast<int32_t*>(base + WM_STAGES * WM_STAGE_BYTES + 1024);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, np = gridDim.x >> 1;
    if (threadIdx.x == 0) {
        WM_STAMP(0);
        for (int s = 0; s < WM_STAGES; ++s) {
            u_mbar_init(u_smem(&full[s]), 1);
            u_mbar_init(u_smem(&empty[s]), 1);
        }
        for (int a = 0; a < 2; ++a) {
            u_mbar_init(u_smem(&tfull[a]), 1);
            u_mbar_init(u_smem(&tempty[a]), 8);  // 4 epilogue warps x 2 CTAs
        }
        u_mbar_init(u_smem(rbar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // launch tag: taken before launch_dependents (below, after the cluster
        // barrier), so every CTA of this launch holds its ticket before any CTA
        // of the next launch on the stream can start: old / grid = launch index
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

    const WmSched S = wm_sched(P, np, pair);

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            uint64_t pfirst, plast;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pfirst));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(plast));
            const uint32_t xbytes = (uint32_t)(P.Tp / 2) * WM_BK * 2;
            const uint32_t bytes = 2u * (WM_W_BYTES + xbytes);
            const int xrow = (int)rank * (P.Tp / 2);
            auto load_w = [&](const WmPiece& pc, int kb, int s) {
                const uint32_t fb = leader_addr(u_smem(&full[s]));
                if (leader) u_mbar_arrive_tx_cluster(fb, bytes);
                u_tma_2d_pair_h(u_smem(base + s * WM_STAGE_BYTES), &P.wmap[pc.g], kb * WM_BK,
                                pc.t * 2 * WM_BM + (int)rank * WM_BM, fb, pfirst);
            };
            auto load_x = [&](const WmPiece& pc, int kb, int s) {
                const uint32_t fb = leader_addr(u_smem(&full[s]));
                u_tma_2d_pair_h(u_smem(base + s * WM_STAGE_BYTES + WM_W_BYTES), &P.xmap[pc.g], kb * WM_BK, xrow, fb,
                                plast);
            };
            // first ring: weight tiles now (immutable), token tiles once the
            // previous kernel (which may produce them) has completed
            int s = 0;
            for (int pi = 0; pi < S.npieces && s < WM_STAGES; ++pi) {
                const WmPiece pc = wm_get(P, S, np, pair, pi);
                for (int kb = pc.k0; kb < pc.k1 && s < WM_STAGES; ++kb) load_w(pc, kb, s++);
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
            WM_STAMP(1);
            uint32_t ph = 0;
            int issued = 0;
            s = 0;
            for (int pi = 0; pi < S.npieces; ++pi) {
                const WmPiece pc = wm_get(P, S, np, pair, pi);
                for (int kb = pc.k0; kb < pc.k1; ++kb, ++issued) {
                    if (issued >= WM_STAGES) {
                        u_mbar_wait(u_smem(&empty[s]), ph ^ 1);
                        load_w(pc, kb, s);
                    }
                    load_x(pc, kb, s);
                    if (++s == WM_STAGES) { s = 0; ph ^= 1; }
                }
            }
            WM_STAMP(2);
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (leader && lane == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P.Tp >> 3) << 17) |
                                   ((uint32_t)((2 * WM_BM) >> 4) << 24);
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int pi = 0; pi < S.npieces; ++pi) {
                const WmPiece pc = wm_get(P, S, np, pair, pi);
                u_mbar_wait(u_smem(&tempty[acc]), aph ^ 1);  // both CTAs drained this accumulator
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(acc * WM_TMAX);
                for (int kb = pc.k0; kb < pc.k1; ++kb) {
                    u_mbar_wait(u_smem(&full[s]), ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = u_smem(base + s * WM_STAGE_BYTES), sb = sa + WM_W_BYTES;
#pragma unroll
                    for (int k = 0; k < WM_BK / 16; ++k)
                        u_mma2(d, u_desc(sa + k * 32), u_desc(sb + k * 32), idesc, (kb > pc.k0 || k > 0) ? 1u : 0u);
                    u_commit2(u_smem(&empty[s]));
                    if (++s == WM_STAGES) { s = 0; ph ^= 1; }
                }
                u_commit2(u_smem(&tfull[acc]));
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2-5, both CTAs)
        asm volatile("griddepcontrol.wait;" ::: "memory");  // outputs may still be read by the previous kernel
        for (int t = threadIdx.x - 64; t < P.T; t += 128) tps[t] = P.tok_pat ? __ldg(P.tok_pat + t) : 0;
        wm_bar_epi();
        const int q = warp & 3;
        int acc = 0;
        uint32_t aph = 0;
        for (int pi = 0; pi < S.npieces; ++pi) {
            const WmPiece pc = wm_get(P, S, np, pair, pi);
            const WmGroup& G = P.g[pc.g];
            u_mbar_wait(u_smem(&tfull[acc]), aph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (warp == 2 && lane == 0 && pi == 0) WM_STAMP(8);
            const uint32_t taddr = tmem + (uint32_t)(acc * WM_TMAX) + ((uint32_t)(q * 32) << 16);
            float* stg = reinterpret_cast<float*>(base + WM_STAGES * WM_STAGE_BYTES + 2048) + q * (WM_STG_BYTES / 4);
            if (!pc.split) wm_epi_direct(P.Tp, P.T, G, taddr, pc.t * 2 * WM_BM + (int)rank * WM_BM + q * 32, tps, stg, lane);
            else wm_epi_partial(P.Tp, taddr, P.partial + (size_t)(pair * 2 + (int)rank) * WM_PART_FLOATS, q, stg, lane);
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) u_mbar_arrive_cluster(leader_addr(u_smem(&tempty[acc])));
            if (pc.split) {  // publish the partial: every epilogue thread's stores, then the tagged flag
                wm_bar_epi();
                if (warp == 2 && lane == 0) {
                    WM_STAMP(9);
                    st_release(P.flags + pair * 2 + (int)rank, tag);
                    WM_STAMP(10);
                }
            }
            if (++acc == 2) { acc = 0; aph ^= 1; }
        }
        if (warp == 2 && lane == 0) WM_STAMP(3);
    }

    // ---------------------------------------------------- split tile: reduce
    // Every participant of a split remainder tile sums one token slice of all
    // the tile's partials (pair order), masks and stores it.  The ring is idle:
    // all MMAs retired before the epilogue saw their accumulators.
    __syncthreads();
    if (S.has_rem && S.rem.split) {
        const WmPiece& pc = S.rem;
        const WmGroup& G = P.g[pc.g];
        const int pf = S.pf, n = S.n, me = pair - pf;
        const int ta = me * P.Tp / n, tb = std::min(P.T, (me + 1) * P.Tp / n);
        const int cnt = std::max(0, tb - ta);
        float* buf = reinterpret_cast<float*>(base);  // [n][cnt][128]
        if (warp == 0 && cnt > 0) {
            // every participant's flag polled in parallel (one lane each)
            for (int pp0 = pf; pp0 < pf + n; pp0 += 32) {
                const int pp = pp0 + lane;
                if (pp < pf + n) {
                    const unsigned* f = P.flags + pp * 2 + (int)rank;
                    while (ld_relaxed(f) != tag) {
                    }
                    (void)ld_acquire(f);
                }
            }
            __syncwarp();
        }
        if (threadIdx.x == 0 && cnt > 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            WM_STAMP(4);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const uint32_t bytes = (uint32_t)cnt * WM_BM * 4;
            u_mbar_arrive_tx(u_smem(rbar), bytes * (uint32_t)n);
            for (int pp = pf; pp < pf + n; ++pp) {
                const float* src = P.partial + (size_t)(pp * 2 + (int)rank) * WM_PART_FLOATS + (size_t)ta * WM_BM;
                bulk_g2s(u_smem(buf + (size_t)(pp - pf) * cnt * WM_BM), src, bytes, u_smem(rbar));
            }
        }
        if (cnt > 0) {
            u_mbar_wait(u_smem(rbar), 0);
            if (threadIdx.x == 0) WM_STAMP(11);
            const int row0 = pc.t * 2 * WM_BM + (int)rank * WM_BM;
            for (int idx = threadIdx.x; idx < cnt * (WM_BM / 4); idx += WM_THREADS) {
                const int tl = idx / (WM_BM / 4), c4 = idx % (WM_BM / 4);
                float4 a = reinterpret_cast<const float4*>(buf + (size_t)tl * WM_BM)[c4];
                for (int pp = 1; pp < n; ++pp) {
                    const float4 b = reinterpret_cast<const float4*>(buf + ((size_t)pp * cnt + tl) * WM_BM)[c4];
                    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
                }
                const int tok = ta + tl, row = row0 + 4 * c4;
                if (G.mask) {
                    const uint8_t* mr = G.mask + (long long)tps[tok] * G.mask_ld + row;
                    const uint32_t mw = *reinterpret_cast<const uint32_t*>(mr);
                    if (!(mw & 0xFFu)) a.x = 0.f;
                    if (!(mw & 0xFF00u)) a.y = 0.f;
                    if (!(mw & 0xFF0000u)) a.z = 0.f;
                    if (!(mw & 0xFF000000u)) a.w = 0.f;
                }
                if (row + 3 < G.Rs) {
                    if (G.out_bf16) {
                        __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
                        uint2 w;
                        w.x = *reinterpret_cast<uint32_t*>(&lo);
                        w.y = *reinterpret_cast<uint32_t*>(&hi);
                        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(G.out) + (long long)tok * G.ldo + row) = w;
                    } else {
                        *reinterpret_cast<float4*>(static_cast<float*>(G.out) + (long long)tok * G.ldo + row) = a;
                    }
                } else {
                    if (row < G.Rs) wm_put(G, tok, row, a.x);
                    if (row + 1 < G.Rs) wm_put(G, tok, row + 1, a.y);
                    if (row + 2 < G.Rs) wm_put(G, tok, row + 2, a.z);
                }
            }
        }
        if (threadIdx.x == 0 && cnt > 0) WM_STAMP(13);
    }

    if (threadIdx.x == 0) WM_STAMP(6);
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    if (threadIdx.x == 0) WM_STAMP(7);
}

// ---------------------------------------------------------------- host side
namespace {
struct WmWorkspace {
    char* p = nullptr;
    size_t bytes = 0;
};
std::mutex g_wm_mu;
// per (device, stream, grid): [epoch 256 B | flags | partials]; the flags carry
// launch tags, so nothing is reset between launches (graph replays included)
std::map<std::tuple<int, cudaStream_t, int>, WmWorkspace> g_wm_ws;

void wm_set_attr() {
    once_per_device(reinterpret_cast<const void*>(&k_union_wm), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_union_wm, cudaFuncAttributeMaxDynamicSharedMemorySize, WM_SMEM));
    });
}

int wm_max_pairs() {  // co-resident CTA pairs (per device)
    static std::atomic<int> cache[128];
    const int dev = current_device();
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v) return v;
    wm_set_attr();
    const int sms = device_sms();
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3((unsigned)(sms / 2 * 2));
    q.blockDim = dim3(WM_THREADS);
    q.dynamicSmemBytes = WM_SMEM;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 2;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    q.attrs = a;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_union_wm, &q) != cudaSuccess || n <= 0) n = sms / 2;
    if (getenv("PG_UMMA_DEBUG")) fprintf(stderr, "union_wm: max active clusters %d (sms %d)\n", n, sms);
    cache[dev].store(n, std::memory_order_relaxed);
    return n;
}
}  // namespace

static unsigned long long* g_wm_dbg = nullptr;
static unsigned long long* wm_debug_buffer() {
    static const bool on = [] {
        const char* e = getenv("PG_WM_DBG");
        return e && atoi(e);
    }();
    if (on && !g_wm_dbg) {
        PG_CUDA_THROW(cudaMalloc(&g_wm_dbg, 1024 * 16 * 8));
        PG_CUDA_THROW(cudaMemset(g_wm_dbg, 0, 1024 * 16 * 8));
    }
    return on ? g_wm_dbg : nullptr;
}

int union_wm_debug_dump(unsigned long long* out, size_t n) {
    if (!g_wm_dbg) return 0;
    PG_CUDA_THROW(cudaMemcpy(out, g_wm_dbg, std::min<size_t>(n, 1024 * 16) * 8, cudaMemcpyDeviceToHost));
    return 1;
}

bool union_wm_enabled() {
    static const int v = [] {
        const char* e = getenv("PG_UNION_WM");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

bool union_wm_ok(int T, const std::vector<WmSpec>& specs) {
    if (!union_wm_enabled() || T < 1 || T > WM_TMAX || specs.empty() || (int)specs.size() > WM_MAXG) return false;
    // measured per GEMM phase of the config-4 layer (ncu, profiles/r2_union_wm.txt):
    // this kernel wins when every pair streams >= ~20 k-blocks (up+gate's second
    // GEMM, down's first); below that the split-tile partials and the pipeline
    // fill/drain cost more than the round-1 tokens-on-M kernel's token re-reads
    static const int min_kb = [] {
        const char* e = getenv("PG_UNION_WM_MINKB");
        return e ? atoi(e) : 20;
    }();
    {
        long long work = 0;
        for (const WmSpec& s : specs)
            work += (long long)((s.R + 2 * WM_BM - 1) / (2 * WM_BM)) * ((s.K + WM_BK - 1) / WM_BK);
        if (work < (long long)min_kb * wm_max_pairs()) return false;
    }
    for (const WmSpec& s : specs) {
        if (s.R < 1 || s.K < 1 || (s.ldw * 2) % 16 || (s.ldx * 2) % 16 || s.ldo % 4) return false;
        if (reinterpret_cast<uintptr_t>(s.out) % 16 || (s.out_bf16 && s.ldo % 8)) return false;
        if (s.mask && (s.mask_ld % 16)) return false;
    }
    return true;
}

void launch_union_wm(const std::vector<WmSpec>& specs, int T, const int32_t* tok_pat, cudaStream_t st) {
    wm_set_attr();
    if (!union_wm_ok(T, specs)) throw Error{PG_INVALID_ARGUMENT, "union_wm: unsupported batch"};
    const int Tp = (T + 31) / 32 * 32;
    auto P = std::make_unique<WmParams>();
    int TT = 0;
    for (size_t g = 0; g < specs.size(); ++g) {
        const WmSpec& s = specs[g];
        WmGroup& G = P->g[g];
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
        P->wmap[g] = make_map(s.w, s.R, s.K, s.ldw, WM_BM);
        P->xmap[g] = make_map(s.x, T, s.K, s.ldx, Tp / 2);
    }
    P->ng = (int)specs.size();
    P->T = T;
    P->Tp = Tp;
    P->tok_pat = tok_pat;
    P->dbg = wm_debug_buffer();
    // whole tiles round-robin over the pairs; the last TT mod pairs tiles are
    // cut along K so every pair streams the same weight bytes
    const int pairs = wm_max_pairs();
    P->full = TT / pairs;
    P->rem = TT % pairs;
    const int grid = 2 * pairs;
    {
        int dev = 0;
        PG_CUDA_THROW(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(g_wm_mu);
        WmWorkspace& w = g_wm_ws[std::make_tuple(dev, st, grid)];
        const size_t flags_bytes = (size_t)pairs * 2 * sizeof(unsigned);
        const size_t need = 256 + (flags_bytes + 255) / 256 * 256 + (size_t)pairs * 2 * WM_PART_FLOATS * 4;
        if (w.bytes < need) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            PG_CUDA_THROW(cudaStreamIsCapturing(st, &cs));
            if (cs != cudaStreamCaptureStatusNone)
                throw Error{PG_RUNTIME_ERROR, "union_wm: workspace must be sized by a call before graph capture"};
            PG_CUDA_THROW(cudaStreamSynchronize(st));
            if (w.p) PG_CUDA_THROW(cudaFree(w.p));
            PG_CUDA_THROW(cudaMalloc(&w.p, need));
            PG_CUDA_THROW(cudaMemsetAsync(w.p, 0, 256 + (flags_bytes + 255) / 256 * 256, st));
            w.bytes = need;
        }
        P->epoch = reinterpret_cast<unsigned long long*>(w.p);
        P->flags = reinterpret_cast<unsigned*>(w.p + 256);
        P->partial = reinterpret_cast<float*>(w.p + 256 + (flags_bytes + 255) / 256 * 256);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(WM_THREADS);
    cfg.dynamicSmemBytes = WM_SMEM;
    cfg.stream = st;
    // cooperative: split-tile participants wait on each other's partial flags
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
    cfg.numAttrs = 3;
    PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_union_wm, *P));
    count_launch();
}

void union_wm_release(cudaStream_t st) {
    int dev = 0;
    PG_CUDA_THROW(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_wm_mu);
    for (auto it = g_wm_ws.begin(); it != g_wm_ws.end();) {
        if (std::get<0>(it->first) == dev && std::get<1>(it->first) == st) {
            if (it->second.p) PG_CUDA_THROW(cudaFree(it->second.p));
            it = g_wm_ws.erase(it);
        } else {
            ++it;
        }
    }
}

}  // namespace pg
