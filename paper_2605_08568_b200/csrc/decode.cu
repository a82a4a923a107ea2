// decode.cu -- K4/K6: single-launch decode chain for the rank-expert layer
// (T = 1 token): y = A_S (B_S^T x), one or more linears per phase sharing x
// (build_plan's fused_B / batched_A groups, exec_engine.hpp:46-68), with the
// MLP's silu(gate)*up (toy_lm.hpp:250-257) as a stage-2 epilogue feeding the
// next phase (down_proj).
//
// One persistent cooperative kernel, one CTA per SM (148 x 512 threads):
//   0. every CTA issues cp.async.bulk.prefetch.L2 for its 1/G share of ALL
//      weight bytes the chain will read, so HBM streams at full rate from the
//      first cycle and the later stages hit L2;
//   1. stage 1: warp items (linear, slot, row-chunk) -> z partials (f32 acc);
//   2. grid barrier; z (+ activity mask) into shared memory;
//   3. stage 2: warps own output rows, A_S row runs dotted with z from smem;
//   4. grid barrier before the next phase consumes this phase's output.
// Roofline: HBM-bound, algorithmic bytes = sum_l K_l (m_l + n_l) * dtype.
// Deterministic: every reduction has a fixed order (warp trees, partials
// summed in chunk order).
#include <algorithm>

#include "chain.cuh"

namespace pg {

template <typename W> struct CVec;
template <> struct CVec<double> { static constexpr int n = 2; };
template <> struct CVec<float> { static constexpr int n = 4; };
template <> struct CVec<__nv_bfloat16> { static constexpr int n = 8; };

template <typename W, typename A>
__device__ __forceinline__ void cunpack(const int4& v, A* o) {
    if constexpr (sizeof(W) == 2) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(h[q]);
            o[2 * q] = f.x;
            o[2 * q + 1] = f.y;
        }
    } else if constexpr (sizeof(W) == 4) {
        const float4 f = *reinterpret_cast<const float4*>(&v);
        o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
    } else {
        const double2 d = *reinterpret_cast<const double2*>(&v);
        o[0] = d.x; o[1] = d.y;
    }
}

__device__ __forceinline__ int c_slot_index(const SlotMap& sm, int s) {
    if (sm.idx) return sm.idx[s];
    return s < sm.run0_len ? s : sm.run1_start + (s - sm.run0_len);
}
__device__ __forceinline__ bool c_slot_active(const SlotMap& sm, int s) {
    if (sm.idx) return sm.idx[s] >= 0;
    if (s < sm.run0_len) return sm.mask == nullptr || sm.mask[s] != 0;
    return true;
}

__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// prefetch [base, base+bytes) split over the grid; lanes of warp 0 issue 16 KB pieces
__device__ void prefetch_range(const char* base, size_t bytes, int cta, int ncta, int lane) {
    if (!base || bytes == 0) return;
    const size_t per = ((bytes + ncta - 1) / ncta + 15) & ~size_t(15);
    const size_t b0 = (size_t)cta * per;
    if (b0 >= bytes) return;
    const size_t b1 = min(bytes, b0 + per);
    for (size_t o = b0 + (size_t)lane * 16384; o < b1; o += 32 * 16384) {
        const size_t left = b1 - o;
        const uint32_t len = (uint32_t)(left < 16384 ? left : 16384) & ~15u;
        if (len) l2_prefetch(base + o, len);
    }
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Monotone counter barrier: each arrival adds 1; generation g completes when
// the counter reaches (g+1)*G.  Requires co-residency (cooperative launch).
__device__ __forceinline__ void grid_barrier(unsigned long long* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long old = atomicAdd(bar, 1ull);
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
        while (ld_acquire(bar) < target) __nanosleep(20);
        __threadfence();
    }
    __syncthreads();
}

template <typename W>
__device__ void chain_prefetch(const ChainParams& P, int lane) {
    const int cta = blockIdx.x, ncta = gridDim.x;
    const size_t es = sizeof(W);
    for (int ph = 0; ph < P.nphase; ++ph) {
        for (int l = 0; l < P.ph[ph].nlin; ++l) {
            const ChainLin& L = P.ph[ph].lin[l];
            const SlotMap sm = resolve(L.sm);
            const char* bt = static_cast<const char*>(L.bt);
            const char* a = static_cast<const char*>(L.a);
            if (sm.idx) continue;  // gather layouts: no contiguous ranges to prefetch
            prefetch_range(bt, (size_t)sm.run0_len * L.ldb * es, cta, ncta, lane);
            prefetch_range(bt + (size_t)sm.run1_start * L.ldb * es, (size_t)sm.run1_len * L.ldb * es, cta,
                           ncta, lane);
            if (sm.run1_len == 0 && L.lda == sm.run0_len) {
                prefetch_range(a, (size_t)L.m * L.lda * es, cta, ncta, lane);
            } else {
                for (int i = cta * 32 + lane; i < L.m; i += ncta * 32) {
                    const char* row = a + (size_t)i * L.lda * es;
                    if (sm.run0_len) l2_prefetch(row, (uint32_t)(sm.run0_len * es));
                    if (sm.run1_len) l2_prefetch(row + (size_t)sm.run1_start * es, (uint32_t)(sm.run1_len * es));
                }
            }
        }
    }
}

template <typename W>
__global__ void __launch_bounds__(kChainThreads, 1) k_chain(const __grid_constant__ ChainParams P) {
    using A = typename Acc<W>::type;
    constexpr int V = CVec<W>::n;
    constexpr int U = 8;  // 16-byte loads in flight per lane per batch
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kChainWarps + warp, nw = gridDim.x * kChainWarps;

    if (P.prefetch && warp == 0) chain_prefetch<W>(P, lane);

    for (int ph = 0; ph < P.nphase; ++ph) {
        const ChainPhase& Q = P.ph[ph];
        const int n = Q.lin[0].n;
        // ---- stage the phase input x into shared memory
        W* xs = reinterpret_cast<W*>(smem);
        {
            const int nv = (n * (int)sizeof(W)) / 16;
            const int4* xv = reinterpret_cast<const int4*>(Q.x);
            for (int v = threadIdx.x; v < nv; v += kChainThreads) reinterpret_cast<int4*>(xs)[v] = xv[v];
            for (int e = nv * 16 / (int)sizeof(W) + threadIdx.x; e < n; e += kChainThreads)
                xs[e] = static_cast<const W*>(Q.x)[e];
        }
        __syncthreads();
        // ---- stage 1: items (linear, slot, chunk)
        const int split = Q.split;
        int nsl[kMaxLin];
        int total = 0;
        for (int l = 0; l < Q.nlin; ++l) {
            nsl[l] = resolve(Q.lin[l].sm).nslots();
            total += nsl[l] * split;
        }
        const int nvec = n / V;
        const int cvec = (nvec + split - 1) / split;
        for (int it = gw; it < total; it += nw) {
            int l = 0, rem = it;
            while (l + 1 < Q.nlin && rem >= nsl[l] * split) { rem -= nsl[l] * split; ++l; }
            const ChainLin& L = Q.lin[l];
            const SlotMap sm = resolve(L.sm);
            const int slot = rem / split, part = rem % split;
            A acc = A(0);
            if (c_slot_active(sm, slot)) {
                const int4* row = reinterpret_cast<const int4*>(static_cast<const W*>(L.bt) +
                                                                (int64_t)c_slot_index(sm, slot) * L.ldb);
                const int v0 = part * cvec, v1 = min(nvec, v0 + cvec);
                for (int vb = v0 + lane; vb < v1; vb += 32 * U) {
                    int4 w4[U];
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (vb + 32 * u < v1) w4[u] = ld_stream(row + vb + 32 * u);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int v = vb + 32 * u;
                        if (v < v1) {
                            A wv[V], xv[V];
                            cunpack<W, A>(w4[u], wv);
                            cunpack<W, A>(*reinterpret_cast<const int4*>(xs + (int64_t)v * V), xv);
#pragma unroll
                            for (int q = 0; q < V; ++q) acc = fma(wv[q], xv[q], acc);
                        }
                    }
                }
                if (part == split - 1) {  // scalar tail when n % V != 0
                    const W* rs = reinterpret_cast<const W*>(row);
                    for (int j = nvec * V + lane; j < n; j += 32) {
                        if constexpr (sizeof(W) == 2) acc = fma(__bfloat162float(rs[j]), __bfloat162float(xs[j]), acc);
                        else acc = fma((A)rs[j], (A)xs[j], acc);
                    }
                }
            }
            acc = warp_sum(acc);
            if (lane == 0) static_cast<A*>(L.zpart)[(int64_t)slot * split + part] = acc;
        }
        grid_barrier(P.bar);
        // ---- z into shared memory (partials summed in chunk order; mask)
        A* zs = reinterpret_cast<A*>(smem);
        int zoff[kMaxLin];
        {
            int o = 0;
            for (int l = 0; l < Q.nlin; ++l) {
                zoff[l] = o;
                const SlotMap sm = resolve(Q.lin[l].sm);
                const A* zp = static_cast<const A*>(Q.lin[l].zpart);
                for (int s = threadIdx.x; s < nsl[l]; s += kChainThreads) {
                    A v = A(0);
                    for (int q = 0; q < split; ++q) v += zp[(int64_t)s * split + q];
                    zs[o + s] = c_slot_active(sm, s) ? v : A(0);
                }
                o += (nsl[l] + 3) & ~3;
            }
        }
        __syncthreads();
        // ---- stage 2: rows
        const int rows_per_lin = Q.lin[0].m;
        int row_total = 0;
        if (Q.epilogue == 1) row_total = rows_per_lin;
        else
            for (int l = 0; l < Q.nlin; ++l) row_total += Q.lin[l].m;
        for (int it = gw; it < row_total; it += nw) {
            int l0 = 0, i = it;
            if (Q.epilogue == 0)
                while (l0 + 1 < Q.nlin && i >= Q.lin[l0].m) { i -= Q.lin[l0].m; ++l0; }
            const int lcount = Q.epilogue == 1 ? 2 : 1;
            A res[2] = {A(0), A(0)};
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (k >= lcount) break;
                const int l = Q.epilogue == 1 ? k : l0;
                const ChainLin& L = Q.lin[l];
                const SlotMap sm = resolve(L.sm);
                const W* row = static_cast<const W*>(L.a) + (int64_t)i * L.lda;
                const A* z = zs + zoff[l];
                A acc = A(0);
                if (sm.idx) {
                    for (int s = lane; s < nsl[l]; s += 32) {
                        const int c = sm.idx[s];
                        if (c < 0) continue;
                        if constexpr (sizeof(W) == 2) acc = fma(__bfloat162float(row[c]), z[s], acc);
                        else acc = fma((A)row[c], z[s], acc);
                    }
                } else {
                    const int nv0 = sm.run0_len / V, nv = nv0 + sm.run1_len / V;
                    for (int vb = lane; vb < nv; vb += 32 * U) {
                        int4 w4[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int v = vb + 32 * u;
                            if (v < nv) {
                                const int col = v < nv0 ? v * V : sm.run1_start + (v - nv0) * V;
                                w4[u] = ld_stream(row + col);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int v = vb + 32 * u;
                            if (v < nv) {
                                A wv[V];
                                cunpack<W, A>(w4[u], wv);
#pragma unroll
                                for (int q = 0; q < V; ++q) acc = fma(wv[q], z[v * V + q], acc);
                            }
                        }
                    }
                }
                res[k] = warp_sum(acc);
            }
            if (lane == 0) {
                if (Q.epilogue == 1) {
                    const float up = (float)res[0], g = (float)res[1];
                    const float v = g / (1.0f + __expf(-g)) * up;
                    W* act = static_cast<W*>(Q.act);
                    if constexpr (sizeof(W) == 2) act[i] = __float2bfloat16_rn(v);
                    else act[i] = (W)(g / (1.0f + expf(-g)) * up);
                } else {
                    void* y = Q.lin[l0].y;
                    if (Q.ydt == PG_F32) static_cast<float*>(y)[i] = (float)res[0];
                    else if (Q.ydt == PG_F64) static_cast<double*>(y)[i] = (double)res[0];
                    else static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn((float)res[0]);
                }
            }
        }
        if (ph + 1 < P.nphase) grid_barrier(P.bar);
    }
}

static int g_num_sms = 0;
int chain_grid() {
    if (!g_num_sms) {
        int dev = 0;
        PG_CUDA_THROW(cudaGetDevice(&dev));
        PG_CUDA_THROW(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return g_num_sms;
}

int chain_split(int total_slots) {
    const int nw = chain_grid() * kChainWarps;
    int s = (nw + total_slots - 1) / std::max(total_slots, 1);
    return std::max(1, std::min(s, 8));
}

template <typename W>
static void launch_chain_t(const ChainParams& P, size_t smem, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_chain<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(chain_grid());
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_chain<W>, P));
    count_launch();
}

void launch_chain(pg_dtype wdt, const ChainParams& P, size_t smem, cudaStream_t st) {
    if (wdt == PG_F64) launch_chain_t<double>(P, smem, st);
    else if (wdt == PG_F32) launch_chain_t<float>(P, smem, st);
    else launch_chain_t<__nv_bfloat16>(P, smem, st);
}

}  // namespace pg
