// cache.cu -- K2: pattern-cache cosine nearest neighbour, bit-identical in
// entry / hit to the reference (include/parse/pattern_cache.hpp:38-47,104-117),
// plus the embed_prompt pooling half (:60-64).
//
// Roofline: the scan streams the N x d f64 embedding table once (8*N*d bytes)
// -- HBM-bound.  The query lives in shared memory.
//
// Exactness: the fast scan accumulates num, na, nb with FMA warp trees and a
// per-entry bound e_i = 2*gamma*(sum|a_j q_j|/(|a||q|) + |sim_i|) + slack,
// gamma = 4(d+4)u, covering both our rounding and the reference's sequential
// rounding.  M = max fast sim; entries with sim_i >= M - 2e are recomputed in
// reference order (three sequential accumulators, num/(sqrt(na)*sqrt(nb)))
// unless only one entry is in the band; the strict-'>' first-maximum rule
// (:109) then runs on exact values.  hit (>=, :115) is decided on the exact
// value whenever the fast value is within the bound of min_similarity.
#include "block_utils.cuh"

namespace pg {

constexpr int kCosWarps = 8;

__global__ void __launch_bounds__(kCosWarps * 32)
k_cosine_scan(const double* __restrict__ emb, const double* __restrict__ q, int N, int d,
              double* __restrict__ sim, double* __restrict__ bnd) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* qs = reinterpret_cast<double*>(smem);
    for (int j = threadIdx.x; j < d; j += blockDim.x) qs[j] = q[j];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const double gam = 4.0 * (double)(d + 4) * kU;
    const bool vec = (d & 1) == 0;
    for (int e = blockIdx.x * kCosWarps + (threadIdx.x >> 5); e < N; e += gridDim.x * kCosWarps) {
        const double* a = emb + (int64_t)e * d;
        double num = 0, na = 0, nb = 0, sab = 0;
        if (vec) {
            for (int j = 2 * lane; j < d; j += 64) {
                const double2 av = __ldg(reinterpret_cast<const double2*>(a + j));
                const double2 qv = *reinterpret_cast<const double2*>(qs + j);
                num = fma(av.x, qv.x, num); num = fma(av.y, qv.y, num);
                na = fma(av.x, av.x, na); na = fma(av.y, av.y, na);
                nb = fma(qv.x, qv.x, nb); nb = fma(qv.y, qv.y, nb);
                sab += fabs(av.x * qv.x) + fabs(av.y * qv.y);
            }
        } else {
            for (int j = lane; j < d; j += 32) {
                const double av = __ldg(a + j), qv = qs[j];
                num = fma(av, qv, num); na = fma(av, av, na); nb = fma(qv, qv, nb);
                sab += fabs(av * qv);
            }
        }
        num = warp_sum(num); na = warp_sum(na); nb = warp_sum(nb); sab = warp_sum(sab);
        if (lane == 0) {
            const double den = sqrt(na) * sqrt(nb);
            const double s = num / den;
            sim[e] = s;
            double b = 2.0 * gam * (sab / den + fabs(s)) * 1.0000001 + 1e-300;
            if (!(den > 1e-150)) b = INFINITY;  // tiny/zero norms: always recompute
            bnd[e] = b;
        }
    }
}

// Wide scan (d a multiple of 8): WPE warps per entry, EPB entries per block,
// each lane keeping 8 double2 loads in flight (the one-warp-per-entry scan
// leaves ~4 KB in flight per warp: latency-bound at N = 1024).  Partial sums
// meet in shared memory; the bound argument is order-independent.
#ifndef COS_WPE
#define COS_WPE 4
#endif
#ifndef COS_EPB
#define COS_EPB 8  // entries per block: 1024 threads, the query staged once per 8 entries
#endif
#ifndef COS_BPS
#define COS_BPS 2  // blocks per SM at most (each stages the query once)
#endif
constexpr int kCosWPE = COS_WPE, kCosEPB = COS_EPB;
__global__ void __launch_bounds__(kCosWPE * kCosEPB * 32)
k_cosine_scan_wide(const double* __restrict__ emb, const double* __restrict__ q, int N, int d,
                   double* __restrict__ sim, double* __restrict__ bnd) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* qs = reinterpret_cast<double*>(smem);
    double* part = qs + d;  // [EPB][WPE][4]
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the select kernel may start its prologue
    for (int j = threadIdx.x; j < d; j += blockDim.x) qs[j] = q[j];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int eg = warp / kCosWPE, wq = warp % kCosWPE;
    const int span = d / kCosWPE;  // doubles per warp (even: d % 8 == 0)
    const double gam = 4.0 * (double)(d + 4) * kU;
    for (int e0 = blockIdx.x * kCosEPB; e0 < N; e0 += gridDim.x * kCosEPB) {
        const int e = e0 + eg;
        double num = 0, na = 0, nb = 0, sab = 0;
        if (e < N) {
            const double* a = emb + (int64_t)e * d + wq * span;
            const double* qq = qs + wq * span;
            for (int j0 = 2 * lane; j0 < span; j0 += 64 * 8) {
                double2 av[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = j0 + 64 * u;
                    av[u] = j < span ? __ldg(reinterpret_cast<const double2*>(a + j)) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = j0 + 64 * u;
                    const double2 qv = j < span ? *reinterpret_cast<const double2*>(qq + j) : make_double2(0.0, 0.0);
                    num = fma(av[u].x, qv.x, num); num = fma(av[u].y, qv.y, num);
                    na = fma(av[u].x, av[u].x, na); na = fma(av[u].y, av[u].y, na);
                    nb = fma(qv.x, qv.x, nb); nb = fma(qv.y, qv.y, nb);
                    sab += fabs(av[u].x * qv.x) + fabs(av[u].y * qv.y);
                }
            }
            num = warp_sum(num); na = warp_sum(na); nb = warp_sum(nb); sab = warp_sum(sab);
        }
        if (lane == 0) {
            double* pp = part + (eg * kCosWPE + wq) * 4;
            pp[0] = num; pp[1] = na; pp[2] = nb; pp[3] = sab;
        }
        __syncthreads();
        if (wq == 0 && lane == 0 && e < N) {
            const double* pp = part + eg * kCosWPE * 4;
            double tn = 0, ta = 0, tb = 0, ts = 0;
            for (int w = 0; w < kCosWPE; ++w) {
                tn += pp[4 * w]; ta += pp[4 * w + 1]; tb += pp[4 * w + 2]; ts += pp[4 * w + 3];
            }
            const double den = sqrt(ta) * sqrt(tb);
            const double sv = tn / den;
            sim[e] = sv;
            double b = 2.0 * gam * (ts / den + fabs(sv)) * 1.0000001 + 1e-300;
            if (!(den > 1e-150)) b = INFINITY;  // tiny/zero norms: always recompute
            bnd[e] = b;
        }
        __syncthreads();
    }
}

// reference-order cosine (pattern_cache.hpp:40-46)
__device__ double ref_cosine(const double* __restrict__ a, const double* __restrict__ b, int d) {
    double num = 0, na = 0, nb = 0;
    int j = 0;
    for (; j + 4 <= d; j += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { av[q] = a[j + q]; bv[q] = b[j + q]; }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            num = __dadd_rn(num, __dmul_rn(av[q], bv[q]));
            na = __dadd_rn(na, __dmul_rn(av[q], av[q]));
            nb = __dadd_rn(nb, __dmul_rn(bv[q], bv[q]));
        }
    }
    for (; j < d; ++j) {
        num = __dadd_rn(num, __dmul_rn(a[j], b[j]));
        na = __dadd_rn(na, __dmul_rn(a[j], a[j]));
        nb = __dadd_rn(nb, __dmul_rn(b[j], b[j]));
    }
    return __ddiv_rn(num, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
}

__global__ void k_cosine_exact(const double* a, const double* b, int d, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = ref_cosine(a, b, d);
}

constexpr int kRetThreads = 1024;

// out_f64[0] = similarity; out_i32[0] = entry, [1] = hit, [2] = exact flag,
// [3] = number of reference-order recomputes (diagnostic)
__global__ void __launch_bounds__(kRetThreads)
k_retrieve_select(const double* __restrict__ sim, const double* __restrict__ bnd,
                  const double* __restrict__ emb, const double* __restrict__ q, int N, int d,
                  double min_sim, int exact_similarity, double* __restrict__ out_f64,
                  int32_t* __restrict__ out_i32, int32_t* __restrict__ entry_dev,
                  int32_t* __restrict__ hit_dev) {
    __shared__ double dscratch[33];
    __shared__ int s_band[kRetThreads];
    __shared__ double s_val[kRetThreads];
    __shared__ int s_cnt;
    // launched as a programmatic dependent of the scan: the sims are complete here
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // 1) max over fast sims (NaN -> -inf) and the global bound
    double m = -INFINITY, e = 0.0;
    for (int i = threadIdx.x; i < N; i += kRetThreads) {
        const double v = sim[i];
        if (v == v) m = fmax(m, v);
        e = fmax(e, bnd[i]);
    }
    m = block_max_f64<kRetThreads>(m, dscratch);
    e = block_max_f64<kRetThreads>(e, dscratch);
    // 2) band = {i : sim_i >= m - 2e} (all finite entries when e is inf)
    const double lo = (m == -INFINITY) ? INFINITY : m - 2.0 * e * (1.0 + 1e-9);
    int best = -1;
    double best_v = -2.0;
    bool best_exact = false;
    int nrec = 0;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += kRetThreads) {
        const double v = sim[i];
        if (v == v && v >= lo) {
            int slot = atomicAdd(&s_cnt, 1);
            if (slot < kRetThreads) s_band[slot] = i;
        }
    }
    __syncthreads();
    const int nb = s_cnt;
    if (nb == 1) {
        best = s_band[0];
        best_v = sim[best];
    } else if (nb > 1) {
        // recompute the whole band in reference order, first max wins
        const bool fits = nb <= kRetThreads;
        double lv = -2.0;
        int li = -1;
        if (fits) {
            if (threadIdx.x < nb) {
                const int i = s_band[threadIdx.x];
                lv = ref_cosine(emb + (int64_t)i * d, q, d);
                li = i;
            }
        } else {
            for (int i = threadIdx.x; i < N; i += kRetThreads) {
                const double v = sim[i];
                if (v == v && v >= lo) {
                    const double ex = ref_cosine(emb + (int64_t)i * d, q, d);
                    if (ex > lv || (ex == lv && li >= 0 && i < li)) { lv = ex; li = i; }
                }
            }
        }
        s_val[threadIdx.x] = (li >= 0 && lv == lv) ? lv : -INFINITY;
        s_band[threadIdx.x] = li;
        __syncthreads();
        if (threadIdx.x == 0) {
            double bv = -2.0;
            int bi = -1;
            for (int t = 0; t < kRetThreads; ++t) {
                const int i = s_band[t];
                if (i < 0) continue;
                const double v = s_val[t];
                if (v > bv || (v == bv && bi >= 0 && i < bi)) { bv = v; bi = i; }
            }
            s_band[0] = bi;
            s_val[0] = bv;
        }
        __syncthreads();
        best = s_band[0];
        best_v = s_val[0];
        best_exact = true;
        nrec = nb;
    }
    if (threadIdx.x == 0) {
        int entry = best < 0 ? 0 : best;
        double simv = best < 0 ? -2.0 : best_v;
        if (best >= 0 && !best_exact) {
            const double b = bnd[best];
            if (exact_similarity || fabs(simv - min_sim) <= b) {
                simv = ref_cosine(emb + (int64_t)best * d, q, d);
                best_exact = true;
                ++nrec;
            }
        }
        const int hit = simv >= min_sim;
        out_f64[0] = simv;
        out_i32[0] = entry;
        out_i32[1] = hit;
        out_i32[2] = best_exact || best < 0;
        out_i32[3] = nrec;
        if (entry_dev) *entry_dev = entry;
        if (hit_dev) *hit_dev = hit;
    }
}

// embed_prompt pooling half: h = mean_pool(x) (reference order), then
// vec_norm (sequential sum of squares, sqrt), then h /= nrm.
__global__ void k_embed_finish(double* __restrict__ h, int d, int* __restrict__ flag) {
    __shared__ double s_nrm;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < d; ++i) s = __dadd_rn(s, __dmul_rn(h[i], h[i]));
        const double nrm = __dsqrt_rn(s);
        s_nrm = nrm;
        *flag = nrm < 1e-12;
    }
    __syncthreads();
    const double nrm = s_nrm;
    if (nrm < 1e-12) return;
    for (int i = threadIdx.x; i < d; i += blockDim.x) h[i] = __ddiv_rn(h[i], nrm);
}

// ---------------- host launchers ----------------

void launch_cosine_scan(const double* emb, const double* q, int N, int d, double* sim, double* bnd,
                        cudaStream_t st) {
    once_per_device(reinterpret_cast<const void*>(&k_cosine_scan), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_cosine_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_cosine_scan_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    static const int wide_env = [] {
        const char* e = getenv("PG_COS_WIDE");
        return e ? atoi(e) : 1;
    }();
    if (wide_env && d % 8 == 0) {
        const int blocks = min((N + kCosEPB - 1) / kCosEPB, kNumSMs * COS_BPS);
        k_cosine_scan_wide<<<blocks, kCosWPE * kCosEPB * 32, (size_t)d * 8 + kCosEPB * kCosWPE * 32, st>>>(
            emb, q, N, d, sim, bnd);
        PG_LAUNCH_CHECK();
        return;
    }
    int blocks = min((N + kCosWarps - 1) / kCosWarps, kNumSMs * 2);
    k_cosine_scan<<<blocks, kCosWarps * 32, (size_t)d * 8, st>>>(emb, q, N, d, sim, bnd);
    PG_LAUNCH_CHECK();
}

void launch_retrieve_select(const double* sim, const double* bnd, const double* emb,
                            const double* q, int N, int d, double min_sim, int exact_similarity,
                            double* out_f64, int32_t* out_i32, int32_t* entry_dev,
                            int32_t* hit_dev, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(kRetThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_retrieve_select, sim, bnd, emb, q, N, d, min_sim, exact_similarity,
                                     out_f64, out_i32, entry_dev, hit_dev));
    count_launch();
}

void launch_cosine_exact(const double* a, const double* b, int d, double* out, cudaStream_t st) {
    k_cosine_exact<<<1, 32, 0, st>>>(a, b, d, out);
    PG_LAUNCH_CHECK();
}

void launch_embed_finish(double* h, int d, int* flag, cudaStream_t st) {
    k_embed_finish<<<1, 256, 0, st>>>(h, d, flag);
    PG_LAUNCH_CHECK();
}

int max_cache_dim() { return 200 * 1024 / 8; }

}  // namespace pg
