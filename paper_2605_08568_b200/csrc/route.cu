// route.cu -- K1: mean_pool -> score -> select_topk on sm_100a, bit-identical to
// the reference's router (include/parse/router.hpp:41-61,80-88).
//
// Roofline: the router GEMV streams theta (r x n f64, 8*r*n bytes per prompt
// batch) once -- HBM-bound.  mean_pool and the top-K are small.
//
// Exactness strategy (SURVEY.md §7 "Hard parts" 1):
//  * mean_pool is computed in the reference's order (one thread per feature,
//    sequential over tokens, __dadd_rn, one final __ddiv_rn) -- cheap.
//  * score runs as a fast warp-tree FMA GEMV that also accumulates
//    S_i = sum_j |theta_ij h_j|.  Both the reference's sequential dot and ours
//    are within gamma_{n+1} (S_i + |b_i|) of the exact value, so
//    |z_fast - z_ref| <= e_i := 4 (n+2) u (S_i + |b_i|) (+ denormal slack).
//  * select: L = K-th largest fast logit, e = max_i e_i.  Rows with
//    |z_i - L| > 2e are on the same side of the exact K-th value as in the
//    reference; rows inside the band are recomputed in reference order
//    (sequential __dmul_rn/__dadd_rn) unless the band is wholly selected.  The
//    final top-K over the mixed vector equals the reference's top-K, including
//    the lower-index tie rule (router.hpp:53-55) and ascending output (:57).
#include "block_utils.cuh"

namespace pg {

// ---------------- mean_pool (router.hpp:80-88) ----------------

// token-major x [Ttot, n]: one thread per (prompt, feature) sums its column in
// token order; loads run kPoolAhead tokens ahead of the (strictly sequential)
// fp64 additions so each thread keeps that many requests in flight.
constexpr int kPoolAhead = 32;
template <typename TX>
__global__ void __launch_bounds__(256) k_mean_pool_tm(const TX* __restrict__ x, int n,
                                                      const int64_t* __restrict__ offs, double* __restrict__ h) {
    const int p = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t t0 = offs[p], t1 = offs[p + 1];
    const TX* col = x + i;
    double s = 0.0;
    int64_t t = t0;
    for (; t + kPoolAhead <= t1; t += kPoolAhead) {
        TX v[kPoolAhead];
#pragma unroll
        for (int u = 0; u < kPoolAhead; ++u) v[u] = col[(t + u) * (int64_t)n];
#pragma unroll
        for (int u = 0; u < kPoolAhead; ++u) s = __dadd_rn(s, to_d(v[u]));
    }
    for (; t < t1; ++t) s = __dadd_rn(s, to_d(col[t * (int64_t)n]));
    h[(int64_t)p * n + i] = __ddiv_rn(s, (double)(t1 - t0));
}

// bf16, n even: two features per thread (one 32-bit load per token feeds two
// sequential chains); batches of kPoolAhead2 tokens are double-buffered in
// registers, so the next batch's loads are in flight while this one's strictly
// ordered fp64 additions run.
constexpr int kPoolAhead2 = 64;
__device__ __forceinline__ void pool_load(uint32_t (&v)[kPoolAhead2], const uint32_t* col, int64_t t, int64_t ld) {
#pragma unroll
    for (int u = 0; u < kPoolAhead2; ++u) v[u] = __ldg(col + (t + u) * ld);
}
__device__ __forceinline__ void pool_add(const uint32_t (&v)[kPoolAhead2], double& s0, double& s1) {
#pragma unroll
    for (int u = 0; u < kPoolAhead2; ++u) {
        s0 = __dadd_rn(s0, (double)__uint_as_float(v[u] << 16));
        s1 = __dadd_rn(s1, (double)__uint_as_float(v[u] & 0xffff0000u));
    }
}
__global__ void __launch_bounds__(128) k_mean_pool_tm_bf16x2(const __nv_bfloat16* __restrict__ x, int n,
                                                             const int64_t* __restrict__ offs,
                                                             double* __restrict__ h) {
    const int p = blockIdx.y;
    const int i2 = blockIdx.x * blockDim.x + threadIdx.x;  // feature pair
    if (2 * i2 >= n) return;
    const int64_t t0 = offs[p], t1 = offs[p + 1];
    const uint32_t* col = reinterpret_cast<const uint32_t*>(x) + i2;
    const int64_t ld = n / 2;
    double s0 = 0.0, s1 = 0.0;
    const int64_t nb = (t1 - t0) / kPoolAhead2;  // whole batches
    uint32_t va[kPoolAhead2], vb[kPoolAhead2];
    if (nb > 0) pool_load(va, col, t0, ld);
    for (int64_t b = 0; b < nb; b += 2) {
        if (b + 1 < nb) pool_load(vb, col, t0 + (b + 1) * kPoolAhead2, ld);
        pool_add(va, s0, s1);
        if (b + 1 >= nb) break;
        if (b + 2 < nb) pool_load(va, col, t0 + (b + 2) * kPoolAhead2, ld);
        pool_add(vb, s0, s1);
    }
    for (int64_t t = t0 + nb * kPoolAhead2; t < t1; ++t) {
        const uint32_t v = __ldg(col + t * ld);
        s0 = __dadd_rn(s0, (double)__uint_as_float(v << 16));
        s1 = __dadd_rn(s1, (double)__uint_as_float(v & 0xffff0000u));
    }
    const double T = (double)(t1 - t0);
    h[(int64_t)p * n + 2 * i2] = __ddiv_rn(s0, T);
    h[(int64_t)p * n + 2 * i2 + 1] = __ddiv_rn(s1, T);
}

// bf16, n % V == 0 (V = 4 or 8): V features per thread (one 8- or 16-byte
// load per token: a warp reads 256 / 512 contiguous bytes of each token row
// instead of 128), V strictly ordered fp64 chains per thread (the reference's
// token order per feature); B tokens per batch, double buffered
template <int V>
struct PoolVec;
template <>
struct PoolVec<4> {
    using T = uint2;
    __device__ static void words(const uint2& v, uint32_t (&w)[2]) { w[0] = v.x; w[1] = v.y; }
};
template <>
struct PoolVec<8> {
    using T = uint4;
    __device__ static void words(const uint4& v, uint32_t (&w)[4]) { w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w; }
};
template <int V>
__device__ __forceinline__ void poolv_add1(const typename PoolVec<V>::T& v, double (&s)[V]) {
    uint32_t w[V / 2];
    PoolVec<V>::words(v, w);
#pragma unroll
    for (int e = 0; e < V / 2; ++e) {
        s[2 * e] = __dadd_rn(s[2 * e], (double)__uint_as_float(w[e] << 16));
        s[2 * e + 1] = __dadd_rn(s[2 * e + 1], (double)__uint_as_float(w[e] & 0xffff0000u));
    }
}
template <int V, int B>
__global__ void __launch_bounds__(64) k_mean_pool_tm_bf16v(const __nv_bfloat16* __restrict__ x, int n,
                                                          const int64_t* __restrict__ offs, double* __restrict__ h) {
    using LT = typename PoolVec<V>::T;
    const int p = blockIdx.y;
    const int iv = blockIdx.x * blockDim.x + threadIdx.x;  // feature group
    if (V * iv >= n) return;
    const int64_t t0 = offs[p], t1 = offs[p + 1];
    const LT* col = reinterpret_cast<const LT*>(x) + iv;
    const int64_t ld = n / V;
    double s[V];
#pragma unroll
    for (int e = 0; e < V; ++e) s[e] = 0.0;
    const int64_t nb = (t1 - t0) / B;  // whole batches
    LT va[B], vb[B];
    auto load = [&](LT (&v)[B], int64_t t) {
#pragma unroll
        for (int u = 0; u < B; ++u) v[u] = __ldg(col + (t + u) * ld);
    };
    auto add = [&](const LT (&v)[B]) {
#pragma unroll
        for (int u = 0; u < B; ++u) poolv_add1<V>(v[u], s);
    };
    if (nb > 0) load(va, t0);
    for (int64_t b = 0; b < nb; b += 2) {
        if (b + 1 < nb) load(vb, t0 + (b + 1) * B);
        add(va);
        if (b + 1 >= nb) break;
        if (b + 2 < nb) load(va, t0 + (b + 2) * B);
        add(vb);
    }
    for (int64_t t = t0 + nb * B; t < t1; ++t) poolv_add1<V>(__ldg(col + t * ld), s);
    const double T = (double)(t1 - t0);
#pragma unroll
    for (int e = 0; e < V; ++e) h[(int64_t)p * n + V * iv + e] = __ddiv_rn(s[e], T);
}
#ifndef POOL_V
#define POOL_V 4
#endif
#ifndef POOL_B
#define POOL_B 16
#endif
#ifndef POOL_MIN_N
#define POOL_MIN_N 8192  // narrower rows keep the two-feature kernel (more warps in flight wins there)
#endif
#ifndef POOL_BLOCK
#define POOL_BLOCK 64
#endif

// feature-major x [n, Ttot]: each warp owns 32 rows; a 32x32 tile is read
// coalesced along tokens, then each lane sums its own row in token order.
template <typename TX>
__global__ void k_mean_pool_fm(const TX* __restrict__ x, int n, int64_t ttot,
                               const int64_t* __restrict__ offs, double* __restrict__ h) {
    __shared__ double tile[4][32][33];
    const int p = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = (blockIdx.x * 4 + w) * 32;
    if (row0 >= n) return;
    const int64_t t0 = offs[p], t1 = offs[p + 1];
    double s = 0.0;
    for (int64_t tc = t0; tc < t1; tc += 32) {
        const int cnt = (int)((t1 - tc) < 32 ? (t1 - tc) : 32);
        for (int rr = 0; rr < 32; ++rr) {
            const int row = row0 + rr;
            double v = 0.0;
            if (row < n && lane < cnt) v = to_d(x[(int64_t)row * ttot + tc + lane]);
            tile[w][rr][lane] = v;
        }
        __syncwarp();
        for (int c = 0; c < cnt; ++c) s = __dadd_rn(s, tile[w][lane][c]);
        __syncwarp();
    }
    const int row = row0 + lane;
    if (row < n) h[(int64_t)p * n + row] = __ddiv_rn(s, (double)(t1 - t0));
}

// ---------------- score (router.hpp:41-46) ----------------


// ||h_p||_2 per prompt (rounded; inflated where it is used)
__global__ void k_hnorm(const double* __restrict__ h, int n, double* __restrict__ out) {
    __shared__ double red[32];
    const double* hp = h + (int64_t)blockIdx.x * n;
    double s = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) s = fma(hp[j], hp[j], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) out[blockIdx.x] = sqrt(v);
    }
}

// fast: logits on the fp64 tensor cores (mma.m8n8k4.f64) plus a rigorous
// error bound.  A block = kScoreSlices warps on 8 theta rows x 16 prompts,
// warp s on the s-th slice of the reduction dimension; partial tiles are
// summed across slices in fixed order.  Any summation order of the n products
// is within gamma_{n+1} sum_j |theta_ij h_j| of the exact value (as is the
// reference's sequential dot), and by Cauchy-Schwarz sum_j |theta_ij h_j| <=
// ||theta_i|| ||h||, so
//   bnd_i = 4 (n+2) u (||theta_i|| ||h|| + |b_i|)   (x 1.0000001 for the
// rounding of the norms themselves) bounds |fast - reference|.
constexpr int kScoreSlices = 8;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(kScoreSlices * 32)
k_score_fast(const double* __restrict__ theta, const double* __restrict__ bias, int r, int n,
             const double* __restrict__ h, const double* __restrict__ hnorm, int P, double* __restrict__ z,
             double* __restrict__ bnd) {
    __shared__ double part[kScoreSlices][32][5];  // per lane: 2 tiles x 2 + row-norm partial
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = blockIdx.x * 8, p0 = blockIdx.y * 16;
    const int rr = lane >> 2, cc = lane & 3;  // fragment row (theta row / prompt), k lane
    const int row = min(row0 + rr, r - 1);
    const double* th = theta + (int64_t)row * n;
    const double* h0 = h + (int64_t)min(p0 + rr, P - 1) * n;
    const double* h1 = h + (int64_t)min(p0 + 8 + rr, P - 1) * n;
    // k slice of this warp, in groups of 8 (two k-steps per 16-byte load: the
    // k order inside a group is permuted identically for theta and h)
    const int ng = (n + 7) / 8;
    const int g0 = (int)((long long)ng * warp / kScoreSlices), g1 = (int)((long long)ng * (warp + 1) / kScoreSlices);
    double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0, nrm = 0.0;
    const bool vec = (n & 1) == 0;
#pragma unroll 4
    for (int gi = g0; gi < g1; ++gi) {
        const int k = gi * 8 + 2 * cc;
        double2 t, a, b;
        if (vec && k + 1 < n) {
            t = __ldg(reinterpret_cast<const double2*>(th + k));
            a = __ldg(reinterpret_cast<const double2*>(h0 + k));
            b = __ldg(reinterpret_cast<const double2*>(h1 + k));
        } else {
            t.x = k < n ? th[k] : 0.0;  t.y = k + 1 < n ? th[k + 1] : 0.0;
            a.x = k < n ? h0[k] : 0.0;  a.y = k + 1 < n ? h0[k + 1] : 0.0;
            b.x = k < n ? h1[k] : 0.0;  b.y = k + 1 < n ? h1[k + 1] : 0.0;
        }
        nrm = fma(t.y, t.y, fma(t.x, t.x, nrm));
        dmma(d00, d01, t.x, a.x);
        dmma(d10, d11, t.x, b.x);
        dmma(d00, d01, t.y, a.y);
        dmma(d10, d11, t.y, b.y);
    }
    // row-norm partial: the four k lanes of a row
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 2);
    part[warp][lane][0] = d00;
    part[warp][lane][1] = d01;
    part[warp][lane][2] = d10;
    part[warp][lane][3] = d11;
    part[warp][lane][4] = nrm;
    __syncthreads();
    if (threadIdx.x < 128) {  // (row i, prompt q) = (t / 16, t % 16)
        const int i = threadIdx.x >> 4, q = threadIdx.x & 15;
        // D fragment: lane L holds D[L >> 2][2 (L & 3) + {0, 1}] of tile q / 8
        const int L = i * 4 + ((q & 7) >> 1), e = (q >= 8 ? 2 : 0) + (q & 1);
        double acc = 0.0, nr = 0.0;
        for (int w = 0; w < kScoreSlices; ++w) {
            acc += part[w][L][e];
            nr += part[w][i * 4][4];
        }
        const int R = row0 + i, p = p0 + q;
        if (R < r && p < P) {
            const double gam = 4.0 * (double)(n + 2) * kU;
            const double tiny = 4.0 * (double)(n + 2) * 4.9406564584124654e-324;
            const double b = bias[R];
            z[(int64_t)p * r + R] = acc + b;
            if (bnd) bnd[(int64_t)p * r + R] = gam * (sqrt(nr) * hnorm[p] + fabs(b)) * 1.0000001 + tiny;
        }
    }
}

// Same as k_score_fast with two 8-row theta tiles per block and 16 k-slices:
// every h fragment load feeds both tiles (half the L2 traffic for h, which
// all blocks re-read), same occupancy.  Partial tiles summed in fixed slice
// order; the error bound argument is unchanged.
constexpr int kScoreSlices2 = 16;
__global__ void __launch_bounds__(kScoreSlices2 * 32)
k_score_fast2(const double* __restrict__ theta, const double* __restrict__ bias, int r, int n,
              const double* __restrict__ h, const double* __restrict__ hnorm, int P, double* __restrict__ z,
              double* __restrict__ bnd) {
    __shared__ double part[kScoreSlices2][32][12];  // per lane: 2 row tiles x (2 prompt tiles x 2) + 2 row-norm + 2 h-norm partials
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = blockIdx.x * 16, p0 = blockIdx.y * 16;
    const int rr = lane >> 2, cc = lane & 3;
    const double* th0 = theta + (int64_t)min(row0 + rr, r - 1) * n;
    const double* th1 = theta + (int64_t)min(row0 + 8 + rr, r - 1) * n;
    const double* h0 = h + (int64_t)min(p0 + rr, P - 1) * n;
    const double* h1 = h + (int64_t)min(p0 + 8 + rr, P - 1) * n;
    const int ng = (n + 7) / 8;
    const int g0 = (int)((long long)ng * warp / kScoreSlices2), g1 = (int)((long long)ng * (warp + 1) / kScoreSlices2);
    double d[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
    double nrm0 = 0.0, nrm1 = 0.0, hn0 = 0.0, hn1 = 0.0;
    const bool vec = (n & 1) == 0;
#pragma unroll 2
    for (int gi = g0; gi < g1; ++gi) {
        const int k = gi * 8 + 2 * cc;
        double2 t0, t1, a, b;
        if (vec && k + 1 < n) {
            t0 = __ldg(reinterpret_cast<const double2*>(th0 + k));
            t1 = __ldg(reinterpret_cast<const double2*>(th1 + k));
            a = __ldg(reinterpret_cast<const double2*>(h0 + k));
            b = __ldg(reinterpret_cast<const double2*>(h1 + k));
        } else {
            t0.x = k < n ? th0[k] : 0.0;  t0.y = k + 1 < n ? th0[k + 1] : 0.0;
            t1.x = k < n ? th1[k] : 0.0;  t1.y = k + 1 < n ? th1[k + 1] : 0.0;
            a.x = k < n ? h0[k] : 0.0;   a.y = k + 1 < n ? h0[k + 1] : 0.0;
            b.x = k < n ? h1[k] : 0.0;   b.y = k + 1 < n ? h1[k + 1] : 0.0;
        }
        nrm0 = fma(t0.y, t0.y, fma(t0.x, t0.x, nrm0));
        nrm1 = fma(t1.y, t1.y, fma(t1.x, t1.x, nrm1));
        hn0 = fma(a.y, a.y, fma(a.x, a.x, hn0));  // ||h|| of the block's prompts, fused (no k_hnorm pass)
        hn1 = fma(b.y, b.y, fma(b.x, b.x, hn1));
        dmma(d[0][0], d[0][1], t0.x, a.x);
        dmma(d[0][2], d[0][3], t0.x, b.x);
        dmma(d[1][0], d[1][1], t1.x, a.x);
        dmma(d[1][2], d[1][3], t1.x, b.x);
        dmma(d[0][0], d[0][1], t0.y, a.y);
        dmma(d[0][2], d[0][3], t0.y, b.y);
        dmma(d[1][0], d[1][1], t1.y, a.y);
        dmma(d[1][2], d[1][3], t1.y, b.y);
    }
    nrm0 += __shfl_xor_sync(0xffffffffu, nrm0, 1);
    nrm0 += __shfl_xor_sync(0xffffffffu, nrm0, 2);
    nrm1 += __shfl_xor_sync(0xffffffffu, nrm1, 1);
    nrm1 += __shfl_xor_sync(0xffffffffu, nrm1, 2);
    hn0 += __shfl_xor_sync(0xffffffffu, hn0, 1);
    hn0 += __shfl_xor_sync(0xffffffffu, hn0, 2);
    hn1 += __shfl_xor_sync(0xffffffffu, hn1, 1);
    hn1 += __shfl_xor_sync(0xffffffffu, hn1, 2);
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) part[warp][lane][t * 4 + e] = d[t][e];
    part[warp][lane][8] = nrm0;
    part[warp][lane][9] = nrm1;
    part[warp][lane][10] = hn0;
    part[warp][lane][11] = hn1;
    __syncthreads();
    if (threadIdx.x < 256) {  // (row i, prompt q) = (t / 16, t % 16), rows of both tiles
        const int i = threadIdx.x >> 4, q = threadIdx.x & 15;
        const int tile = i >> 3, ii = i & 7;
        const int L = ii * 4 + ((q & 7) >> 1), e = (q >= 8 ? 2 : 0) + (q & 1);
        double acc = 0.0, nr = 0.0, hn = 0.0;
        for (int w = 0; w < kScoreSlices2; ++w) {
            acc += part[w][L][tile * 4 + e];
            nr += part[w][ii * 4][8 + tile];
            hn += part[w][(q & 7) * 4][10 + (q >> 3)];
        }
        const int R = row0 + i, p = p0 + q;
        if (R < r && p < P) {
            const double gam = 4.0 * (double)(n + 2) * kU;
            const double tiny = 4.0 * (double)(n + 2) * 4.9406564584124654e-324;
            const double b = bias[R];
            z[(int64_t)p * r + R] = acc + b;
            // norms carry O(n u) relative rounding, far inside the 1e-7 inflation
            if (bnd) bnd[(int64_t)p * r + R] = gam * (sqrt(nr) * sqrt(hn) + fabs(b)) * 1.0000001 + tiny;
        }
    }
}

// reference order: dot (matrix.hpp:189-193) then + bias; one lane per row,
// theta tiles staged through shared memory so global reads stay coalesced.
__device__ __forceinline__ double ref_dot_row(const double* __restrict__ th,
                                              const double* __restrict__ hv, int n) {
    double s = 0.0;
    int j = 0;
    for (; j + 8 <= n; j += 8) {
        double a[8], b[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) { a[q] = th[j + q]; b[q] = hv[j + q]; }
#pragma unroll
        for (int q = 0; q < 8; ++q) s = __dadd_rn(s, __dmul_rn(a[q], b[q]));
    }
    for (; j < n; ++j) s = __dadd_rn(s, __dmul_rn(th[j], hv[j]));
    return s;
}

__global__ void k_score_exact(const double* __restrict__ theta, const double* __restrict__ bias,
                              int r, int n, const double* __restrict__ h, int P,
                              double* __restrict__ z) {
    __shared__ double tile[4][32][33];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = (blockIdx.x * 4 + w) * 32;
    const int p = blockIdx.y;
    if (row0 >= r) return;
    const double* hv = h + (int64_t)p * n;
    double s = 0.0;
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int cnt = min(32, n - j0);
        for (int rr = 0; rr < 32; ++rr) {
            const int row = row0 + rr;
            tile[w][rr][lane] = (row < r && lane < cnt) ? theta[(int64_t)row * n + j0 + lane] : 0.0;
        }
        __syncwarp();
        for (int c = 0; c < cnt; ++c) s = __dadd_rn(s, __dmul_rn(tile[w][lane][c], hv[j0 + c]));
        __syncwarp();
    }
    const int row = row0 + lane;
    if (row < r) z[(int64_t)p * r + row] = __dadd_rn(s, bias[row]);
}

// ---------------- select_topk (router.hpp:49-61) ----------------

constexpr int kSelThreads = 1024;

// Final exact top-K on zs (smem) with (value desc, index asc) order; writes
// ascending indices.  flags: r bytes smem.
__device__ void topk_emit(const double* zs, int r, int K, uint64_t tkey, int need_eq,
                          uint8_t* flags, int* scratch, uint32_t* out) {
    // per-thread contiguous chunk keeps index order for the tie scan
    const int per = (r + kSelThreads - 1) / kSelThreads;
    const int b0 = threadIdx.x * per, b1 = min(r, b0 + per);
    int eq = 0;
    for (int i = b0; i < b1; ++i) eq += (f64_key(zs[i]) == tkey);
    int tot;
    int eq_before = block_excl_scan<kSelThreads>(eq, scratch, &tot);
    int sel_cnt = 0;
    for (int i = b0; i < b1; ++i) {
        const uint64_t k = f64_key(zs[i]);
        bool s = k > tkey;
        if (k == tkey) {
            s = eq_before < need_eq;
            ++eq_before;
        }
        flags[i] = s;
        sel_cnt += s;
    }
    int pos = block_excl_scan<kSelThreads>(sel_cnt, scratch, &tot);
    for (int i = b0; i < b1; ++i)
        if (flags[i]) out[pos++] = (uint32_t)i;
}

// Plain top-K on given logits (pg_select_topk): pure comparisons, exact.
__global__ void __launch_bounds__(kSelThreads)
k_select_topk(const double* __restrict__ logits, int r, int K, uint32_t* __restrict__ sel) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* zs = reinterpret_cast<double*>(smem);
    uint8_t* flags = reinterpret_cast<uint8_t*>(zs + r);
    __shared__ int hist[256];
    __shared__ int selv[2];
    __shared__ int scratch[40];
    const int p = blockIdx.x;
    for (int i = threadIdx.x; i < r; i += kSelThreads) zs[i] = logits[(int64_t)p * r + i];
    __syncthreads();
    int need_eq;
    uint64_t tkey = radix_select_kth<kSelThreads>(zs, r, K, hist, selv, &need_eq);
    topk_emit(zs, r, K, tkey, need_eq, flags, scratch, sel + (int64_t)p * K);
}

// Routing select with the error-bounded band (see file header).
__global__ void __launch_bounds__(kSelThreads)
k_route_select(const double* __restrict__ zfast, const double* __restrict__ bnd,
               const double* __restrict__ theta, const double* __restrict__ bias,
               const double* __restrict__ h, int r, int n, int K, uint32_t* __restrict__ sel,
               double* __restrict__ logits_out, int* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* zs = reinterpret_cast<double*>(smem);
    int* band = reinterpret_cast<int*>(zs + r);
    uint8_t* flags = reinterpret_cast<uint8_t*>(band + r);
    __shared__ int hist[256];
    __shared__ int selv[2];
    __shared__ int scratch[40];
    __shared__ double dscratch[33];
    const int p = blockIdx.x;
    const double* zf = zfast + (int64_t)p * r;
    const double* bd = bnd + (int64_t)p * r;
    double emax = 0.0;
    for (int i = threadIdx.x; i < r; i += kSelThreads) {
        zs[i] = zf[i];
        emax = fmax(emax, bd[i]);
    }
    emax = block_max_f64<kSelThreads>(emax, dscratch);  // includes __syncthreads
    int need_eq;
    uint64_t tkey = radix_select_kth<kSelThreads>(zs, r, K, hist, selv, &need_eq);
    int recomputed = 0;
    if (emax > 0.0) {
        const double L = key_f64(tkey);
        const double e2 = 2.0 * emax * (1.0 + 1e-9);
        const double hi = L + e2, lo = L - e2;
        int g = 0, b = 0;
        for (int i = threadIdx.x; i < r; i += kSelThreads) {
            const double v = zs[i];
            g += v > hi;
            b += (v >= lo && v <= hi);
        }
        const int G = block_sum_int<kSelThreads>(g, scratch);
        const int B = block_sum_int<kSelThreads>(b, scratch);
        if (K - G != B) {
            // compact band rows that carry rounding uncertainty, recompute them
            int mine = 0;
            const int per = (r + kSelThreads - 1) / kSelThreads;
            const int b0 = threadIdx.x * per, b1 = min(r, b0 + per);
            for (int i = b0; i < b1; ++i) mine += (zs[i] >= lo && zs[i] <= hi && bd[i] > 0.0);
            int tot;
            int pos = block_excl_scan<kSelThreads>(mine, scratch, &tot);
            for (int i = b0; i < b1; ++i)
                if (zs[i] >= lo && zs[i] <= hi && bd[i] > 0.0) band[pos++] = i;
            __syncthreads();
            const double* hv = h + (int64_t)p * n;
            for (int q = threadIdx.x; q < tot; q += kSelThreads) {
                const int i = band[q];
                zs[i] = __dadd_rn(ref_dot_row(theta + (int64_t)i * n, hv, n), bias[i]);
            }
            recomputed = tot;
            __syncthreads();
            tkey = radix_select_kth<kSelThreads>(zs, r, K, hist, selv, &need_eq);
        }
    }
    topk_emit(zs, r, K, tkey, need_eq, flags, scratch, sel + (int64_t)p * K);
    if (logits_out)
        for (int i = threadIdx.x; i < r; i += kSelThreads) logits_out[(int64_t)p * r + i] = zs[i];
    if (stats && threadIdx.x == 0) stats[p] = recomputed;
}

// ---------------- host launchers ----------------

template <typename TX>
static void launch_mean_pool_t(const void* x, pg_layout lay, int n, int64_t ttot,
                               const int64_t* offs_dev, int P, double* h, cudaStream_t st) {
    static const int poolv = [] {  // 0: two features per thread (round-1 kernel)
        const char* e = getenv("PG_POOLV");
        return e ? atoi(e) : 1;
    }();
    if (poolv && n >= POOL_MIN_N && lay == PG_TOKEN_MAJOR && sizeof(TX) == 2 && n % POOL_V == 0 &&
        reinterpret_cast<uintptr_t>(x) % (2 * POOL_V) == 0) {
        dim3 g((n / POOL_V + POOL_BLOCK - 1) / POOL_BLOCK, P);
        k_mean_pool_tm_bf16v<POOL_V, POOL_B><<<g, POOL_BLOCK, 0, st>>>(static_cast<const __nv_bfloat16*>(x), n,
                                                                       offs_dev, h);
    } else if (lay == PG_TOKEN_MAJOR && sizeof(TX) == 2 && n % 2 == 0 && reinterpret_cast<uintptr_t>(x) % 4 == 0) {
        dim3 g((n / 2 + 127) / 128, P);
        k_mean_pool_tm_bf16x2<<<g, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(x), n, offs_dev, h);
    } else if (lay == PG_TOKEN_MAJOR) {
        dim3 g((n + 255) / 256, P);
        k_mean_pool_tm<TX><<<g, 256, 0, st>>>(static_cast<const TX*>(x), n, offs_dev, h);
    } else {
        dim3 g((n + 127) / 128, P);
        k_mean_pool_fm<TX><<<g, 128, 0, st>>>(static_cast<const TX*>(x), n, ttot, offs_dev, h);
    }
    PG_LAUNCH_CHECK();
}

void launch_mean_pool(const void* x, pg_dtype dt, pg_layout lay, int n, int64_t ttot,
                      const int64_t* offs_dev, int P, double* h, cudaStream_t st) {
    switch (dt) {
        case PG_F64: launch_mean_pool_t<double>(x, lay, n, ttot, offs_dev, P, h, st); break;
        case PG_F32: launch_mean_pool_t<float>(x, lay, n, ttot, offs_dev, P, h, st); break;
        default: launch_mean_pool_t<__nv_bfloat16>(x, lay, n, ttot, offs_dev, P, h, st); break;
    }
}

void launch_score(const double* theta, const double* bias, int r, int n, const double* h, int P,
                  double* z, double* bnd, int exact, cudaStream_t st, double* hnorm) {
    if (exact) {
        dim3 g((r + 127) / 128, P);
        k_score_exact<<<g, 128, 0, st>>>(theta, bias, r, n, h, P, z);
    } else {
        static const int v2 = [] {
            const char* e = getenv("PG_SCORE_V2");
            return e ? atoi(e) : 1;
        }();
        if (!v2) {  // hnorm: caller scratch of P doubles (v2 fuses the norm)
            k_hnorm<<<P, 256, 0, st>>>(h, n, hnorm);
            PG_LAUNCH_CHECK();
        }
        if (v2) {
            dim3 g((r + 15) / 16, (P + 15) / 16);
            k_score_fast2<<<g, kScoreSlices2 * 32, 0, st>>>(theta, bias, r, n, h, hnorm, P, z, bnd);
        } else {
            dim3 g((r + 7) / 8, (P + 15) / 16);
            k_score_fast<<<g, kScoreSlices * 32, 0, st>>>(theta, bias, r, n, h, hnorm, P, z, bnd);
        }
    }
    PG_LAUNCH_CHECK();
}

static size_t sel_smem(int r, bool band) {
    return (size_t)r * 8 + (band ? (size_t)r * 4 : 0) + (size_t)r + 16;
}

void select_smem_setup() {
    once_per_device(reinterpret_cast<const void*>(&k_select_topk), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_select_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_route_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
}

int max_select_rows() { return (200 * 1024 - 64) / 13; }

void launch_select_topk(const double* logits, int r, int P, int K, uint32_t* sel, cudaStream_t st) {
    select_smem_setup();
    k_select_topk<<<P, kSelThreads, sel_smem(r, false), st>>>(logits, r, K, sel);
    PG_LAUNCH_CHECK();
}

void launch_route_select(const double* zfast, const double* bnd, const double* theta,
                         const double* bias, const double* h, int r, int n, int K, int P,
                         uint32_t* sel, double* logits_out, int* stats, cudaStream_t st) {
    select_smem_setup();
    k_route_select<<<P, kSelThreads, sel_smem(r, true), st>>>(zfast, bnd, theta, bias, h, r, n, K,
                                                              sel, logits_out, stats);
    PG_LAUNCH_CHECK();
}

}  // namespace pg
