// values.cu -- K3 expert gather + K4 decode GEMV stages + SIMT GEMM fallback for
// the two-stage rank-expert contraction y = A_S (B_S^T x)
// (include/parse/rank_experts.hpp:52-72, exec_engine.hpp:169-252).
//
// Device layout: B^T is expert-major [r_store, n] so each
// selected expert's V-row is one contiguous n-vector; A is [m, r_store] (or a
// packed [m, ld] arena) so each output row's selected columns are one or two
// contiguous runs.  A "slot" is one selected expert; SlotMap maps slots to
// storage rows/columns (gather list, or <=2 aligned runs + an activity mask).
//
// Roofline: decode (T <= 8) is HBM-bound on the weight bytes
// dtype*(nslots*n + m*nslots); the SIMT GEMM is the fp32/f64 prefill path
// (FFMA/DFMA-bound), bf16 prefill goes to the tcgen05 kernel (umma.cu).
#include <algorithm>

#include "pg_common.cuh"

namespace pg {

template <typename W> struct Vec;
template <> struct Vec<double> { static constexpr int n = 2; };
template <> struct Vec<float> { static constexpr int n = 4; };
template <> struct Vec<__nv_bfloat16> { static constexpr int n = 8; };

__device__ __forceinline__ void unpack(const int4& v, double* o) {
    const double2 d = *reinterpret_cast<const double2*>(&v);
    o[0] = d.x; o[1] = d.y;
}
__device__ __forceinline__ void unpack(const int4& v, float* o) {
    const float4 f = *reinterpret_cast<const float4*>(&v);
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
}
__device__ __forceinline__ void unpack_bf16(const int4& v, float* o) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        o[2 * q] = f.x; o[2 * q + 1] = f.y;
    }
}
template <typename W, typename A>
__device__ __forceinline__ void unpack_vec(const int4& v, A* o) {
    if constexpr (sizeof(W) == 2) unpack_bf16(v, o);
    else unpack(v, o);
}
template <typename W, typename A> __device__ __forceinline__ A wval(W v) {
    if constexpr (sizeof(W) == 2) return __bfloat162float(v);
    else return (A)v;
}

__device__ __forceinline__ int slot_index(const SlotMap& sm, int s) {
    if (sm.idx) return sm.idx[s];
    return s < sm.run0_len ? s : sm.run1_start + (s - sm.run0_len);
}
__device__ __forceinline__ bool slot_active(const SlotMap& sm, int s) {
    if (sm.idx) return sm.idx[s] >= 0;
    if (s < sm.run0_len) return sm.mask == nullptr || sm.mask[s] != 0;
    return true;
}

// ---------------------------------------------------------------------------
// K3: expert gather (aggregate_layout's column copies, exec_engine.hpp:136-158)
// ---------------------------------------------------------------------------

// dst[j, :] = src[idx[j], :] (idx < 0 -> zeros); rows of `cols` elements.
template <typename W>
__global__ void k_gather_rows(const W* __restrict__ src, int64_t lds, const int32_t* __restrict__ idx,
                              int cnt, int cnt_pad, int cols, W* __restrict__ dst, int64_t ldd) {
    const int j = blockIdx.x;
    if (j >= cnt_pad) return;
    const int s = j < cnt ? idx[j] : -1;
    W* d = dst + (int64_t)j * ldd;
    if ((cols * sizeof(W)) % 16 == 0 && (lds * sizeof(W)) % 16 == 0 && (ldd * sizeof(W)) % 16 == 0) {
        const int nv = cols * sizeof(W) / 16;
        int4* dv = reinterpret_cast<int4*>(d);
        if (s < 0) {
            for (int v = threadIdx.x; v < nv; v += blockDim.x) dv[v] = make_int4(0, 0, 0, 0);
        } else {
            const int4* sv = reinterpret_cast<const int4*>(src + (int64_t)s * lds);
            for (int v = threadIdx.x; v < nv; v += blockDim.x) dv[v] = ld_stream(sv + v);
        }
    } else {
        for (int c = threadIdx.x; c < cols; c += blockDim.x)
            d[c] = s < 0 ? W(0) : src[(int64_t)s * lds + c];
    }
}

// dst[i, j] = src[i, idx[j]] for j < cnt, 0 for cnt <= j < cnt_pad.
template <typename W>
__global__ void k_gather_cols(const W* __restrict__ src, int64_t lds, const int32_t* __restrict__ idx,
                              int cnt, int cnt_pad, int m, W* __restrict__ dst, int64_t ldd) {
    const int lane = threadIdx.x & 31;
    for (int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < m;
         i += gridDim.x * (blockDim.x / 32)) {
        const W* s = src + (int64_t)i * lds;
        W* d = dst + (int64_t)i * ldd;
        for (int j = lane; j < cnt_pad; j += 32) {
            const int c = j < cnt ? idx[j] : -1;
            d[j] = c < 0 ? W(0) : s[c];
        }
    }
}

// K3 for routed batches (config-3 prefill): every prompt p of a batch packs its
// own K selected experts sel[p*k + j] (device, ascending -- the router's
// output, no host round trip) into contiguous zero-padded arenas
//   bt_out[p][j][:]  = B^T[sel_pj][:]          (rows; 16-byte vectors)
//   a_out [p][i][j]  = A[i][sel_pj]            (columns; A rows staged in smem)
// for j < kp (kp = k rounded up to 8; padding rows / columns are zero).
// Bytes: read B^T rows and A once per prompt-tile, write P * kp * (n + m) * 2.
__global__ void k_pack_rows_batched(const int4* __restrict__ src, int64_t lds16, const int32_t* __restrict__ sel,
                                    int k, int kp, int nv, int4* __restrict__ dst, int64_t ldd16) {
    const int j = blockIdx.x, p = blockIdx.y;
    int4* d = dst + ((int64_t)p * kp + j) * ldd16;
    if (j >= k) {
        for (int v = threadIdx.x; v < nv; v += blockDim.x) d[v] = make_int4(0, 0, 0, 0);
        return;
    }
    const int4* s = src + (int64_t)__ldg(sel + (int64_t)p * k + j) * lds16;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) d[v] = ld_stream(s + v);
}

#ifndef PACK_ROWS
#define PACK_ROWS 8
#endif
constexpr int kPackRows = PACK_ROWS;  // A rows staged per CTA (amortises each prompt's selection list)
// (measured: staging every prompt's ids at once instead of one prompt at a
// time was slower -- the random 2-byte shared-memory gathers bound the kernel)
__global__ void __launch_bounds__(256) k_pack_cols_batched(const uint16_t* __restrict__ src, int64_t lds, int r,
                                                           const int32_t* __restrict__ sel, int k, int kp, int P,
                                                           int m, uint16_t* __restrict__ dst) {
    extern __shared__ __align__(16) uint16_t arow[];  // [kPackRows][rs] A rows, then [kp] selection ids
    const int rs = (r + 7) / 8 * 8;
    int32_t* ssel = reinterpret_cast<int32_t*>(arow + kPackRows * rs);
    const int i0 = blockIdx.x * kPackRows;
    const int nrow = min(kPackRows, m - i0);
    for (int e = threadIdx.x; e < nrow * (rs / 8); e += blockDim.x) {
        const int rr = e / (rs / 8), c8 = e % (rs / 8);
        const uint16_t* srow = src + (int64_t)(i0 + rr) * lds;
        if ((lds % 8) == 0 && c8 * 8 + 8 <= r) {
            *reinterpret_cast<int4*>(arow + rr * rs + c8 * 8) = ld_stream(srow + c8 * 8);
        } else {
            for (int q = 0; q < 8; ++q) arow[rr * rs + c8 * 8 + q] = c8 * 8 + q < r ? srow[c8 * 8 + q] : 0;
        }
    }
    const int kv = kp / 8;
    for (int p = 0; p < P; ++p) {
        __syncthreads();  // rows staged / previous prompt's ids consumed
        for (int j = threadIdx.x; j < kp; j += blockDim.x) ssel[j] = j < k ? __ldg(sel + (int64_t)p * k + j) : -1;
        __syncthreads();
        uint16_t* dp = dst + ((int64_t)p * m + i0) * kp;  // this CTA's rows of prompt p: contiguous
        for (int e = threadIdx.x; e < nrow * kv; e += blockDim.x) {
            const int rr = e / kv, j8 = (e % kv) * 8;
            const uint16_t* ar = arow + rr * rs;
            const int4 sa = *reinterpret_cast<const int4*>(ssel + j8), sb = *reinterpret_cast<const int4*>(ssel + j8 + 4);
            const int id[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
            uint32_t v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = id[q] >= 0 ? ar[id[q]] : 0u;
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = v[2 * q] | (v[2 * q + 1] << 16);
            *reinterpret_cast<uint4*>(dp + (int64_t)rr * kp + j8) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

void launch_pack_selected(const void* bt, int64_t ldb, const void* a, int64_t lda, int r, int n, int m,
                          const int32_t* sel, int k, int P, void* bt_out, void* a_out, cudaStream_t st) {
    const int kp = (k + 7) / 8 * 8;
    if (P <= 0 || k <= 0) return;
    if (bt_out) {  // (null: the prefill gathers the B^T rows itself, pg_prefill_gathered)
        k_pack_rows_batched<<<dim3(kp, P), 128, 0, st>>>(static_cast<const int4*>(bt), ldb / 8, sel, k, kp,
                                                         (n + 7) / 8, static_cast<int4*>(bt_out), ldb / 8);
        PG_LAUNCH_CHECK();
    }
    const size_t smem = (size_t)kPackRows * ((r + 7) / 8 * 8) * 2 + (size_t)kp * 4;
    if (smem > 48 * 1024)
        PG_CUDA_THROW(cudaFuncSetAttribute(k_pack_cols_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_pack_cols_batched<<<(m + kPackRows - 1) / kPackRows, 256, smem, st>>>(
        static_cast<const uint16_t*>(a), lda, r, sel, k, kp, P, m, static_cast<uint16_t*>(a_out));
    PG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// K4 stage 1: z[s, c] = sum_j Bt[row(s), j] * x[c, j]   (one warp per slot)
// ---------------------------------------------------------------------------

template <typename W, int TM>
__global__ void __launch_bounds__(256)
k_stage1_gemv(const W* __restrict__ bt, int64_t ldb, SlotMap sm, int nslots, int n,
              const W* __restrict__ x, int fm, int T, typename Acc<W>::type* __restrict__ z) {
    using A = typename Acc<W>::type;
    constexpr int V = Vec<W>::n;
    extern __shared__ __align__(16) unsigned char smem[];
    sm = resolve(sm);
    nslots = sm.nslots();
    W* xs = reinterpret_cast<W*>(smem);  // [T][nx] token-major, row stride padded to 16 B
    const int nx = (n + V - 1) / V * V;
    const int nt = T * n;
    if (!fm || T == 1) {
        for (int e = threadIdx.x; e < nt; e += blockDim.x) {
            const int c = e / n, j = e - c * n;
            xs[c * nx + j] = x[e];
        }
    } else {
        for (int e = threadIdx.x; e < nt; e += blockDim.x) {
            const int j = e / T, c = e % T;  // x feature-major [n][T]
            xs[c * nx + j] = x[e];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x / 32;
    const int nvec = n / V;
    for (int s = blockIdx.x * warps + (threadIdx.x >> 5); s < nslots; s += gridDim.x * warps) {
        A acc[TM];
#pragma unroll
        for (int c = 0; c < TM; ++c) acc[c] = A(0);
        if (slot_active(sm, s)) {
            const W* row = bt + (int64_t)slot_index(sm, s) * ldb;
            const int4* rv = reinterpret_cast<const int4*>(row);
            int v = lane;
            for (; v + 96 < nvec; v += 128) {
                int4 w4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) w4[u] = ld_stream(rv + v + 32 * u);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    A wv[V];
                    unpack_vec<W>(w4[u], wv);
                    const int j0 = (v + 32 * u) * V;
#pragma unroll
                    for (int c = 0; c < TM; ++c) {
                        if (c < T) {
                            A xv[V];
                            unpack_vec<W>(*reinterpret_cast<const int4*>(xs + c * nx + j0), xv);
#pragma unroll
                            for (int q = 0; q < V; ++q) acc[c] = fma(wv[q], xv[q], acc[c]);
                        }
                    }
                }
            }
            for (; v < nvec; v += 32) {
                const int4 w4 = ld_stream(rv + v);
                A wv[V];
                unpack_vec<W>(w4, wv);
                const int j0 = v * V;
#pragma unroll
                for (int c = 0; c < TM; ++c) {
                    if (c < T) {
                        A xv[V];
                        unpack_vec<W>(*reinterpret_cast<const int4*>(xs + c * nx + j0), xv);
#pragma unroll
                        for (int q = 0; q < V; ++q) acc[c] = fma(wv[q], xv[q], acc[c]);
                    }
                }
            }
            for (int j = nvec * V + lane; j < n; j += 32) {  // tail (n % V != 0)
                const A wv = wval<W, A>(row[j]);
#pragma unroll
                for (int c = 0; c < TM; ++c)
                    if (c < T) acc[c] = fma(wv, wval<W, A>(xs[c * nx + j]), acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < TM; ++c) acc[c] = warp_sum(acc[c]);
        if (lane == 0)
            for (int c = 0; c < T && c < TM; ++c) z[(int64_t)s * T + c] = acc[c];
    }
}

// ---------------------------------------------------------------------------
// K4 stage 2: y[i, c] = sum_s A[i, col(s)] * z[s, c]   (one warp per row)
// ---------------------------------------------------------------------------

template <typename W, typename OutT, int TM, bool GATHER>
__global__ void __launch_bounds__(256)
k_stage2_gemv(const W* __restrict__ a, int64_t lda, SlotMap sm, int nslots, int m,
              const typename Acc<W>::type* __restrict__ z, int T, int fm_out,
              OutT* __restrict__ y) {
    using A = typename Acc<W>::type;
    constexpr int V = Vec<W>::n;
    extern __shared__ __align__(16) unsigned char smem[];
    A* zs = reinterpret_cast<A*>(smem);  // [nslots][T]
    sm = resolve(sm);
    nslots = sm.nslots();
    for (int e = threadIdx.x; e < nslots * T; e += blockDim.x) zs[e] = z[e];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x / 32;
    for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < m; i += gridDim.x * warps) {
        const W* row = a + (int64_t)i * lda;
        A acc[TM];
#pragma unroll
        for (int c = 0; c < TM; ++c) acc[c] = A(0);
        if constexpr (GATHER) {
            for (int s = lane; s < nslots; s += 32) {
                const int col = sm.idx[s];
                if (col < 0) continue;
                const A av = wval<W, A>(row[col]);
#pragma unroll
                for (int c = 0; c < TM; ++c)
                    if (c < T) acc[c] = fma(av, zs[s * T + c], acc[c]);
            }
        } else {
            // two aligned runs: slots [0, run0) at cols [0, run0), slots
            // [run0, run0+run1) at cols [run1_start, ...); lengths multiple of V
            const int nv0 = sm.run0_len / V, nv1 = sm.run1_len / V;
            const int nv = nv0 + nv1;
            for (int v0 = lane; v0 < nv; v0 += 128) {
                int4 w4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int v = v0 + 32 * u;
                    if (v < nv) {
                        const int col = v < nv0 ? v * V : sm.run1_start + (v - nv0) * V;
                        w4[u] = ld_stream(row + col);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int v = v0 + 32 * u;
                    if (v < nv) {
                        A wv[V];
                        unpack_vec<W>(w4[u], wv);
                        const int s0 = v * V;
#pragma unroll
                        for (int q = 0; q < V; ++q)
#pragma unroll
                            for (int c = 0; c < TM; ++c)
                                if (c < T) acc[c] = fma(wv[q], zs[(s0 + q) * T + c], acc[c]);
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < TM; ++c) acc[c] = warp_sum(acc[c]);
        if (lane == 0) {
            for (int c = 0; c < T && c < TM; ++c) {
                const int64_t o = fm_out ? (int64_t)i * T + c : (int64_t)c * m + i;
                if constexpr (sizeof(OutT) == 2) y[o] = __float2bfloat16_rn((float)acc[c]);
                else y[o] = (OutT)acc[c];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// SIMT GEMM: C[t, o] = sum_k P(t, k) Q(o, k), 64x64 tiles, 4x4 per thread,
// split-K over blockIdx.z with deterministic partials.
// ---------------------------------------------------------------------------

constexpr int GBM = 64, GBN = 64, GBK = 16;

template <typename W>
struct PX {  // stage-1 P operand: activations (token- or feature-major)
    const W* x; int64_t ldx; int fm; int T;
    __device__ __forceinline__ typename Acc<W>::type operator()(int t, int k) const {
        return wval<W, typename Acc<W>::type>(fm ? x[(int64_t)k * T + t] : x[(int64_t)t * ldx + k]);
    }
};
template <typename A>
struct PZ {  // stage-2 P operand: z [T, ldz] in accumulator precision
    const A* z; int64_t ldz;
    __device__ __forceinline__ A operator()(int t, int k) const { return z[(int64_t)t * ldz + k]; }
};
template <typename W>
struct QRows {  // stage-1 Q operand: Bt rows by slot
    const W* bt; int64_t ldb; SlotMap sm;
    __device__ __forceinline__ typename Acc<W>::type operator()(int o, int k) const {
        if (!slot_active(sm, o)) return 0;
        return wval<W, typename Acc<W>::type>(bt[(int64_t)slot_index(sm, o) * ldb + k]);
    }
};
template <typename W>
struct QCols {  // stage-2 Q operand: A row o, column of slot k
    const W* a; int64_t lda; SlotMap sm;
    __device__ __forceinline__ typename Acc<W>::type operator()(int o, int k) const {
        const int c = slot_index(sm, k);
        if (c < 0) return 0;
        return wval<W, typename Acc<W>::type>(a[(int64_t)o * lda + c]);
    }
};

template <typename A, typename PF, typename QF>
__global__ void __launch_bounds__(256)
k_gemm_nt(PF P, QF Q, int M, int N, int K, int k_per_split, A* __restrict__ part) {
    __shared__ A Ps[GBK][GBM + 4];
    __shared__ A Qs[GBK][GBN + 4];
    const int tid = threadIdx.x;
    const int tm = tid / 16, tn = tid % 16;
    const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
    const int kb = blockIdx.z * k_per_split, ke = min(K, kb + k_per_split);
    A acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = A(0);
    for (int k0 = kb; k0 < ke; k0 += GBK) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int e = tid + 256 * l;  // 1024 = 64 x 16
            const int r = e / GBK, kk = e % GBK;
            const int k = k0 + kk;
            Ps[kk][r] = (m0 + r < M && k < ke) ? P(m0 + r, k) : A(0);
            Qs[kk][r] = (n0 + r < N && k < ke) ? Q(n0 + r, k) : A(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GBK; ++kk) {
            A pv[4], qv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pv[i] = Ps[kk][tm * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) qv[j] = Qs[kk][tn * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(pv[i], qv[j], acc[i][j]);
        }
        __syncthreads();
    }
    A* out = part + (int64_t)blockIdx.z * M * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = m0 + tm * 4 + i;
        if (t >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int o = n0 + tn * 4 + j;
            if (o < N) out[(int64_t)t * N + o] = acc[i][j];
        }
    }
}

// sum split partials in split order, mask, convert, write in layout
template <typename A, typename OutT>
__global__ void k_gemm_epilogue(const A* __restrict__ part, int splits, int M, int N, SlotMap sm,
                                int use_mask, int fm_out, OutT* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)M * N) return;
    A s = part[e];
    for (int q = 1; q < splits; ++q) s += part[(int64_t)q * M * N + e];
    const int t = (int)(e / N), o = (int)(e % N);
    if (use_mask && !slot_active(sm, o)) s = A(0);
    const int64_t dst = fm_out ? (int64_t)o * M + t : e;
    if constexpr (sizeof(OutT) == 2) out[dst] = __float2bfloat16_rn((float)s);
    else out[dst] = (OutT)s;
}

// act = silu(gate) * up (toy_lm.hpp:250-257 glue for the MLP block)
template <typename In, typename OutT>
__global__ void k_silu_mul(const In* __restrict__ g, const In* __restrict__ u, size_t count,
                           OutT* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        const In gv = g[i];
        const In v = gv / (In(1) + exp(-gv)) * u[i];
        if constexpr (sizeof(OutT) == 2) out[i] = __float2bfloat16_rn((float)v);
        else out[i] = (OutT)v;
    }
}

// dst[c, r] = src[r, c] (32x32 smem tiles)
template <typename T>
__global__ void k_transpose(const T* __restrict__ src, int rows, int cols, T* __restrict__ dst) {
    __shared__ T tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = src[(int64_t)r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[(int64_t)c * rows + r] = tile[threadIdx.x][i];
    }
}

void launch_transpose(pg_dtype dt, const void* src, int rows, int cols, void* dst, cudaStream_t st) {
    dim3 g((cols + 31) / 32, (rows + 31) / 32), b(32, 8);
    if (dt == PG_F64) k_transpose<double><<<g, b, 0, st>>>(static_cast<const double*>(src), rows, cols, static_cast<double*>(dst));
    else if (dt == PG_F32) k_transpose<float><<<g, b, 0, st>>>(static_cast<const float*>(src), rows, cols, static_cast<float*>(dst));
    else k_transpose<__nv_bfloat16><<<g, b, 0, st>>>(static_cast<const __nv_bfloat16*>(src), rows, cols,
                                                     static_cast<__nv_bfloat16*>(dst));
    PG_LAUNCH_CHECK();
}

void launch_silu_mul(const void* g, const void* u, pg_dtype in_dt, size_t count, void* act,
                     pg_dtype act_dt, cudaStream_t st) {
    const int blocks = (int)std::min<size_t>((count + 255) / 256, kNumSMs * 4);
    if (in_dt == PG_F64) {
        if (act_dt != PG_F64) throw Error{PG_INVALID_ARGUMENT, "silu_mul: f64 inputs need f64 output"};
        k_silu_mul<double, double><<<blocks, 256, 0, st>>>(static_cast<const double*>(g),
            static_cast<const double*>(u), count, static_cast<double*>(act));
    } else if (act_dt == PG_BF16) {
        k_silu_mul<float, __nv_bfloat16><<<blocks, 256, 0, st>>>(static_cast<const float*>(g),
            static_cast<const float*>(u), count, static_cast<__nv_bfloat16*>(act));
    } else {
        k_silu_mul<float, float><<<blocks, 256, 0, st>>>(static_cast<const float*>(g),
            static_cast<const float*>(u), count, static_cast<float*>(act));
    }
    PG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

int decode_tmax(int T) { return T <= 1 ? 1 : T <= 2 ? 2 : T <= 4 ? 4 : T <= 8 ? 8 : 0; }

template <typename W>
void launch_gather_rows_t(const void* src, int64_t lds, const int32_t* idx, int cnt, int cnt_pad,
                          int cols, void* dst, int64_t ldd, cudaStream_t st) {
    if (cnt_pad == 0) return;
    k_gather_rows<W><<<cnt_pad, 128, 0, st>>>(static_cast<const W*>(src), lds, idx, cnt, cnt_pad,
                                              cols, static_cast<W*>(dst), ldd);
    PG_LAUNCH_CHECK();
}
template <typename W>
void launch_gather_cols_t(const void* src, int64_t lds, const int32_t* idx, int cnt, int cnt_pad,
                          int m, void* dst, int64_t ldd, cudaStream_t st) {
    if (cnt_pad == 0) return;
    int blocks = min((m + 7) / 8, kNumSMs * 8);
    k_gather_cols<W><<<blocks, 256, 0, st>>>(static_cast<const W*>(src), lds, idx, cnt, cnt_pad, m,
                                             static_cast<W*>(dst), ldd);
    PG_LAUNCH_CHECK();
}

void launch_gather_rows(pg_dtype dt, const void* src, int64_t lds, const int32_t* idx, int cnt,
                        int cnt_pad, int cols, void* dst, int64_t ldd, cudaStream_t st) {
    if (dt == PG_F64) launch_gather_rows_t<double>(src, lds, idx, cnt, cnt_pad, cols, dst, ldd, st);
    else if (dt == PG_F32) launch_gather_rows_t<float>(src, lds, idx, cnt, cnt_pad, cols, dst, ldd, st);
    else launch_gather_rows_t<__nv_bfloat16>(src, lds, idx, cnt, cnt_pad, cols, dst, ldd, st);
}
void launch_gather_cols(pg_dtype dt, const void* src, int64_t lds, const int32_t* idx, int cnt,
                        int cnt_pad, int m, void* dst, int64_t ldd, cudaStream_t st) {
    if (dt == PG_F64) launch_gather_cols_t<double>(src, lds, idx, cnt, cnt_pad, m, dst, ldd, st);
    else if (dt == PG_F32) launch_gather_cols_t<float>(src, lds, idx, cnt, cnt_pad, m, dst, ldd, st);
    else launch_gather_cols_t<__nv_bfloat16>(src, lds, idx, cnt, cnt_pad, m, dst, ldd, st);
}

template <typename W, int TM>
static void stage1_t(const W* bt, int64_t ldb, SlotMap sm, int nslots, int n, const W* x, int fm,
                     int T, typename Acc<W>::type* z, cudaStream_t st) {
    const size_t smem = (size_t)T * ((n + Vec<W>::n - 1) / Vec<W>::n * Vec<W>::n) * sizeof(W) + 16;
    once_per_device(reinterpret_cast<const void*>(&k_stage1_gemv<W, TM>), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_stage1_gemv<W, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    });
    const int blocks = min((nslots + 7) / 8, kNumSMs * 4);
    k_stage1_gemv<W, TM><<<blocks, 256, smem, st>>>(bt, ldb, sm, nslots, n, x, fm, T, z);
    PG_LAUNCH_CHECK();
}

template <typename W, typename OutT, int TM>
static void stage2_t(const W* a, int64_t lda, SlotMap sm, int nslots, int m,
                     const typename Acc<W>::type* z, int T, int fm_out, OutT* y, cudaStream_t st) {
    using A = typename Acc<W>::type;
    const size_t smem = (size_t)nslots * T * sizeof(A) + 16;
    once_per_device(reinterpret_cast<const void*>(&k_stage2_gemv<W, OutT, TM, true>), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_stage2_gemv<W, OutT, TM, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        PG_CUDA_THROW(cudaFuncSetAttribute(k_stage2_gemv<W, OutT, TM, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    });
    const int blocks = min((m + 7) / 8, kNumSMs * 4);
    if (sm.idx)
        k_stage2_gemv<W, OutT, TM, true><<<blocks, 256, smem, st>>>(a, lda, sm, nslots, m, z, T, fm_out, y);
    else
        k_stage2_gemv<W, OutT, TM, false><<<blocks, 256, smem, st>>>(a, lda, sm, nslots, m, z, T, fm_out, y);
    PG_LAUNCH_CHECK();
}

template <typename W, int TM>
static void decode_tm(const W* bt, int64_t ldb, const W* a, int64_t lda, SlotMap sm, int n, int m,
                      const W* x, int fm, int T, typename Acc<W>::type* z, void* y, pg_dtype ydt,
                      cudaStream_t st) {
    const int ns = sm.cap ? sm.cap : sm.nslots();
    stage1_t<W, TM>(bt, ldb, sm, ns, n, x, fm, T, z, st);
    if (ydt == PG_F32) stage2_t<W, float, TM>(a, lda, sm, ns, m, z, T, fm, static_cast<float*>(y), st);
    else if (ydt == PG_F64) stage2_t<W, double, TM>(a, lda, sm, ns, m, z, T, fm, static_cast<double*>(y), st);
    else stage2_t<W, __nv_bfloat16, TM>(a, lda, sm, ns, m, z, T, fm, static_cast<__nv_bfloat16*>(y), st);
}

// decode path (T <= 8): z workspace holds nslots*T accumulators
template <typename W>
static void decode_t(const void* bt, int64_t ldb, const void* a, int64_t lda, SlotMap sm, int n, int m,
                     const void* x, int fm, int T, void* z, void* y, pg_dtype ydt, cudaStream_t st) {
    using A = typename Acc<W>::type;
    const W* b_ = static_cast<const W*>(bt);
    const W* a_ = static_cast<const W*>(a);
    const W* x_ = static_cast<const W*>(x);
    A* z_ = static_cast<A*>(z);
    switch (decode_tmax(T)) {
        case 1: decode_tm<W, 1>(b_, ldb, a_, lda, sm, n, m, x_, fm, T, z_, y, ydt, st); break;
        case 2: decode_tm<W, 2>(b_, ldb, a_, lda, sm, n, m, x_, fm, T, z_, y, ydt, st); break;
        case 4: decode_tm<W, 4>(b_, ldb, a_, lda, sm, n, m, x_, fm, T, z_, y, ydt, st); break;
        default: decode_tm<W, 8>(b_, ldb, a_, lda, sm, n, m, x_, fm, T, z_, y, ydt, st); break;
    }
}

void launch_decode(pg_dtype wdt, const void* bt, int64_t ldb, const void* a, int64_t lda, SlotMap sm,
                   int n, int m, const void* x, int fm, int T, void* z, void* y, pg_dtype ydt,
                   cudaStream_t st) {
    if (wdt == PG_F64) decode_t<double>(bt, ldb, a, lda, sm, n, m, x, fm, T, z, y, ydt, st);
    else if (wdt == PG_F32) decode_t<float>(bt, ldb, a, lda, sm, n, m, x, fm, T, z, y, ydt, st);
    else decode_t<__nv_bfloat16>(bt, ldb, a, lda, sm, n, m, x, fm, T, z, y, ydt, st);
}

size_t decode_smem_need(pg_dtype wdt, int n, int nslots, int T) {
    const size_t xs = (size_t)T * (n + 8) * dtype_size(wdt);
    const size_t zs = (size_t)nslots * T * (wdt == PG_F64 ? 8 : 4);
    return xs > zs ? xs : zs;
}

static int pick_splits(int M, int N, int K) {
    const int tiles = ((M + GBM - 1) / GBM) * ((N + GBN - 1) / GBN);
    int s = 1;
    while (tiles * s < kNumSMs && K / (s * 2) >= 256) s *= 2;
    return s;
}

template <typename A, typename PF, typename QF>
static void gemm_run(PF P, QF Q, int M, int N, int K, A* part, int splits, cudaStream_t st) {
    int kps = (K + splits - 1) / splits;
    kps = (kps + GBK - 1) / GBK * GBK;
    dim3 g((N + GBN - 1) / GBN, (M + GBM - 1) / GBM, splits);
    k_gemm_nt<A, PF, QF><<<g, 256, 0, st>>>(P, Q, M, N, K, kps, part);
    PG_LAUNCH_CHECK();
}

template <typename A, typename OutT>
static void epi_run(const A* part, int splits, int M, int N, SlotMap sm, int use_mask, int fm_out,
                    OutT* out, cudaStream_t st) {
    const int64_t tot = (int64_t)M * N;
    k_gemm_epilogue<A, OutT><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(part, splits, M, N, sm,
                                                                           use_mask, fm_out, out);
    PG_LAUNCH_CHECK();
}

// SIMT two-stage path for T > 8.  ws must hold max(splits1*T*ns, T*ns +
// splits2*T*m) accumulators (see simt_ws_elems).
template <typename W>
static void simt_t(const void* bt, int64_t ldb, const void* a, int64_t lda, SlotMap sm, int n, int m,
                   const void* x, int fm, int T, void* ws, void* y, pg_dtype ydt, cudaStream_t st) {
    using A = typename Acc<W>::type;
    const int ns = sm.nslots();
    A* wsA = static_cast<A*>(ws);
    A* zbuf = wsA;                          // [T, ns]
    A* part = wsA + (int64_t)T * ns;        // partials
    const int s1 = pick_splits(T, ns, n);
    PX<W> px{static_cast<const W*>(x), (int64_t)n, fm, T};
    QRows<W> qr{static_cast<const W*>(bt), ldb, sm};
    gemm_run<A>(px, qr, T, ns, n, part, s1, st);
    epi_run<A, A>(part, s1, T, ns, sm, 1, 0, zbuf, st);
    const int s2 = pick_splits(T, m, ns);
    PZ<A> pz{zbuf, (int64_t)ns};
    QCols<W> qc{static_cast<const W*>(a), lda, sm};
    gemm_run<A>(pz, qc, T, m, ns, part, s2, st);
    if (ydt == PG_F32) epi_run<A, float>(part, s2, T, m, sm, 0, fm, static_cast<float*>(y), st);
    else if (ydt == PG_F64) epi_run<A, double>(part, s2, T, m, sm, 0, fm, static_cast<double*>(y), st);
    else epi_run<A, __nv_bfloat16>(part, s2, T, m, sm, 0, fm, static_cast<__nv_bfloat16*>(y), st);
}

size_t simt_ws_elems(int n, int m, int ns, int T) {
    const size_t s1 = pick_splits(T, ns, n), s2 = pick_splits(T, m, ns);
    const size_t a = s1 * (size_t)T * ns, b = s2 * (size_t)T * m;
    return (size_t)T * ns + (a > b ? a : b);
}

void launch_simt(pg_dtype wdt, const void* bt, int64_t ldb, const void* a, int64_t lda, SlotMap sm,
                 int n, int m, const void* x, int fm, int T, void* ws, void* y, pg_dtype ydt,
                 cudaStream_t st) {
    if (wdt == PG_F64) simt_t<double>(bt, ldb, a, lda, sm, n, m, x, fm, T, ws, y, ydt, st);
    else if (wdt == PG_F32) simt_t<float>(bt, ldb, a, lda, sm, n, m, x, fm, T, ws, y, ydt, st);
    else simt_t<__nv_bfloat16>(bt, ldb, a, lda, sm, n, m, x, fm, T, ws, y, ydt, st);
}

}  // namespace pg
