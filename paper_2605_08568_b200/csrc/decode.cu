// decode.cu -- K4/K6: single-launch decode chain for the rank-expert layer
// (T = 1 token): y = A_S (B_S^T x), one or more linears per phase sharing x
// (build_plan's fused_B / batched_A groups, exec_engine.hpp:46-68), with the
// MLP's silu(gate)*up (toy_lm.hpp:250-257) as a stage-2 epilogue feeding the
// next phase (down_proj).
//
// One persistent cooperative kernel, one CTA per SM, warp-specialised:
//   * warp 15 (one elected thread) is the TMA producer: it walks this CTA's
//     share of every weight row the chain reads -- stage-1 B^T rows of its slot
//     range, then stage-2 A rows of its output-row range, phase by phase --
//     and streams them with cp.async.bulk into a shared-memory ring
//     (full/empty mbarriers).  Weight rows never depend on activations, so the
//     producer keeps HBM busy straight through the grid barriers;
//   * warps 0-14 consume chunks in order: stage 1 dots B^T rows with x (in
//     smem) and publishes z; a grid barrier; z into smem; stage 2 dots A_S rows
//     with z and writes y (or act = silu(gate)*up for the MLP, then phase 1).
// Roofline: HBM-bound, algorithmic bytes = sum_l K_l (m_l + n_l) * dtype.
// Deterministic: fixed reduction orders (warp trees) and fixed CTA ranges.
#include <algorithm>

#include "chain.cuh"
#ifndef CHAIN_RELAXED_POLL
#define CHAIN_RELAXED_POLL 1
#endif

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

// ---- shared-memory tables ----
struct LinS {
    const char* bt;
    const char* a;
    const uint8_t* mask;  // run0 activity (nullable)
    void* z;
    void* y;
    long long ldb_b, lda_b;  // row strides (bytes)
    int run0, run1_start, run1, nslots;
    int n, m;
    int s0, s1;  // this CTA's stage-1 slot range
    int i0, i1;  // this CTA's stage-2 row range
    int pad[2];
};
static_assert(sizeof(LinS) <= kLinSBytes, "LinS table entry");
struct Desc {
    int seg, lin, count, gidx, last;
    int ids[kMaxChunkItems];
    int pad[11];
};
static_assert(sizeof(Desc) == 128, "Desc layout");

// ---- PTX helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// one LDS.128 (the compiler otherwise splits int4 views of bf16 data into
// four 4-way-conflicted LDS.32)
__device__ __forceinline__ int4 lds128(const void* p) {
    int4 r;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(smem_u32(p)));
    return r;
}
__device__ __forceinline__ float4 lds128f(const void* p) {
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(smem_u32(p)));
    return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// streamed-once weights: evict-first in L2 so they do not displace the exchange words
__device__ __forceinline__ void bulk_g2s_ef(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ void consumer_sync() {  // named barrier over the 15 consumer warps
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define STAMP(k) \
    if (P.dbg && threadIdx.x == 0) P.dbg[blockIdx.x * 16 + (k)] = gtimer()

__device__ __forceinline__ unsigned long long xget(const unsigned long long* p);
// Grid-wide barrier among consumer warps (the producer never blocks on it).
// Monotone counter: generation g completes when the count reaches (g+1)*G.
// The CTA barrier orders every consumer's z/act stores before thread 0's
// release-add (release is cumulative), and the acquire poll orders the
// subsequent reads -- no MEMBAR.GPU, which would also wait for the SM's
// in-flight bulk copies.
__device__ __forceinline__ void grid_sync_consumers(unsigned long long* bar) {
    consumer_sync();
    if (threadIdx.x == 0) {
        unsigned long long old;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
#if CHAIN_RELAXED_POLL
        while (xget(bar) < target) {
        }
        (void)ld_acquire(bar);
#else
        while (ld_acquire(bar) < target) {
        }
#endif
    }
    consumer_sync();
}

// ---- z exchange: tagged 64-bit words {payload (low 32), launch tag (high 32)},
// one relaxed gpu-scope store each, polled by the readers until the tag
// matches.  No fence -- a release would compile to MEMBAR.GPU, which waits
// for the SM's in-flight bulk copies (the whole ring).
__device__ __forceinline__ void xput(unsigned long long* p, uint32_t payload, uint32_t tag) {
    const unsigned long long v = ((unsigned long long)tag << 32) | payload;
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long xget(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <typename A>
__device__ __forceinline__ void xput_acc(unsigned long long* zx, int s, A v, uint32_t tag) {
    if constexpr (sizeof(A) == 4) {
        xput(zx + s, __float_as_uint(v), tag);
    } else {
        const unsigned long long b = (unsigned long long)__double_as_longlong(v);
        xput(zx + 2 * s, (uint32_t)b, tag);
        xput(zx + 2 * s + 1, (uint32_t)(b >> 32), tag);
    }
}

// Copy `count` elements global -> shared with every thread's loads issued
// before any store (one latency instead of one per loop trip).
template <typename T, int B>
__device__ __forceinline__ void stage_batched(T* dst, const T* __restrict__ src, int count, int tid, int nthr) {
    for (int base = 0; base < count; base += B * nthr) {
        T v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int e = base + u * nthr + tid;
            if (e < count) v[u] = __ldcg(src + e);  // L2: x may be another CTA's output of this launch
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int e = base + u * nthr + tid;
            if (e < count) dst[e] = v[u];
        }
    }
}

// z value t of 16-byte weight vector v: bf16 uses the two-plane layout (see
// the z staging), f32/f64 the plain one; the compiler fuses these into
// vector LDS.
template <int V, typename A>
__device__ __forceinline__ A zv(const A* z, int pl, int v, int t) {
    if constexpr (V == 8) return t < 4 ? z[v * 4 + t] : z[pl + v * 4 + (t - 4)];
    else return z[v * V + t];
}

// acc += dot(16-byte weight vector v, matching z values), z loads as 16-byte LDS
template <typename W, typename A>
__device__ __forceinline__ A zdot(const int4& wraw, const A* z, int pl, int v, A acc) {
    constexpr int V = CVec<W>::n;
    A wv[V];
    cunpack<W, A>(wraw, wv);
    if constexpr (V == 8) {
        const float4 lo = lds128f(z + v * 4);
        const float4 hi = lds128f(z + pl + v * 4);
        acc = fma(wv[0], lo.x, acc); acc = fma(wv[1], lo.y, acc);
        acc = fma(wv[2], lo.z, acc); acc = fma(wv[3], lo.w, acc);
        acc = fma(wv[4], hi.x, acc); acc = fma(wv[5], hi.y, acc);
        acc = fma(wv[6], hi.z, acc); acc = fma(wv[7], hi.w, acc);
    } else if constexpr (V == 4) {
        const float4 q = lds128f(z + v * 4);
        acc = fma(wv[0], q.x, acc); acc = fma(wv[1], q.y, acc);
        acc = fma(wv[2], q.z, acc); acc = fma(wv[3], q.w, acc);
    } else {
        const double2 q = *reinterpret_cast<const double2*>(z + v * 2);
        acc = fma(wv[0], q.x, acc); acc = fma(wv[1], q.y, acc);
    }
    return acc;
}


// ---- bf16 fast paths: f32x2 FMAs (sm_100 FFMA2) on bf16 pairs, every load of
// a row issued before the math, no per-vector branches (a vector past the row
// re-reads vector 0 and is zeroed by a select).
__device__ __forceinline__ void ffma2(float2& d, const float2& a, const float2& b) {
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n mov.b64 rd, {%0, %1};\n"
        " fma.rn.f32x2 rd, ra, rb, rd;\n mov.b64 {%0, %1}, rd;\n}"
        : "+f"(d.x), "+f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
}
__device__ __forceinline__ float2 bf2(uint32_t h) {  // bf16 pair -> (lo, hi) f32
    return make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u));
}
constexpr int kRowJ = 5;  // 16-byte vectors per lane per batch of a stage-2 row
// stage 2: A_S row (bf16, nv vectors) . z (f32, two-plane smem layout)
__device__ __forceinline__ float row_dot_bf16(const int4* r, int nv, const float* z, int pl, int lane) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
    for (int v0 = 0; v0 < nv; v0 += 32 * kRowJ) {
        int4 w[kRowJ];
        float4 zl[kRowJ], zh[kRowJ];
#pragma unroll
        for (int j = 0; j < kRowJ; ++j) {
            const int v = v0 + 32 * j + lane;
            const bool ok = v < nv;
            const int vv = ok ? v : 0;
            const int4 t = lds128(r + vv);
            w[j] = ok ? t : make_int4(0, 0, 0, 0);
            zl[j] = lds128f(z + vv * 4);
            zh[j] = lds128f(z + pl + vv * 4);
        }
#pragma unroll
        for (int j = 0; j < kRowJ; ++j) {
            ffma2(a0, bf2((uint32_t)w[j].x), make_float2(zl[j].x, zl[j].y));
            ffma2(a1, bf2((uint32_t)w[j].y), make_float2(zl[j].z, zl[j].w));
            ffma2(a0, bf2((uint32_t)w[j].z), make_float2(zh[j].x, zh[j].y));
            ffma2(a1, bf2((uint32_t)w[j].w), make_float2(zh[j].z, zh[j].w));
        }
    }
    return (a0.x + a0.y) + (a1.x + a1.y);
}
// stage 2 with z in registers: zr[j] = the 8 z values of vector lane + 32 j
// (zero past the row), loaded once per phase; only the weights come from smem.
struct ZReg {
    float2 p[kRowJ][4];
};
__device__ __forceinline__ void zreg_load(ZReg& zr, const float* z, int pl, int nv, int lane) {
#pragma unroll
    for (int j = 0; j < kRowJ; ++j) {
        const int v = 32 * j + lane;
        const bool ok = v < nv;
        const float4 lo = lds128f(z + (ok ? v : 0) * 4), hi = lds128f(z + pl + (ok ? v : 0) * 4);
        zr.p[j][0] = ok ? make_float2(lo.x, lo.y) : make_float2(0.f, 0.f);
        zr.p[j][1] = ok ? make_float2(lo.z, lo.w) : make_float2(0.f, 0.f);
        zr.p[j][2] = ok ? make_float2(hi.x, hi.y) : make_float2(0.f, 0.f);
        zr.p[j][3] = ok ? make_float2(hi.z, hi.w) : make_float2(0.f, 0.f);
    }
}
__device__ __forceinline__ float row_dot_zreg(const int4* r, int nv, const ZReg& zr, int lane) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
    int4 w[kRowJ];
#pragma unroll
    for (int j = 0; j < kRowJ; ++j) w[j] = lds128(r + min(32 * j + lane, nv - 1));  // z is 0 past the row
#pragma unroll
    for (int j = 0; j < kRowJ; ++j) {
        ffma2(a0, bf2((uint32_t)w[j].x), zr.p[j][0]);
        ffma2(a1, bf2((uint32_t)w[j].y), zr.p[j][1]);
        ffma2(a0, bf2((uint32_t)w[j].z), zr.p[j][2]);
        ffma2(a1, bf2((uint32_t)w[j].w), zr.p[j][3]);
    }
    return (a0.x + a0.y) + (a1.x + a1.y);
}
// stage 1: B^T row (bf16, nv vectors) . x (bf16 smem)
__device__ __forceinline__ float row_dot_x_bf16(const int4* r, const int4* x, int nv, int lane) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll 4
    for (int v = lane; v < nv; v += 32) {
        const int4 w = lds128(r + v), xx = lds128(x + v);
        ffma2(a0, bf2((uint32_t)w.x), bf2((uint32_t)xx.x));
        ffma2(a1, bf2((uint32_t)w.y), bf2((uint32_t)xx.y));
        ffma2(a0, bf2((uint32_t)w.z), bf2((uint32_t)xx.z));
        ffma2(a1, bf2((uint32_t)w.w), bf2((uint32_t)xx.w));
    }
    return (a0.x + a0.y) + (a1.x + a1.y);
}

__device__ __forceinline__ bool slot_on(const LinS& L, int s) {
    return s >= L.run0 || L.mask == nullptr || L.mask[s] != 0;
}
__device__ __forceinline__ int slot_row(const LinS& L, int s) {
    return s < L.run0 ? s : L.run1_start + (s - L.run0);
}

// ---------------------------------------------------------------- producer
template <typename W>
__device__ void chain_producer(const ChainParams& P, const LinS* lins, Desc* descs, uint64_t* full,
                               uint64_t* empty, unsigned char* ring, int nst) {
    constexpr int es = sizeof(W);
    const int CH = P.chunk_bytes;
    int k = 0;
    int throttle_left = -1;  // chunks still allowed before the z exchange completes (-1: unlimited)
    int zphase = 0;
    uint64_t* zbar = empty + kRingStages + 1;
    unsigned uses = 0;      // parity of the next empty-wait per stage (bit k)
    unsigned used_once = 0;
    int gidx = 0;
    int c_used = 0, c_cnt = 0;
    Desc* d = nullptr;
    auto open = [&](int seg, int lin) {
        if (throttle_left == 0) {  // hold the stream until the consumers finished the z exchange
            mbar_wait(smem_u32(zbar), (uint32_t)(zphase & 1));
            ++zphase;
            throttle_left = -1;
        } else if (throttle_left > 0) {
            --throttle_left;
        }
        if (used_once & (1u << k)) {
            mbar_wait(smem_u32(&empty[k]), (uses >> k) & 1u);
            uses ^= 1u << k;
        }
        used_once |= 1u << k;
        d = &descs[k];
        d->seg = seg;
        d->lin = lin;
        d->gidx = gidx;
        d->last = 0;
        c_used = 0;
        c_cnt = 0;
    };
    auto close = [&](int last) {
        d->count = c_cnt;
        d->last = last;
        gidx += c_cnt;
        mbar_arrive(smem_u32(&full[k]));
        k = (k + 1 == nst) ? 0 : k + 1;
        d = nullptr;
    };
    uint64_t pol = 0;
    if (P.l2hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    auto copy = [&](const char* src, int bytes) {
        const uint32_t bar = smem_u32(&full[k]);
        mbar_expect_tx(bar, (uint32_t)bytes);
        if (P.l2hint) bulk_g2s_ef(smem_u32(ring + (size_t)k * CH + c_used), src, (uint32_t)bytes, bar, pol);
        else bulk_g2s(smem_u32(ring + (size_t)k * CH + c_used), src, (uint32_t)bytes, bar);
        c_used += bytes;
    };
    for (int ph = 0; ph < P.nphase; ++ph) {
        const ChainPhase& Q = P.ph[ph];
        const LinS* L = lins + ph * kMaxLin;
        if (P.throttle >= 0 && zphase < ph) {  // absorb the previous phase's exchange signal
            mbar_wait(smem_u32(zbar), (uint32_t)(zphase & 1));
            ++zphase;
            throttle_left = -1;
        }
        // ---- stage-1 segment: B^T rows of this CTA's slot range.  Slots of one
        // run are consecutive B^T rows, so a chunk is ONE bulk copy; masked slots
        // ride along and are zeroed when z is staged.
        for (int l = 0; l < Q.nlin; ++l) {
            const int rb = (int)L[l].ldb_b;
            const int per = max(1, min(kMaxChunkItems, CH / rb));
            int s = L[l].s0;
            while (s < L[l].s1) {
                // stay inside one run so the rows are contiguous
                const int run_end = s < L[l].run0 ? min(L[l].s1, L[l].run0) : L[l].s1;
                const int cnt = min(per, run_end - s);
                open(2 * ph, l);
                for (int q = 0; q < cnt; ++q) d->ids[q] = s + q;
                c_cnt = cnt;
                copy(L[l].bt + (size_t)slot_row(L[l], s) * L[l].ldb_b, cnt * rb);
                s += cnt;
                close(0);
            }
        }
        open(2 * ph, 0);
        close(1);
        if (P.throttle >= 0) throttle_left = P.throttle;
        // ---- stage-2 segment: A_S rows of this CTA's row range.  Single-run
        // arenas (lda == nslots) are contiguous: one copy per matrix per chunk.
        if (Q.epilogue == 1) {
            const int rb0 = L[0].nslots * es, rb1 = L[1].nslots * es;
            const bool contig = L[0].run1 == 0 && L[1].run1 == 0 && L[0].lda_b == rb0 && L[1].lda_b == rb1;
            const int per = max(1, min(kMaxChunkItems, CH / (rb0 + rb1)));
            for (int i = L[0].i0; i < L[0].i1;) {
                const int cnt = min(per, L[0].i1 - i);
                open(2 * ph + 1, 0);
                for (int q = 0; q < cnt; ++q) d->ids[q] = i + q;
                c_cnt = cnt;
                for (int l = 0; l < 2; ++l) {
                    if (contig) {
                        copy(L[l].a + (size_t)i * L[l].lda_b, cnt * (l ? rb1 : rb0));
                    } else {
                        for (int q = 0; q < cnt; ++q) {
                            const char* row = L[l].a + (size_t)(i + q) * L[l].lda_b;
                            copy(row, L[l].run0 * es);
                            if (L[l].run1) copy(row + (size_t)L[l].run1_start * es, L[l].run1 * es);
                        }
                    }
                }
                i += cnt;
                close(0);
            }
        } else {
            for (int l = 0; l < Q.nlin; ++l) {
                const int rb = L[l].nslots * es;
                const bool contig = L[l].run1 == 0 && L[l].lda_b == rb;
                const int per = max(1, min(kMaxChunkItems, CH / rb));
                for (int i = L[l].i0; i < L[l].i1;) {
                    const int cnt = min(per, L[l].i1 - i);
                    open(2 * ph + 1, l);
                    for (int q = 0; q < cnt; ++q) d->ids[q] = i + q;
                    c_cnt = cnt;
                    if (contig) {
                        copy(L[l].a + (size_t)i * L[l].lda_b, cnt * rb);
                    } else {
                        for (int q = 0; q < cnt; ++q) {
                            const char* row = L[l].a + (size_t)(i + q) * L[l].lda_b;
                            copy(row, L[l].run0 * es);
                            if (L[l].run1) copy(row + (size_t)L[l].run1_start * es, L[l].run1 * es);
                        }
                    }
                    i += cnt;
                    close(0);
                }
            }
        }
        open(2 * ph + 1, 0);
        close(1);
    }
}

// ---------------------------------------------------------------- kernel
template <typename W, bool PEER>
__global__ void __launch_bounds__(kChainThreads, 1) k_chain(const __grid_constant__ ChainParams P) {
    using A = typename Acc<W>::type;
    constexpr int V = CVec<W>::n;
    constexpr int es = sizeof(W);
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;

    // ---- carve shared memory: [tables][x][z][descs][full][empty][ring]
    LinS* lins = reinterpret_cast<LinS*>(smem);
    const int tb = P.tab_bytes;
    W* xs = reinterpret_cast<W*>(smem + tb);
    A* zs = reinterpret_cast<A*>(smem + tb + P.xs_bytes);
    Desc* descs = reinterpret_cast<Desc*>(smem + tb + P.xs_bytes + P.zs_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(descs + kRingStages);
    uint64_t* empty = full + kRingStages;
    const size_t ring_off = ((size_t)(reinterpret_cast<unsigned char*>(empty + kRingStages) - smem) + 16 + 127) & ~size_t(127);
    unsigned char* ring = smem + ring_off;
    const int nst = (int)min((size_t)min(P.max_stages, kRingStages), (size_t)(227 * 1024 - ring_off) / (size_t)P.chunk_bytes);

    STAMP(0);
    for (int t = threadIdx.x; t < P.nphase * kMaxLin; t += blockDim.x) {
        const int ph = t / kMaxLin, l = t % kMaxLin;
        const ChainPhase& Q = P.ph[ph];
        if (l < Q.nlin) {
            const ChainLin& C = Q.lin[l];
            const SlotMap sm = resolve(C.sm);
            LinS& L = lins[t];
            L.bt = static_cast<const char*>(C.bt);
            L.a = static_cast<const char*>(C.a);
            L.mask = sm.mask;
            L.z = C.zpart;
            L.y = C.y;
            L.ldb_b = C.ldb * es;
            L.lda_b = C.lda * es;
            L.run0 = sm.run0_len;
            L.run1_start = sm.run1_start;
            L.run1 = sm.run1_len;
            L.nslots = sm.run0_len + sm.run1_len;
            L.n = C.n;
            L.m = C.m;
            L.s0 = (int)((long long)L.nslots * c / G);
            L.s1 = (int)((long long)L.nslots * (c + 1) / G);
            L.i0 = (int)((long long)C.m * c / G);
            L.i1 = (int)((long long)C.m * (c + 1) / G);
        }
    }
    if (threadIdx.x == 0) {
        for (int k = 0; k < kRingStages; ++k) {
            mbar_init(smem_u32(&full[k]), 1);
            mbar_init(smem_u32(&empty[k]), kConsumerWarps);
        }
        mbar_init(smem_u32(empty + kRingStages + 1), 1);  // z exchange done (producer throttle)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // launch tag: every CTA adds 1 to the workspace's epoch counter BEFORE it
    // lets dependents launch (the __syncthreads below orders the ticket before
    // launch_dependents), so every CTA of launch N holds its ticket before any
    // CTA of launch N+1 can be scheduled -- even on SMs this grid leaves free --
    // and old / G is the launch index.
    unsigned long long epoch_old = 0;
    if (threadIdx.x == 0) epoch_old = atomicAdd(P.epoch, 1ull);
    __syncthreads();

    // Let the next launch in the stream start its prologue / weight stream as
    // soon as SMs free up (programmatic dependent launch).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == kConsumerWarps) {
        // weights are immutable: the producer never waits on the previous grid
        if (lane == 0) {
            chain_producer<W>(P, lins, descs, full, empty, ring, nst);
            if (P.dbg) P.dbg[blockIdx.x * 16 + 12] = gtimer();  // every copy issued
        }
        return;
    }
    uint32_t* tag_s = reinterpret_cast<uint32_t*>(empty + kRingStages);
    // consumers read x and write z / act / y: wait for the previous grid
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- consumers
    const int tid = threadIdx.x, nct = kConsumerWarps * 32;
    int k = 0;
    unsigned par = 0;  // full-barrier parity per stage
    for (int ph = 0; ph < P.nphase; ++ph) {
        const ChainPhase& Q = P.ph[ph];
        const LinS* L = lins + ph * kMaxLin;
        const int nlin = Q.nlin;
        // stage x (phase 0: the input; phase 1: act, complete after the barrier)
        {
            const int n = L[0].n;
            const int nbytes = n * es;
            stage_batched<int4, 4>(reinterpret_cast<int4*>(xs), reinterpret_cast<const int4*>(Q.x), nbytes / 16,
                                   tid, nct);
            for (int e = (nbytes / 16) * 16 / es + tid; e < n; e += nct) xs[e] = __ldcg(static_cast<const W*>(Q.x) + e);
            for (int e = n + tid; e < (n + V - 1) / V * V; e += nct) xs[e] = W(0);
        }
        if (ph == 0) STAMP(6);  // x staged (thread 0), before the launch tag is needed
        if (ph == 0 && threadIdx.x == 0) *tag_s = (uint32_t)(epoch_old / (unsigned long long)G) + 1u;
        consumer_sync();
        const uint32_t tag = *tag_s;
        if (ph < 2) STAMP(ph * 6 + 1);
        // ---- stage 1: z_s = B^T[s] . x
        for (;;) {
            mbar_wait(smem_u32(&full[k]), (par >> k) & 1u);
            par ^= 1u << k;
            const Desc& D = descs[k];
            const int cnt = D.count, g0 = D.gidx, last = D.last, l = D.lin;
            if (cnt && ph == 1) STAMP(14);  // phase-1 stage-1 data seen (last write wins)
            if (cnt) {
                const LinS& Ls = L[l];
                const int rb = (int)Ls.ldb_b;
                const int nv = (Ls.n + V - 1) / V;
                const unsigned char* base = ring + (size_t)k * P.chunk_bytes;
                for (int q = (warp - g0 % kConsumerWarps + kConsumerWarps) % kConsumerWarps; q < cnt;
                     q += kConsumerWarps) {
                    const int4* rv = reinterpret_cast<const int4*>(base + (size_t)q * rb);
                    const int4* xv = reinterpret_cast<const int4*>(xs);
                    A acc = A(0);
                    if constexpr (sizeof(W) == 2) {
                        acc = row_dot_x_bf16(rv, xv, nv, lane);
                    } else {
#pragma unroll 4
                        for (int v = lane; v < nv; v += 32) {
                            A wv[V], xx[V];
                            cunpack<W, A>(lds128(rv + v), wv);
                            cunpack<W, A>(lds128(xv + v), xx);
#pragma unroll
                            for (int t = 0; t < V; ++t) acc = fma(wv[t], xx[t], acc);
                        }
                    }
                    acc = warp_sum(acc);
                    if (lane == 0) {
                        const int s = D.ids[q];  // masked slots publish 0 (exec_engine.hpp:221-223)
                        const A zv = slot_on(Ls, s) ? acc : A(0);
                        if (P.ztag) xput_acc<A>(static_cast<unsigned long long*>(Ls.z), s, zv, tag);
                        else static_cast<A*>(Ls.z)[s] = zv;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[k]));
            k = (k + 1 == nst) ? 0 : k + 1;
            if (last) break;
        }
        if (ph < 2) STAMP(ph * 6 + 2);
        if (!P.ztag) grid_sync_consumers(P.bar);
        if (ph < 2) STAMP(ph * 6 + 3);
        // ---- z into shared memory (inactive slots -> 0)
        int zoff[kMaxLin] = {0, 0, 0};
        {
            int o = 0;
#pragma unroll
            for (int l = 0; l < kMaxLin; ++l) {  // unrolled: zoff stays in registers
                if (l >= nlin) break;
                zoff[l] = o;
                const unsigned long long* zx = static_cast<const unsigned long long*>(L[l].z);
                const int ns = L[l].nslots;
                // every thread's polls of a batch are issued before any is
                // checked (one L2 round trip per batch, not one per slot)
                constexpr int B = 8;
                constexpr int zw = sizeof(A) / 4;
                const int pl = (ns + 7) / 8 * 4;
                for (int base = 0; base < ns; base += B * nct) {
                    unsigned long long v[B][zw];
#pragma unroll
                    for (int u = 0; u < B; ++u) {
                        const int s = base + u * nct + tid;
                        if (P.ztag) {
#pragma unroll
                            for (int h = 0; h < zw; ++h) v[u][h] = s < ns ? xget(zx + (size_t)s * zw + h) : 0ull;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < B; ++u) {
                        const int s = base + u * nct + tid;
                        if (s < ns) {
                            A val;
                            if (P.ztag) {
                                unsigned long long w[zw];
#pragma unroll
                                for (int h = 0; h < zw; ++h) {
                                    w[h] = v[u][h];
                                    while ((uint32_t)(w[h] >> 32) != tag) w[h] = xget(zx + (size_t)s * zw + h);
                                }
                                if constexpr (zw == 1) val = __uint_as_float((uint32_t)w[0]);
                                else val = __longlong_as_double((long long)((w[1] << 32) | (w[0] & 0xffffffffull)));
                            } else {
                                val = reinterpret_cast<const A*>(zx)[s];  // published before the barrier
                            }
                            // bf16: two planes (slots 0-3 / 4-7 of every 8) so each
                            // lane's 8 z-values are two conflict-free 16-byte loads
                            if constexpr (V == 8) zs[o + (s >> 3) * 4 + (s & 3) + ((s & 4) ? pl : 0)] = val;
                            else zs[o + s] = val;
                        }
                    }
                }
                o += (V == 8) ? 2 * pl : ((ns + 3) & ~3);
            }
        }
        consumer_sync();
        if (ph < 2) STAMP(ph * 6 + 4);
        if (P.throttle >= 0 && threadIdx.x == 0) mbar_arrive(smem_u32(empty + kRingStages + 1));
        // bf16 with <= 2 linears of <= 32 * 8 * kRowJ slots: z into registers
        ZReg zr0, zr1;
        bool zreg = false;
        if constexpr (sizeof(W) == 2) {
            zreg = nlin <= 2;
            for (int l = 0; l < nlin; ++l) zreg = zreg && L[l].nslots <= 32 * V * kRowJ;
            if (zreg) {
                const int ns0 = L[0].nslots;
                zreg_load(zr0, zs + zoff[0], (ns0 + 7) / 8 * 4, ns0 / V, lane);
                if (nlin > 1) {
                    const int ns1 = L[1].nslots;
                    zreg_load(zr1, zs + zoff[1], (ns1 + 7) / 8 * 4, ns1 / V, lane);
                }
            }
        }
        // ---- stage 2: y_i = A_S[i] . z
        for (int c2 = 0;; ++c2) {
            mbar_wait(smem_u32(&full[k]), (par >> k) & 1u);
            par ^= 1u << k;
            const Desc& D = descs[k];
            const int cnt = D.count, g0 = D.gidx, last = D.last, l = D.lin;
            if (P.nphase == 1) {  // single-phase launches: stage-2 data arrival (first / last chunk)
                if (c2 == 0) STAMP(7);
                STAMP(8);
            }
            if (cnt) {
                const unsigned char* base = ring + (size_t)k * P.chunk_bytes;
                for (int q = (warp - g0 % kConsumerWarps + kConsumerWarps) % kConsumerWarps; q < cnt;
                     q += kConsumerWarps) {
                    const int i = D.ids[q];
                    if (Q.epilogue == 1) {
                        const int ns0 = L[0].nslots, ns1 = L[1].nslots;
                        const int4* r0 = reinterpret_cast<const int4*>(base + (size_t)q * ns0 * es);
                        const int4* r1 = reinterpret_cast<const int4*>(base + (size_t)cnt * ns0 * es + (size_t)q * ns1 * es);
                        const A* z0 = zs + zoff[0];
                        const A* z1 = zs + zoff[1];
                        const int pl0 = (ns0 + 7) / 8 * 4, pl1 = (ns1 + 7) / 8 * 4;
                        A a0 = A(0), a1 = A(0);
                        if constexpr (sizeof(W) == 2) {
                            if (zreg) {
                                a0 = row_dot_zreg(r0, ns0 / V, zr0, lane);
                                a1 = row_dot_zreg(r1, ns1 / V, zr1, lane);
                            } else {
                                a0 = row_dot_bf16(r0, ns0 / V, z0, pl0, lane);
                                a1 = row_dot_bf16(r1, ns1 / V, z1, pl1, lane);
                            }
                        } else {
                            for (int v = lane; v < ns0 / V; v += 32) {
                                a0 = zdot<W, A>(lds128(r0 + v), z0, pl0, v, a0);
                            }
                            for (int v = lane; v < ns1 / V; v += 32) {
                                a1 = zdot<W, A>(lds128(r1 + v), z1, pl1, v, a1);
                            }
                        }
                        a0 = warp_sum(a0);
                        a1 = warp_sum(a1);
                        if constexpr (PEER) {  // push the up/gate partials to every rank; act after the sum below
                            if (lane < P.npeer) {
                                unsigned long long* rb = P.peer_recv[lane] +
                                                         ((size_t)(tag & 1u) * P.npeer + P.prank) * P.peer_words;
                                xput(rb + i, __float_as_uint((float)a0), tag);
                                xput(rb + L[0].m + i, __float_as_uint((float)a1), tag);
                            }
                        } else if (lane == 0) {
                            W* act = static_cast<W*>(Q.act);
                            if constexpr (sizeof(W) == 2) {
                                const float up = (float)a0, g = (float)a1;
                                act[i] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * up);
                            } else {
                                act[i] = (W)(a1 / (A(1) + exp(-a1)) * a0);
                            }
                        }
                    } else {
                        const int ns = L[l].nslots;
                        const int4* r = reinterpret_cast<const int4*>(base + (size_t)q * ns * es);
                        // selects, not a dynamic index: keeps zoff in registers (no stack frame)
                        const A* z = zs + (l == 0 ? zoff[0] : (l == 1 ? zoff[1] : zoff[2]));
                        const int pl = (ns + 7) / 8 * 4;
                        A acc = A(0);
                        if constexpr (sizeof(W) == 2) {
                            if (zreg) acc = l == 0 ? row_dot_zreg(r, ns / V, zr0, lane) : row_dot_zreg(r, ns / V, zr1, lane);
                            else acc = row_dot_bf16(r, ns / V, z, pl, lane);
                        } else {
                            for (int v = lane; v < ns / V; v += 32) {
                                acc = zdot<W, A>(lds128(r + v), z, pl, v, acc);
                            }
                        }
                        acc = warp_sum(acc);
                        if constexpr (PEER) {  // push the partial to every rank (peer memory), reduce below
                            if (lane < P.npeer) {
                                xput(P.peer_recv[lane] + ((size_t)(tag & 1u) * P.npeer + P.prank) * P.peer_words +
                                         P.peer_last_off + i,
                                     __float_as_uint((float)acc), tag);
                            }
                        } else if (lane == 0) {
                            void* y = L[l].y;
                            if (Q.ydt == PG_F32) static_cast<float*>(y)[i] = (float)acc;
                            else if (Q.ydt == PG_F64) static_cast<double*>(y)[i] = (double)acc;
                            else static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn((float)acc);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[k]));
            k = (k + 1 == nst) ? 0 : k + 1;
            if (last) break;
        }
        if (ph < 2) STAMP(ph * 6 + 5);
        if constexpr (PEER) {
            if (Q.epilogue == 1) {
                // expert-sharded MLP block: this CTA's act rows from the ranks'
                // up/gate partials, summed in rank order (identical on every
                // rank), so every rank holds the whole act for its down shard
                const int m0 = L[0].m;
                const unsigned long long* mine = P.peer_recv[P.prank] + (size_t)(tag & 1u) * P.npeer * P.peer_words;
                W* act = static_cast<W*>(Q.act);
                for (int i = L[0].i0 + tid; i < L[0].i1; i += nct) {
                    float u = 0.f, g = 0.f;
                    for (int p = 0; p < P.npeer; ++p) {
                        unsigned long long wu = xget(mine + (size_t)p * P.peer_words + i);
                        unsigned long long wg = xget(mine + (size_t)p * P.peer_words + m0 + i);
                        while ((uint32_t)(wu >> 32) != tag) wu = xget(mine + (size_t)p * P.peer_words + i);
                        while ((uint32_t)(wg >> 32) != tag) wg = xget(mine + (size_t)p * P.peer_words + m0 + i);
                        u += __uint_as_float((uint32_t)wu);
                        g += __uint_as_float((uint32_t)wg);
                    }
                    if constexpr (sizeof(W) == 2) act[i] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * u);
                    else act[i] = (W)(g / (1.0f + expf(-g)) * u);
                }
            }
        }
        if (ph + 1 < P.nphase) grid_sync_consumers(P.bar);  // act complete before phase ph+1 reads it
    }
    if constexpr (PEER) {
        // this CTA's rows: the npeer partials from this rank's receive buffer,
        // summed in rank order (deterministic on every rank)
        const LinS& Lr = lins[(P.nphase - 1) * kMaxLin];
        const uint32_t tag = *tag_s;
        const unsigned long long* mine =
            P.peer_recv[P.prank] + (size_t)(tag & 1u) * P.npeer * P.peer_words + P.peer_last_off;
        for (int i = Lr.i0 + threadIdx.x; i < Lr.i1; i += kConsumerWarps * 32) {
            unsigned long long w[kMaxPeers];
#pragma unroll
            for (int p = 0; p < kMaxPeers; ++p) w[p] = p < P.npeer ? xget(mine + (size_t)p * P.peer_words + i) : 0ull;
            float v = 0.f;
#pragma unroll
            for (int p = 0; p < kMaxPeers; ++p) {
                if (p < P.npeer) {
                    while ((uint32_t)(w[p] >> 32) != tag) w[p] = xget(mine + (size_t)p * P.peer_words + i);
                    v += __uint_as_float((uint32_t)w[p]);
                }
            }
            const int ydt = P.ph[P.nphase - 1].ydt;
            if (ydt == PG_F32) static_cast<float*>(Lr.y)[i] = v;
            else if (ydt == PG_F64) static_cast<double*>(Lr.y)[i] = (double)v;
            else static_cast<__nv_bfloat16*>(Lr.y)[i] = __float2bfloat16_rn(v);
        }
    }
    STAMP(13);
}

int chain_grid() { return device_sms(); }

template <typename W, bool PEER>
static void launch_chain_t(const ChainParams& P, size_t smem, cudaStream_t st, int grid) {
    once_per_device(reinterpret_cast<const void*>(&k_chain<W, PEER>), [] {
        PG_CUDA_THROW(cudaFuncSetAttribute(k_chain<W, PEER>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid > 0 ? std::min(grid, chain_grid()) : chain_grid());
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    static const int coop = [] {
        const char* e = getenv("PG_CHAIN_COOP");
        return e ? atoi(e) : 1;
    }();
    static const int pdl = [] {
        const char* e = getenv("PG_CHAIN_PDL");
        return e ? atoi(e) : 1;
    }();
    cudaLaunchAttribute at[2];
    int na = 0;
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    if (pdl) {  // programmatic dependent launch: the producer may start streaming
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    PG_CUDA_THROW(cudaLaunchKernelEx(&cfg, k_chain<W, PEER>, P));
    count_launch();
}

void launch_chain(pg_dtype wdt, const ChainParams& P, size_t smem, cudaStream_t st, int grid) {
    // the peer-reduction variant is a separate instantiation so the hot MLP
    // kernel keeps its register budget
    if (P.npeer) {
        if (wdt == PG_F32) launch_chain_t<float, true>(P, smem, st, grid);
        else if (wdt == PG_BF16) launch_chain_t<__nv_bfloat16, true>(P, smem, st, grid);
        else throw Error{PG_INVALID_ARGUMENT, "decode chain: peer reduction needs bf16/f32"};
        return;
    }
    if (wdt == PG_F64) launch_chain_t<double, false>(P, smem, st, grid);
    else if (wdt == PG_F32) launch_chain_t<float, false>(P, smem, st, grid);
    else launch_chain_t<__nv_bfloat16, false>(P, smem, st, grid);
}

}  // namespace pg
