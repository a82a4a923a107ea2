/*
 * parse_oracle.c -- TEST INFRASTRUCTURE ONLY (see parse_oracle.h).
 *
 * CPU restatement of the reference hot path.  Every function cites the
 * reference line range it follows (paths relative to /root/reference/proj).
 * Loop orders and accumulation orders are kept exactly so results are
 * bit-identical to the reference when built with -O2 -ffp-contract=off.
 */
#include "parse_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- include/parse/rng.hpp:10-41 ---------------- */
uint64_t po_rng_next_u64(po_rng* r) {
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
double po_rng_uniform(po_rng* r) { return (double)(po_rng_next_u64(r) >> 11) * 0x1.0p-53; }
uint64_t po_rng_below(po_rng* r, uint64_t n) { return po_rng_next_u64(r) % n; }
double po_rng_gaussian(po_rng* r) {
    double u1 = po_rng_uniform(r);
    double u2 = po_rng_uniform(r);
    while (u1 <= 0) u1 = po_rng_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
po_rng po_rng_fork(const po_rng* r, uint64_t salt) {
    po_rng f;
    f.state = r->state ^ (salt * 0xd1342543de82ef95ULL + 0x2545f4914f6cdd1dULL);
    po_rng_next_u64(&f);
    return f;
}
void po_fill_gaussian(uint64_t seed, double* out, size_t count) {
    po_rng r = {seed};
    for (size_t i = 0; i < count; ++i) out[i] = po_rng_gaussian(&r);
}

/* ---------------- include/parse/factorize.hpp ---------------- */
size_t po_store_rank(size_t k, size_t r_max, double mult) { /* :86-89 */
    size_t want = (size_t)ceil(mult * (double)k);
    size_t hi = k > want ? k : want;
    return r_max < hi ? r_max : hi;
}
/* allocate_budgets (:135-195) for a single layer: every candidate costs m+n,
 * K grows from 1 while used + cost <= (1-ratio)*m*n, capped at r_max. */
size_t po_single_layer_k(size_t m, size_t n, double ratio) {
    const double budget = (1.0 - ratio) * ((double)m * (double)n);
    const double cost = (double)(m + n);
    const size_t r_max = m < n ? m : n;
    size_t k = 1;
    double used = cost;
    while (k < r_max && used + cost <= budget) {
        used += cost;
        ++k;
    }
    return k;
}

/* ---------------- include/parse/matrix.hpp:189-193 ---------------- */
static double seq_dot(const double* a, const double* b, size_t n) {
    double s = 0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* ---------------- include/parse/router.hpp ---------------- */
void po_mean_pool(const double* x, size_t n, size_t T, double* h) { /* :80-88 */
    for (size_t i = 0; i < n; ++i) {
        double s = 0;
        for (size_t t = 0; t < T; ++t) s += x[i * T + t];
        h[i] = s / (double)T;
    }
}

void po_score(const double* theta, const double* bias, size_t r, size_t n, const double* h,
              double* z) { /* :41-46 */
    for (size_t i = 0; i < r; ++i) z[i] = seq_dot(theta + i * n, h, n) + bias[i];
}

static const double* g_sort_keys;
/* stable_sort by logit descending == sort by (logit desc, index asc) */
static int cmp_desc_then_index(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    double va = g_sort_keys[a], vb = g_sort_keys[b];
    if (va > vb) return -1;
    if (vb > va) return 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static int cmp_u32(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

int po_select_topk(const double* logits, size_t r, size_t k, uint32_t* out) { /* :49-61 */
    if (k == 0 || k > r) return 1;
    uint32_t* idx = (uint32_t*)malloc(r * sizeof(uint32_t));
    for (size_t i = 0; i < r; ++i) idx[i] = (uint32_t)i;
    g_sort_keys = logits;
    qsort(idx, r, sizeof(uint32_t), cmp_desc_then_index);
    qsort(idx, k, sizeof(uint32_t), cmp_u32);
    memcpy(out, idx, k * sizeof(uint32_t));
    free(idx);
    return 0;
}

/* ---------------- include/parse/pattern_cache.hpp ---------------- */
double po_cosine(const double* a, const double* b, size_t d) { /* :38-47 */
    double num = 0, na = 0, nb = 0;
    for (size_t i = 0; i < d; ++i) {
        num += a[i] * b[i];
        na += a[i] * a[i];
        nb += b[i] * b[i];
    }
    return num / (sqrt(na) * sqrt(nb));
}

int po_retrieve(const double* emb, size_t n_entries, size_t d, double min_similarity,
                const double* query, po_retrieve_result* out) { /* :104-117 */
    if (n_entries == 0) return 3;
    double best = -2.0;
    size_t entry = 0;
    for (size_t i = 0; i < n_entries; ++i) {
        const double sim = po_cosine(emb + i * d, query, d);
        if (sim > best) {
            best = sim;
            entry = i;
        }
    }
    out->entry = entry;
    out->similarity = best;
    out->hit = best >= min_similarity;
    return 0;
}

int po_embed_normalize(const double* x, size_t d, size_t T, double* out) { /* :60-64 */
    po_mean_pool(x, d, T, out);
    double s = 0; /* vec_norm, matrix.hpp:195-199 */
    for (size_t i = 0; i < d; ++i) s += out[i] * out[i];
    const double nrm = sqrt(s);
    if (nrm < 1e-12) return 3;
    for (size_t i = 0; i < d; ++i) out[i] /= nrm;
    return 0;
}

/* ---------------- include/parse/rank_experts.hpp ---------------- */
int po_check_selection(const uint32_t* sel, size_t k, size_t r_store) { /* :30-37 */
    if (k == 0) return 1;
    for (size_t i = 1; i < k; ++i)
        if (sel[i] <= sel[i - 1]) return 1;
    if (sel[k - 1] >= r_store) return 2;
    return 0;
}

int po_masked_forward(const double* A, const double* B, size_t m, size_t n, size_t r,
                      const uint32_t* sel, size_t k, const double* x, size_t T,
                      double* out) { /* :52-72 */
    int err = po_check_selection(sel, k, r);
    if (err) return err;
    memset(out, 0, m * T * sizeof(double));
    double* z = (double*)malloc((T ? T : 1) * sizeof(double));
    for (size_t q = 0; q < k; ++q) {
        const uint32_t e = sel[q];
        for (size_t c = 0; c < T; ++c) {
            double s = 0;
            for (size_t j = 0; j < n; ++j) s += B[j * r + e] * x[j * T + c];
            z[c] = s;
        }
        for (size_t i = 0; i < m; ++i) {
            const double a = A[i * r + e];
            double* row = out + i * T;
            for (size_t c = 0; c < T; ++c) row[c] += a * z[c];
        }
    }
    free(z);
    return 0;
}

/* ---------------- include/parse/exec_engine.hpp ---------------- */
struct po_agg {
    size_t m, n, r, s, P;
    int elem;
    uint32_t* shared_ids; /* ascending */
    void* shared_A;       /* m x s */
    void* shared_B;       /* n x s */
    size_t* res_count;
    uint32_t** res_ids;
    void** res_A; /* m x cnt */
    void** res_B; /* n x cnt */
    uint8_t** use_shared;
    size_t* arena_offset;
};

static void put(void* base, int elem, size_t idx, double v) {
    if (elem == 4) ((float*)base)[idx] = (float)v;
    else ((double*)base)[idx] = v;
}

po_agg* po_aggregate_layout(const double* A, const double* B, size_t m, size_t n, size_t r,
                            const uint32_t* patterns, const size_t* ks, size_t P, double psi,
                            int elem, int* err) { /* :112-164 */
    *err = 0;
    if (P == 0) { *err = 1; return NULL; }
    if (psi <= 0 || psi > 1) { *err = 1; return NULL; }
    size_t* freq = (size_t*)calloc(r, sizeof(size_t));
    size_t off = 0;
    for (size_t p = 0; p < P; ++p) {
        for (size_t q = 0; q < ks[p]; ++q) {
            uint32_t e = patterns[off + q];
            if (e >= r) { free(freq); *err = 2; return NULL; }
            freq[e] += 1;
        }
        off += ks[p];
    }
    po_agg* g = (po_agg*)calloc(1, sizeof(po_agg));
    g->m = m; g->n = n; g->r = r; g->P = P; g->elem = elem;
    g->shared_ids = (uint32_t*)malloc((r ? r : 1) * sizeof(uint32_t));
    size_t s = 0;
    for (size_t e = 0; e < r; ++e)
        if ((double)freq[e] >= psi * (double)P) g->shared_ids[s++] = (uint32_t)e;
    g->s = s;
    g->shared_A = malloc((m * s ? m * s : 1) * (size_t)elem);
    g->shared_B = malloc((n * s ? n * s : 1) * (size_t)elem);
    for (size_t j = 0; j < s; ++j) {
        const uint32_t e = g->shared_ids[j];
        for (size_t i = 0; i < m; ++i) put(g->shared_A, elem, i * s + j, A[i * r + e]);
        for (size_t i = 0; i < n; ++i) put(g->shared_B, elem, i * s + j, B[i * r + e]);
    }
    g->res_count = (size_t*)calloc(P, sizeof(size_t));
    g->res_ids = (uint32_t**)calloc(P, sizeof(uint32_t*));
    g->res_A = (void**)calloc(P, sizeof(void*));
    g->res_B = (void**)calloc(P, sizeof(void*));
    g->use_shared = (uint8_t**)calloc(P, sizeof(uint8_t*));
    g->arena_offset = (size_t*)calloc(P, sizeof(size_t));
    size_t arena = s;
    off = 0;
    for (size_t p = 0; p < P; ++p) {
        g->use_shared[p] = (uint8_t*)calloc(s ? s : 1, 1);
        g->res_ids[p] = (uint32_t*)malloc((ks[p] ? ks[p] : 1) * sizeof(uint32_t));
        size_t cnt = 0;
        for (size_t q = 0; q < ks[p]; ++q) {
            const uint32_t e = patterns[off + q];
            /* lower_bound over shared_ids */
            size_t lo = 0, hi = s;
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (g->shared_ids[mid] < e) lo = mid + 1; else hi = mid;
            }
            if (lo < s && g->shared_ids[lo] == e) g->use_shared[p][lo] = 1;
            else g->res_ids[p][cnt++] = e;
        }
        g->res_count[p] = cnt;
        g->res_A[p] = malloc((m * cnt ? m * cnt : 1) * (size_t)elem);
        g->res_B[p] = malloc((n * cnt ? n * cnt : 1) * (size_t)elem);
        for (size_t j = 0; j < cnt; ++j) {
            const uint32_t e = g->res_ids[p][j];
            for (size_t i = 0; i < m; ++i) put(g->res_A[p], elem, i * cnt + j, A[i * r + e]);
            for (size_t i = 0; i < n; ++i) put(g->res_B[p], elem, i * cnt + j, B[i * r + e]);
        }
        g->arena_offset[p] = arena;
        arena += cnt;
        off += ks[p];
    }
    free(freq);
    return g;
}

void po_agg_free(po_agg* g) {
    if (!g) return;
    for (size_t p = 0; p < g->P; ++p) {
        free(g->res_ids[p]); free(g->res_A[p]); free(g->res_B[p]); free(g->use_shared[p]);
    }
    free(g->res_count); free(g->res_ids); free(g->res_A); free(g->res_B);
    free(g->use_shared); free(g->arena_offset);
    free(g->shared_ids); free(g->shared_A); free(g->shared_B);
    free(g);
}
size_t po_agg_shared_count(const po_agg* g) { return g->s; }
void po_agg_shared_ids(const po_agg* g, uint32_t* out) {
    memcpy(out, g->shared_ids, g->s * sizeof(uint32_t));
}
size_t po_agg_residual_count(const po_agg* g, size_t p) { return g->res_count[p]; }
void po_agg_residual_ids(const po_agg* g, size_t p, uint32_t* out) {
    memcpy(out, g->res_ids[p], g->res_count[p] * sizeof(uint32_t));
}
size_t po_agg_arena_offset(const po_agg* g, size_t p) { return g->arena_offset[p]; }
void po_agg_use_shared(const po_agg* g, size_t p, uint8_t* out) { memcpy(out, g->use_shared[p], g->s); }

/* rank1_accumulate (:169-186), instantiated per element type */
#define DEFINE_RANK1(T, NAME)                                                              \
    static void NAME(const T* a_col, size_t a_stride, size_t m, const T* b_col,            \
                     size_t b_stride, size_t n, const T* x, size_t t, T* out, T* z) {      \
        for (size_t c = 0; c < t; ++c) z[c] = (T)0;                                        \
        for (size_t j = 0; j < n; ++j) {                                                   \
            const T b = b_col[j * b_stride];                                               \
            if (b == (T)0) continue;                                                       \
            const T* xr = x + j * t;                                                       \
            for (size_t c = 0; c < t; ++c) z[c] += b * xr[c];                              \
        }                                                                                  \
        for (size_t i = 0; i < m; ++i) {                                                   \
            const T a = a_col[i * a_stride];                                               \
            T* orow = out + i * t;                                                         \
            for (size_t c = 0; c < t; ++c) orow[c] += a * z[c];                            \
        }                                                                                  \
    }
DEFINE_RANK1(float, rank1_f32)
DEFINE_RANK1(double, rank1_f64)

typedef struct { uint32_t expert; int shared; size_t col; } po_src;
static int cmp_src(const void* pa, const void* pb) {
    const po_src* a = (const po_src*)pa;
    const po_src* b = (const po_src*)pb;
    return a->expert < b->expert ? -1 : (a->expert > b->expert ? 1 : 0);
}

/* aggregated_forward<T> (:193-236): merge used-shared and residual columns by
 * global expert id, then rank-1 accumulate in that order. */
#define DEFINE_AGG_FWD(T, NAME, RANK1, ELEM)                                               \
    int NAME(const po_agg* g, size_t pid, const T* x, size_t t, T* out) {                  \
        if (pid >= g->P) return 2;                                                         \
        if (g->elem != ELEM) return 1;                                                     \
        const size_t s = g->s, cnt = g->res_count[pid];                                    \
        po_src* order = (po_src*)malloc((s + cnt + 1) * sizeof(po_src));                   \
        size_t no = 0;                                                                     \
        for (size_t j = 0; j < s; ++j)                                                     \
            if (g->use_shared[pid][j]) { order[no].expert = g->shared_ids[j];              \
                order[no].shared = 1; order[no].col = j; ++no; }                           \
        for (size_t j = 0; j < cnt; ++j) { order[no].expert = g->res_ids[pid][j];          \
            order[no].shared = 0; order[no].col = j; ++no; }                               \
        qsort(order, no, sizeof(po_src), cmp_src);                                         \
        memset(out, 0, g->m * t * sizeof(T));                                              \
        T* z = (T*)malloc((t ? t : 1) * sizeof(T));                                        \
        for (size_t q = 0; q < no; ++q) {                                                  \
            const T* am = (const T*)(order[q].shared ? g->shared_A : g->res_A[pid]);       \
            const T* bm = (const T*)(order[q].shared ? g->shared_B : g->res_B[pid]);       \
            const size_t cols = order[q].shared ? s : cnt;                                 \
            RANK1(am + order[q].col, cols, g->m, bm + order[q].col, cols, g->n, x, t,      \
                  out, z);                                                                 \
        }                                                                                  \
        free(z);                                                                           \
        free(order);                                                                       \
        return 0;                                                                          \
    }
DEFINE_AGG_FWD(float, po_aggregated_forward_f32, rank1_f32, 4)
DEFINE_AGG_FWD(double, po_aggregated_forward_f64, rank1_f64, 8)

void po_scattered_forward_f32(const float* A, const float* B, size_t m, size_t n, size_t r,
                              const uint32_t* sel, size_t k, const float* x, size_t T,
                              float* out) { /* :239-252 */
    memset(out, 0, m * T * sizeof(float));
    float* z = (float*)malloc((T ? T : 1) * sizeof(float));
    for (size_t q = 0; q < k; ++q)
        rank1_f32(A + sel[q], r, m, B + sel[q], r, n, x, T, out, z);
    free(z);
}

static int cmp_size(const void* pa, const void* pb) {
    size_t a = *(const size_t*)pa, b = *(const size_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}
size_t po_maximal_runs(const size_t* cols, size_t count, size_t* starts, size_t* lens) {
    /* :77-88 sort, unique, merge */
    size_t* c = (size_t*)malloc((count ? count : 1) * sizeof(size_t));
    memcpy(c, cols, count * sizeof(size_t));
    qsort(c, count, sizeof(size_t), cmp_size);
    size_t nr = 0;
    for (size_t i = 0; i < count; ++i) {
        if (i > 0 && c[i] == c[i - 1]) continue;
        if (nr > 0 && starts[nr - 1] + lens[nr - 1] == c[i]) lens[nr - 1] += 1;
        else { starts[nr] = c[i]; lens[nr] = 1; ++nr; }
    }
    free(c);
    return nr;
}

void po_make_patterns(uint64_t seed, size_t n_patterns, const size_t* r_stores,
                      const size_t* ks, size_t n_layers, uint32_t* out) {
    po_rng rng = {seed};
    size_t max_r = 1;
    for (size_t l = 0; l < n_layers; ++l) if (r_stores[l] > max_r) max_r = r_stores[l];
    uint32_t* pool = (uint32_t*)malloc(max_r * sizeof(uint32_t));
    size_t w = 0;
    for (size_t p = 0; p < n_patterns; ++p) {
        for (size_t l = 0; l < n_layers; ++l) {
            size_t psz = r_stores[l];
            for (size_t i = 0; i < psz; ++i) pool[i] = (uint32_t)i;
            uint32_t* sel = out + w;
            for (size_t i = 0; i < ks[l]; ++i) {
                size_t pick = po_rng_below(&rng, 2) ? 0 : (size_t)po_rng_below(&rng, psz);
                sel[i] = pool[pick];
                memmove(pool + pick, pool + pick + 1, (psz - pick - 1) * sizeof(uint32_t));
                --psz;
            }
            qsort(sel, ks[l], sizeof(uint32_t), cmp_u32);
            w += ks[l];
        }
    }
    free(pool);
}
