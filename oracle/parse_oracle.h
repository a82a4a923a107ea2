/*
 * parse_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU hot path (PARSE rank-expert
 * layer: router, pattern cache, rank experts, aggregated execution), used as
 * the parity CHECKER for the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product library (paper_2605_08568_b200/lib/libparse_gpu.so) never links or
 * calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference compiled from /root/reference (oracle/_ref/libparse_ref.so, built
 * by oracle/build.py) and against the known-answer vectors of the reference's
 * own doctest suites (tests/test_oracle_golden.py, tests/golden/).
 *
 * Build flags matter for bit-exactness: -O2 -ffp-contract=off, no -march=native
 * (the reference's sequential fp64 dots must not be FMA-contracted).
 */
#ifndef PARSE_ORACLE_H
#define PARSE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:10-41 (splitmix64 + Box-Muller without spare) ---- */
typedef struct { uint64_t state; } po_rng;
uint64_t po_rng_next_u64(po_rng* r);
double po_rng_uniform(po_rng* r);
uint64_t po_rng_below(po_rng* r, uint64_t n);
double po_rng_gaussian(po_rng* r);
po_rng po_rng_fork(const po_rng* r, uint64_t salt);
/* Rng(seed); out[i] = gaussian() for i in [0,count) -- the fixture idiom
 * `for (double& v : a.raw()) v = rng.gaussian();` (test_router.cpp:13-18). */
void po_fill_gaussian(uint64_t seed, double* out, size_t count);

/* ---- factorize.hpp:86-89 store_rank; :135-195 single-layer budget ---- */
size_t po_store_rank(size_t k, size_t r_max, double store_multiplier);
size_t po_single_layer_k(size_t m, size_t n, double ratio);

/* ---- router.hpp inference half ---- */
void po_mean_pool(const double* x, size_t n, size_t T, double* h);            /* :80-88 */
void po_score(const double* theta, const double* bias, size_t r, size_t n,
              const double* h, double* z);                                      /* :41-46 */
/* :49-61; returns 0 ok, 1 invalid_argument (K out of range). out: K ascending */
int po_select_topk(const double* logits, size_t r, size_t k, uint32_t* out);

/* ---- pattern_cache.hpp ---- */
/* :38-47; returns NaN and sets *err=1 on length mismatch (callers pass equal d) */
double po_cosine(const double* a, const double* b, size_t d);
typedef struct {
    size_t entry;
    double similarity;
    int hit;
} po_retrieve_result;
/* :104-117; emb is N x d row-major; returns 0 ok, 3 runtime_error (empty cache) */
int po_retrieve(const double* emb, size_t n_entries, size_t d, double min_similarity,
                const double* query, po_retrieve_result* out);
/* :50-65 pooling half: mean_pool(d x T block output) then L2-normalise with
 * vec_norm (matrix.hpp:195-199); returns 0 ok, 3 runtime_error (degenerate) */
int po_embed_normalize(const double* x, size_t d, size_t T, double* out);

/* ---- rank_experts.hpp ---- */
/* :30-37: 0 ok, 1 invalid_argument (empty / not strictly increasing), 2 out_of_range */
int po_check_selection(const uint32_t* sel, size_t k, size_t r_store);
/* :52-72 canonical fp64 value path. A m x r, B n x r, x n x T (all row-major) */
int po_masked_forward(const double* A, const double* B, size_t m, size_t n, size_t r,
                      const uint32_t* sel, size_t k, const double* x, size_t T,
                      double* out);

/* ---- exec_engine.hpp aggregated layout (:97-164) and forwards (:169-252) ---- */
typedef struct po_agg po_agg;
/* patterns: concatenated index lists, pattern p has ks[p] ids.  elem: 4 (float)
 * or 8 (double) -- the template parameter T of aggregate_layout<T>.
 * *err: 0 ok, 1 invalid_argument, 2 out_of_range. */
po_agg* po_aggregate_layout(const double* A, const double* B, size_t m, size_t n, size_t r,
                            const uint32_t* patterns, const size_t* ks, size_t n_patterns,
                            double psi, int elem, int* err);
void po_agg_free(po_agg* g);
size_t po_agg_shared_count(const po_agg* g);
void po_agg_shared_ids(const po_agg* g, uint32_t* out);
size_t po_agg_residual_count(const po_agg* g, size_t p);
void po_agg_residual_ids(const po_agg* g, size_t p, uint32_t* out);
size_t po_agg_arena_offset(const po_agg* g, size_t p);
void po_agg_use_shared(const po_agg* g, size_t p, uint8_t* out);
/* aggregated_forward<T> (:193-236); x n x T, out m x T of the agg's element type */
int po_aggregated_forward_f32(const po_agg* g, size_t pattern, const float* x, size_t T,
                              float* out);
int po_aggregated_forward_f64(const po_agg* g, size_t pattern, const double* x, size_t T,
                              double* out);
/* scattered_forward<float> (:239-252) over full fp32 casts of A (m x r), B (n x r) */
void po_scattered_forward_f32(const float* A, const float* B, size_t m, size_t n, size_t r,
                              const uint32_t* sel, size_t k, const float* x, size_t T,
                              float* out);
/* exec_engine.hpp:77-88 maximal_runs: writes (start,len) pairs, returns count */
size_t po_maximal_runs(const size_t* cols, size_t count, size_t* starts, size_t* lens);

/* ---- the reference's seeded prefix-biased pattern generator ----
 * test_exec_engine.cpp:27-46 / test_acceptance.cpp:412-425: one Rng(seed);
 * for each pattern, for each layer (in the order given), draw K ids by
 * `pick = rng.below(2) ? 0 : rng.below(pool.size())`, erase, then sort.
 * out receives n_patterns * sum(ks) ids (pattern-major, then layer). */
void po_make_patterns(uint64_t seed, size_t n_patterns, const size_t* r_stores,
                      const size_t* ks, size_t n_layers, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
