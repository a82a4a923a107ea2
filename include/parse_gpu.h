/*
 * parse_gpu.h -- C-ABI of the B200 (sm_100a) rank-expert hot path.
 *
 * Drop-in boundary for the reference's C++ operator surface
 * (/root/reference/proj/include/parse/*.hpp).  Plain pointers and sizes, no
 * torch types.  Every entry point cites the reference interface it replaces.
 * The C++ mirror that keeps the reference signatures intact is
 * include/parse_gpu.hpp (namespace parse::gpu); the Python mirror is the
 * paper_2605_08568_b200 package.
 *
 * Conventions
 *  - Return value: PG_OK or an error class mirroring the reference's exception
 *    types (std::invalid_argument / std::out_of_range / std::runtime_error), plus
 *    PG_CUDA_ERROR.  pg_last_error() returns a thread-local message (the
 *    reference's exception text where one exists, e.g. "select_topk: K out of
 *    range").
 *  - "dev" pointers are device memory; "host" pointers are host memory.
 *  - Calls taking a pg_stream are asynchronous on that stream (cudaStream_t, 0 =
 *    legacy default).  Device buffers passed in are borrowed until the stream
 *    is synchronised.  Calls that return host values synchronise the stream.
 *  - Layouts: PG_FEATURE_MAJOR is the reference's Mat layout for activations
 *    (X is n x T row-major, toy_lm.hpp:110); PG_TOKEN_MAJOR is T x n.  For
 *    T == 1 they are the same bytes.
 *  - Handles are immutable after creation (concurrent readers
 *    allowed); the library is thread-safe for distinct streams.
 */
#ifndef PARSE_GPU_H
#define PARSE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_OK 0
#define PG_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define PG_OUT_OF_RANGE 2     /* std::out_of_range */
#define PG_RUNTIME_ERROR 3    /* std::runtime_error */
#define PG_CUDA_ERROR 4

typedef enum { PG_F64 = 0, PG_F32 = 1, PG_BF16 = 2 } pg_dtype;
typedef enum { PG_FEATURE_MAJOR = 0, PG_TOKEN_MAJOR = 1 } pg_layout;
typedef void* pg_stream; /* cudaStream_t */

typedef struct pg_router_s* pg_router; /* RouterParams (router.hpp:15-20) on device   */
typedef struct pg_layer_s* pg_layer;   /* FactorizedLayer (factorize.hpp:28-37)       */
typedef struct pg_agg_s* pg_agg;       /* AggregatedLayer<T> (exec_engine.hpp:97-110) */
typedef struct pg_cache_s* pg_cache;   /* PatternCache embeddings (pattern_cache.hpp:31-36) */

const char* pg_last_error(void);
int pg_abi_version(void);
/* Number of this library's kernels launched so far on this host thread's process
 * (monotone counter; bench.py reports deltas as gpu_launches). */
uint64_t pg_launch_count(void);

/* ------------------------------------------------------------------ */
/* a5-a7: routing  (router.hpp:41-61,80-88)                            */
/* ------------------------------------------------------------------ */

/* mean_pool (router.hpp:80-88), bit-exact: h[p*n+i] = (sequential sum over the
 * prompt's tokens of x(i,t)) / T_p.  x dtype f64/f32/bf16 (widened exactly to
 * f64).  offsets_host[P+1] are token offsets of each prompt into x
 * (P=1, offsets {0,T} for one sequence).  h_dev: P x n f64. */
int pg_mean_pool(const void* x_dev, pg_dtype x_dtype, pg_layout layout, size_t n,
                 const int64_t* offsets_host, size_t n_prompts, double* h_dev, pg_stream stream);

/* score (router.hpp:41-46): z = theta*h + bias.  exact=1 reproduces the
 * reference's sequential dot bit-for-bit; exact=0 is the fast warp-tree GEMV
 * (|z - z_ref| <= 4(n+2)u(sum|theta_ij h_j| + |b_i|), u = 2^-53). */
int pg_router_create(pg_router* out, size_t r, size_t n, const double* theta_host,
                     const double* bias_host);
/* theta_dev r x n and bias_dev r (f64) already on device; copy=0 borrows them. */
int pg_router_create_device(pg_router* out, size_t r, size_t n, const double* theta_dev,
                            const double* bias_dev, int copy);
int pg_router_destroy(pg_router r);
int pg_score(pg_router router, const double* h_dev, size_t n_prompts, double* logits_dev,
             int exact, pg_stream stream);

/* select_topk (router.hpp:49-61) on given logits: K largest, ties toward the
 * lower index, output ascending.  Exact (pure comparisons). */
int pg_select_topk(const double* logits_dev, size_t r, size_t n_prompts, size_t k,
                   uint32_t* sel_dev, pg_stream stream);

/* Fused RoutingProvider::apply routing step (model.hpp:100-104):
 * select_topk(score(theta, mean_pool(x)), K) per prompt, bit-identical to the
 * reference (fast GEMV + error-bounded band + reference-order recompute of the
 * rows that straddle the K-th logit).  sel_dev: n_prompts x K ascending u32.
 * logits_dev (nullable, n_prompts x r) receives the logits used for selection. */
int pg_route_select(pg_router router, const void* x_dev, pg_dtype x_dtype, pg_layout layout,
                    const int64_t* offsets_host, size_t n_prompts, size_t k, uint32_t* sel_dev,
                    double* logits_dev, pg_stream stream);

/* The same routing step from already pooled inputs h_dev (n_prompts x n f64,
 * mean_pool output): linears that share an input (q/k/v, up/gate,
 * toy_lm.hpp:220-249) pool it once and route every router from it. */
int pg_route_select_pooled(pg_router router, const double* h_dev, size_t n_prompts, size_t k,
                           uint32_t* sel_dev, double* logits_dev, pg_stream stream);

/* ------------------------------------------------------------------ */
/* a9-a12: pattern cache  (pattern_cache.hpp:38-65,95-124)             */
/* ------------------------------------------------------------------ */

typedef struct {
    size_t entry;      /* RetrieveResult::entry      */
    double similarity; /* RetrieveResult::similarity */
    int hit;           /* RetrieveResult::hit        */
    int exact_similarity; /* 1 if similarity is the reference-order value */
} pg_retrieve_result;

/* cosine (pattern_cache.hpp:38-47), reference order, bit-exact. out_dev: 1 f64 */
int pg_cosine(const double* a_dev, const double* b_dev, size_t d, double* out_dev,
              pg_stream stream);
int pg_cache_create(pg_cache* out, size_t d, size_t capacity, double min_similarity);
int pg_cache_destroy(pg_cache c);
int pg_cache_size(pg_cache c, size_t* size_out);
/* cache_insert (pattern_cache.hpp:120-124): append iff size < capacity.
 * emb: d f64 (host or device per emb_on_device).  *inserted = 0 when full. */
int pg_cache_insert(pg_cache c, const double* emb, int emb_on_device, int* inserted,
                    pg_stream stream);
/* Bulk load of N x d embeddings (load_cache, pattern_cache.hpp:294-327). */
int pg_cache_load(pg_cache c, const double* emb_host, size_t n_entries);
/* retrieve (pattern_cache.hpp:104-117): exhaustive cosine scan, first maximum,
 * hit = sim >= min_similarity.  entry/hit bit-exact vs the reference; the
 * similarity is the reference-order value when exact_similarity=1 (or when the
 * guard had to recompute it), else within 4(d+4)u(...)-relative.
 * query_dev: d f64.  result_host (nullable) synchronises the stream;
 * entry_dev (nullable, int32) / hit_dev (nullable, int32) stay on device so a
 * forward can consume the hit without a host round trip. */
int pg_retrieve(pg_cache c, const double* query_dev, int exact_similarity,
                pg_retrieve_result* result_host, int32_t* entry_dev, int32_t* hit_dev,
                pg_stream stream);
/* embed_prompt's pooling half (pattern_cache.hpp:60-64): mean_pool of the
 * block-0 output (d x T) then divide by vec_norm; bit-exact.  Degenerate
 * (norm < 1e-12) -> PG_RUNTIME_ERROR "degenerate embedding" (synchronises). */
int pg_embed_normalize(const void* x_dev, pg_dtype x_dtype, pg_layout layout, size_t d,
                       size_t T, double* emb_dev, pg_stream stream);

/* ------------------------------------------------------------------ */
/* a2, a13, a16: factorized layer + value path (rank_experts.hpp:52-72) */
/* ------------------------------------------------------------------ */

/* Upload a FactorizedLayer: A m x r_store, B n x r_store (host f64, the
 * reference's Matd layout, factorize.hpp:32-33).  Stored on device as
 * expert-major B^T [r_store x n] and A [m x r_store] in `storage`. */
int pg_layer_create(pg_layer* out, size_t m, size_t n, size_t r_store, size_t K,
                    const double* A_host, const double* B_host, pg_dtype storage);
/* Device factors already in the device layout (bt_dev r_store x n, a_dev
 * m x r_store, both `storage` dtype); copy=0 borrows them. */
int pg_layer_create_device(pg_layer* out, size_t m, size_t n, size_t r_store, size_t K,
                           const void* bt_dev, const void* a_dev, pg_dtype storage, int copy);
int pg_layer_destroy(pg_layer l);
int pg_layer_info(pg_layer l, size_t* m, size_t* n, size_t* r_store, size_t* K,
                  pg_dtype* storage);

/* check_selection (rank_experts.hpp:30-37) on a host selection. */
int pg_check_selection(pg_layer l, const uint32_t* sel_host, size_t k);

/* masked_forward (rank_experts.hpp:52-72) == scattered_forward
 * (exec_engine.hpp:239-252): y = sum_{e in S} A[:,e] (B[:,e]^T x), fp32
 * accumulation (f64 for f64 storage).  x dtype == storage; y dtype is
 * storage or PG_F32.  sel is host (validated, uploaded) when sel_on_device=0,
 * else a device array trusted to be valid (e.g. pg_route_select output). */
int pg_masked_forward(pg_layer l, const uint32_t* sel, size_t k, int sel_on_device,
                      const void* x_dev, pg_layout layout, size_t T, void* y_dev,
                      pg_dtype y_dtype, pg_stream stream);

/* ------------------------------------------------------------------ */
/* a14-a15, a19: aggregated layout (exec_engine.hpp:97-236)             */
/* ------------------------------------------------------------------ */

/* aggregate_layout<T> (exec_engine.hpp:112-164) built on device by gather:
 * shared experts (freq >= psi*P) at the arena head, each pattern's residual
 * experts in its own block.  patterns_host: concatenated ids, ks_host[P]. */
int pg_aggregate_layout(pg_agg* out, pg_layer l, const uint32_t* patterns_host,
                        const size_t* ks_host, size_t n_patterns, double psi, pg_stream stream);
int pg_agg_destroy(pg_agg g);
int pg_agg_patterns(pg_agg g, size_t* n_patterns);
int pg_agg_shared(pg_agg g, size_t* count, uint32_t* ids_host /* nullable */);
/* residual ids (ascending), the reference's arena_offset, use_shared flags */
int pg_agg_residual(pg_agg g, size_t pattern, size_t* count, uint32_t* ids_host,
                    size_t* arena_offset, uint8_t* use_shared_host);
/* AccessTrace (exec_engine.hpp:90-92): arena columns one forward touches, in
 * the reference's column numbering; *count then cols_host (nullable). */
int pg_agg_trace(pg_agg g, size_t pattern, size_t* count, size_t* cols_host);
/* Device bytes of the arena (storage_overhead accounting, :310-318). */
int pg_agg_bytes(pg_agg g, size_t* bytes);

/* aggregated_forward<T> (exec_engine.hpp:193-236) for one pattern.
 * pattern_dev (nullable int32 on device) overrides `pattern` without a host
 * round trip (e.g. the entry index written by pg_retrieve). */
int pg_aggregated_forward(pg_agg g, size_t pattern, const int32_t* pattern_dev,
                          const void* x_dev, pg_layout layout, size_t T, void* y_dev,
                          pg_dtype y_dtype, pg_stream stream);

/* Heterogeneous batch (prefill or decode): prompt p owns tokens
 * [offsets_host[p], offsets_host[p+1]) of token-major x and is served with
 * pattern patterns_host[p] of the aggregated layout.  y token-major. */
int pg_aggregated_forward_batched(pg_agg g, const int32_t* patterns_host,
                                  const int64_t* offsets_host, size_t n_prompts,
                                  const void* x_dev, void* y_dev, pg_dtype y_dtype,
                                  pg_stream stream);

/* K6 module fusion for decode (T = 1): build_plan's fused_B + batched_A groups
 * (exec_engine.hpp:46-68) executed as ONE kernel -- 1..3 linears sharing the
 * input x (e.g. {q,k,v} or {up,gate}); ys[l] receives linear l's output.
 * patterns_host[l] selects each linear's pattern, or pattern_dev (int32 on
 * device, same pattern id for all linears) overrides them. */
int pg_module_forward(const pg_agg* layers, size_t n_linears, const size_t* patterns_host,
                      const int32_t* pattern_dev, const void* x_dev, void* const* ys_dev,
                      pg_dtype y_dtype, pg_stream stream);

/* Whole MLP block decode step (T = 1) in one kernel: up/gate share x (fused B
 * side), act = silu(gate)*up in the stage-2 epilogue (toy_lm.hpp:250-257),
 * then down_proj on act.  act_dev (nullable, m_ff elements of the storage
 * dtype) receives the activation; y_dev the block output. */
int pg_mlp_forward(pg_agg up, pg_agg gate, pg_agg down, const size_t* patterns_host,
                   const int32_t* pattern_dev, const void* x_dev, void* act_dev, void* y_dev,
                   pg_dtype y_dtype, pg_stream stream);
/* A chain of S MLP blocks as in pg_mlp_forward, block s+1 reading block s's
 * output (x_{s+1} = y_s; y in the weight dtype when S > 1): patterns [S][3]
 * (up, gate, down), acts[s] optional (null array or entries: workspace),
 * ys[s] the blocks' outputs.  Up to 8 blocks per launch: the weight stream
 * runs through each block's last exchange and the launch boundary. */
int pg_mlp_forward_chain(const pg_agg* ups, const pg_agg* gates, const pg_agg* downs, const size_t* patterns,
                         size_t S, const void* x_dev, void* const* acts_dev, void* const* ys_dev, pg_dtype y_dtype,
                         pg_stream stream);

/* Union-masked heterogeneous batch (BASELINE config 4: decode batch of
 * prompts, each with its own selection): masked_forward (rank_experts.hpp:52-72)
 * for every token t of token-major x [T, n] with the selection of pattern
 * tok_pat_dev[t], reading the layer's weights once for the whole batch (two
 * tcgen05 GEMMs over all r_store experts, non-selected experts zeroed per token
 * in the first GEMM's epilogue).  bf16 layers; y token-major [T, m] (bf16/f32).
 * masks_dev: [P, stride] bytes from pg_selection_masks (stride from
 * pg_selection_mask_stride); tok_pat_dev values must lie in [0, P). */
int pg_selection_mask_stride(pg_layer layer, size_t* stride);
int pg_selection_masks(pg_layer layer, const uint32_t* sels_concat, const size_t* ks, size_t P,
                       uint8_t* masks_dev, pg_stream stream);
int pg_masked_forward_union(pg_layer layer, const uint8_t* masks_dev, size_t P, const int32_t* tok_pat_dev,
                            size_t T, const void* x_dev, void* y_dev, pg_dtype y_dtype, pg_stream stream);
/* The same for 1..32 linears sharing the input x (q/k/v, up/gate): each
 * stage is one grouped launch over all linears.  masks_dev[l] / P[l] per
 * linear (pg_selection_masks of that layer), one pattern id per token. */
int pg_module_forward_union(const pg_layer* layers, const uint8_t* const* masks_dev, const size_t* P,
                            size_t n_linears, const int32_t* tok_pat_dev, size_t T, const void* x_dev,
                            void* const* ys_dev, pg_dtype y_dtype, pg_stream stream);

/* A whole heterogeneous decode step as ONE persistent launch (config 4):
 * the union program records modules (linears sharing an input, as
 * pg_module_forward_union, T <= 256 tokens) and runs all their GEMM stages in
 * one launch, each k-block of a stage waiting (device-side ready counters) for
 * the output tile of the stage that produces it, weights streamed across stage
 * and layer boundaries.  The executed form of the reference's ExecPlan
 * (exec_engine.hpp:19-68: fused_B / batched_A per module) for a whole stack.
 * x_dev / ys_dev addresses are bound at add time; a module whose x_dev is an
 * earlier module's output consumes it tile by tile.  Every output buffer must
 * be distinct and never overwrite an input of an earlier module (per-layer
 * buffers).  tok_offset: this module's T tokens are entries [tok_offset,
 * tok_offset + T) of the run's token -> pattern table (independent token
 * groups as separate chains in one program); weights_reused: another chain
 * reads the same weights soon (keep them in L2 instead of evict-first).  The first pg_union_prog_run allocates the workspace (not
 * capturable); later runs are single launches, capturable in CUDA graphs. */
typedef struct pg_union_prog_s* pg_union_prog;
int pg_union_prog_create(pg_union_prog* out, size_t T);
int pg_union_prog_add_module(pg_union_prog prog, const pg_layer* layers, const uint8_t* const* masks_dev,
                             const size_t* P, size_t n_linears, const void* x_dev, void* const* ys_dev,
                             pg_dtype y_dtype, size_t tok_offset, int weights_reused);
int pg_union_prog_run(pg_union_prog prog, const int32_t* tok_pat_dev, pg_stream stream);
int pg_union_prog_info(pg_union_prog prog, size_t* phases, size_t* grid);
int pg_union_prog_destroy(pg_union_prog prog);
/* Diagnostics: with PG_PROG_DBG=1 at the first run, per-CTA %globaltimer stamps
 * [grid][64] of the last run (*have = 0 otherwise). */
int pg_union_prog_debug(pg_union_prog prog, uint64_t* out_host, size_t n, int* have);

/* Expert-sharded decode (BASELINE config 5) with the all-reduce fused into
 * the rank-expert kernel: rank `rank` of `npeer` serves its expert shard
 * (aggregated layout of its experts, `pattern` = the local selection) for one
 * token; the stage-2 epilogue pushes every output row's partial as a tagged
 * word into each rank's receive buffer (peer_bufs[r], device pointers of all
 * ranks' buffers -- NVLink peer memory, opened with pg_ipc_open_handle), and
 * each CTA then sums its rows over the ranks in rank order, so every rank ends
 * with the full y (deterministic, identical on all ranks).  Buffers: zeroed
 * device memory of pg_peer_buffer_bytes(m, npeer) each; all ranks must issue
 * the same sequence of chain launches on their stream and use the same grid
 * (0 = all SMs). */
int pg_peer_buffer_bytes(size_t m, size_t npeer, size_t* bytes);
int pg_agg_forward_peer(pg_agg shard, size_t pattern, const void* x_dev, void* y_dev, pg_dtype y_dtype, int rank,
                        int npeer, void* const* peer_bufs, int grid, pg_stream stream);
/* Expert-sharded MLP block (config 5 decode, toy_lm.hpp:250-257 with every
 * linear sharded e mod npeer) in ONE launch: up/gate partials are pushed to
 * every rank and summed in rank order per act row (so each rank forms the
 * whole act = silu(gate) * up for its down shard), then down's partials are
 * reduced the same way.  patterns[3] = local up/gate/down pattern ids; act
 * (nullable) receives the reduced act; buffers: pg_peer_buffer_bytes(2 * m_ff
 * + d, npeer) each, same rules as pg_agg_forward_peer. */
int pg_mlp_forward_peer(pg_agg up, pg_agg gate, pg_agg down, const size_t* patterns, const void* x_dev,
                        void* act_dev, void* y_dev, pg_dtype y_dtype, int rank, int npeer, void* const* peer_bufs,
                        int grid, pg_stream stream);
int pg_ipc_get_handle(const void* dev_ptr, void* handle64_out);
int pg_ipc_open_handle(const void* handle64, void** dev_ptr);
int pg_ipc_close(void* dev_ptr);

/* Heterogeneous prefill (config 3): prompt p owns tokens
 * [offsets_host[p], offsets_host[p+1]) of token-major x (bf16) and its own
 * aggregated layout aggs[p] (served with pattern 0, e.g. the single pattern
 * packed after routing / a cache hit).  All prompts' stage-1 GEMMs run as one
 * grouped tcgen05 launch, then all stage-2 GEMMs.  y token-major. */
int pg_prefill_batched(const pg_agg* aggs, const int64_t* offsets_host, size_t n_prompts,
                       const void* x_dev, void* y_dev, pg_dtype y_dtype, pg_stream stream);

/* Routed prefill with the expert pack on device (config 3; exec_engine.hpp:
 * 112-164's column copies for one pattern per prompt, then
 * aggregated_forward<T> :193-236 as tcgen05 GEMMs).  sel_dev [P, k] int32 holds
 * every prompt's K ascending expert ids on the device (pg_route_select /
 * pg_route_select_pooled output: no host round trip).  pg_pack_selected packs
 * them into caller buffers bt_out [P][kp][ldb] and a_out [P][m][kp] (kp = k
 * rounded up to 8, zero padded; sizes from pg_pack_bytes); pg_prefill_packed
 * runs prompt p (tokens offsets_host[p]:offsets_host[p+1] of token-major x)
 * through its packed experts.  bf16 layers; asynchronous on `stream`. */
int pg_pack_bytes(pg_layer layer, size_t k, size_t n_prompts, size_t* bt_bytes, size_t* a_bytes);
int pg_pack_selected(pg_layer layer, const int32_t* sel_dev, size_t k, size_t n_prompts, void* bt_out,
                     void* a_out, pg_stream stream);
int pg_prefill_packed(pg_layer layer, const void* bt_packed, const void* a_packed, size_t k,
                      const int64_t* offsets_host, size_t n_prompts, const void* x_dev, void* y_dev,
                      pg_dtype y_dtype, pg_stream stream);
/* pg_prefill_gathered: pg_prefill_packed without the packed B^T arena -- the
 * stage-1 GEMM gathers each prompt's selected B^T rows sel_dev[p*k + j]
 * straight from the layer (TMA gather4); a_packed from pg_pack_selected with
 * bt_out = NULL (A columns only).  Every prompt needs 0 or >= 256 tokens.
 * Results are bit-identical to pg_prefill_packed. */
int pg_prefill_gathered(pg_layer layer, const int32_t* sel_dev, const void* a_packed, size_t k, const int64_t* offsets,
                        size_t n_prompts, const void* x, void* y, pg_dtype y_dtype, pg_stream stream);

/* K5 primitive: C[M, N] = A[M, K] . B[N, K]^T on the tcgen05 tensor cores
 * (bf16 operands, both K-major with 16-byte aligned rows, f32 accumulation;
 * out bf16 when out_bf16 else f32).  The prefill paths are two of these per
 * prompt, grouped across prompts. */
int pg_gemm_bf16(const void* a_dev, int64_t lda, const void* b_dev, int64_t ldb, void* out_dev,
                 int64_t ldo, size_t M, size_t N, size_t K, int out_bf16, pg_stream stream);

/* MLP glue between upgate() and down_proj() (toy_lm.hpp:250-257):
 * act[i] = silu(gate[i]) * up[i], computed in f32 (f64 for f64 inputs) and
 * stored in act_dtype.  gate/up dtype in_dtype (PG_F32 or PG_F64). */
int pg_silu_mul(const void* gate_dev, const void* up_dev, pg_dtype in_dtype, size_t count,
                void* act_dev, pg_dtype act_dtype, pg_stream stream);

/* ------------------------------------------------------------------ */
/* host utilities                                                      */
/* ------------------------------------------------------------------ */

/* Rng (rng.hpp:10-41): count gaussians from Rng(seed) -- bit-identical to the
 * reference's fixtures. */
void pg_rng_fill_gaussian(uint64_t seed, double* out_host, size_t count);
/* The reference's prefix-biased pattern generator (test_acceptance.cpp:412-425)
 * in O(K log r) per draw: same ids as the reference's O(K r) vector::erase. */
void pg_make_patterns(uint64_t seed, size_t n_patterns, const size_t* r_stores,
                      const size_t* ks, size_t n_layers, uint32_t* out_host);
/* Device-side synthetic fill (bench weights too large for host f64):
 * out[i] = scale * N(0,1) from a counter-based hash of (seed, i). */
int pg_fill_normal_device(void* out_dev, pg_dtype dtype, size_t count, uint64_t seed,
                          double scale, pg_stream stream);

/* Step I/O as a kernel: copy `bytes` between device-accessible buffers
 * (device memory, or pinned host memory at its UVA address) on `stream`,
 * chained to the neighbouring kernels by programmatic dependent launch -- the
 * per-token H2D of x and D2H of y without copy-engine nodes in the step. */
int pg_copy_io(const void* src, void* dst, size_t bytes, pg_stream stream);

/* Release the per-stream workspaces the library keeps per (device, stream,
 * grid size) for `stream` (decode chain: barrier counter, launch epoch, z/act
 * exchange words; union batch: launch epoch, split-tile flags and partials); call before destroying a per-request stream.  Synchronises the
 * stream first.  The next chain launch on that stream re-creates them. */
int pg_chain_workspace_release(pg_stream stream);

/* Diagnostics: with PG_CHAIN_DBG=1 the decode-chain kernel records per-CTA
 * %globaltimer stamps [cta][16] of its phases; copies the last launch's. */
int pg_chain_debug_dump(uint64_t* out_host, size_t n);

#ifdef __cplusplus
}
#endif
#endif
