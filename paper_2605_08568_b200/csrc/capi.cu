// capi.cu -- the extern "C" boundary (include/parse_gpu.h): handles, argument
// validation with the reference's exception classes/messages, workspace, and
// dispatch to the sm_100a kernels.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "chain.cuh"
#include "umma.cuh"
#include "union_prog.cuh"
#include "union_wm.cuh"

namespace pg {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_err;
void set_error(int code, const std::string& msg) {
    (void)code;
    t_err = msg;
}

// ---- kernel launchers (route.cu, cache.cu, values.cu, umma.cu) ----
void launch_mean_pool(const void* x, pg_dtype dt, pg_layout lay, int n, int64_t ttot,
                      const int64_t* offs_dev, int P, double* h, cudaStream_t st);
void launch_copy_io(const void* src, void* dst, size_t bytes, cudaStream_t st);
void launch_score(const double* theta, const double* bias, int r, int n, const double* h, int P,
                  double* z, double* bnd, int exact, cudaStream_t st, double* hnorm = nullptr);
void launch_select_topk(const double* logits, int r, int P, int K, uint32_t* sel, cudaStream_t st);
void launch_route_select(const double* zfast, const double* bnd, const double* theta,
                         const double* bias, const double* h, int r, int n, int K, int P,
                         uint32_t* sel, double* logits_out, int* stats, cudaStream_t st);
int max_select_rows();
void launch_cosine_scan(const double* emb, const double* q, int N, int d, double* sim, double* bnd,
                        cudaStream_t st);
void launch_retrieve_select(const double* sim, const double* bnd, const double* emb,
                            const double* q, int N, int d, double min_sim, int exact_similarity,
                            double* out_f64, int32_t* out_i32, int32_t* entry_dev,
                            int32_t* hit_dev, cudaStream_t st);
void launch_cosine_exact(const double* a, const double* b, int d, double* out, cudaStream_t st);
void launch_embed_finish(double* h, int d, int* flag, cudaStream_t st);
int max_cache_dim();
void launch_gather_rows(pg_dtype dt, const void* src, int64_t lds, const int32_t* idx, int cnt,
                        int cnt_pad, int cols, void* dst, int64_t ldd, cudaStream_t st);
void launch_pack_selected(const void* bt, int64_t ldb, const void* a, int64_t lda, int r, int n, int m,
                          const int32_t* sel, int k, int P, void* bt_out, void* a_out, cudaStream_t st);
void launch_gather_cols(pg_dtype dt, const void* src, int64_t lds, const int32_t* idx, int cnt,
                        int cnt_pad, int m, void* dst, int64_t ldd, cudaStream_t st);
int decode_tmax(int T);
size_t decode_smem_need(pg_dtype wdt, int n, int nslots, int T);
void launch_decode(pg_dtype wdt, const void* bt, int64_t ldb, const void* a, int64_t lda, SlotMap sm,
                   int n, int m, const void* x, int fm, int T, void* z, void* y, pg_dtype ydt,
                   cudaStream_t st);
size_t simt_ws_elems(int n, int m, int ns, int T);
void launch_simt(pg_dtype wdt, const void* bt, int64_t ldb, const void* a, int64_t lda, SlotMap sm,
                 int n, int m, const void* x, int fm, int T, void* ws, void* y, pg_dtype ydt,
                 cudaStream_t st);
void launch_fill_normal(void* out, pg_dtype dt, size_t count, uint64_t seed, double scale,
                        cudaStream_t st);
void launch_silu_mul(const void* g, const void* u, pg_dtype in_dt, size_t count, void* act,
                     pg_dtype act_dt, cudaStream_t st);
void launch_transpose(pg_dtype dt, const void* src, int rows, int cols, void* dst, cudaStream_t st);

// ---- stream-ordered scratch (freed when the scope ends, after queued work) ----
static void init_pool() {
    once_per_device(reinterpret_cast<const void*>(&init_pool), [] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, current_device()) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

struct Scratch {
    void* p = nullptr;
    cudaStream_t st;
    Scratch(size_t bytes, cudaStream_t s) : st(s) {
        init_pool();
        if (bytes) PG_CUDA_THROW(cudaMallocAsync(&p, (bytes + 255) / 256 * 256, st));
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, st);
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};

static void* dev_alloc(size_t bytes) {
    void* p = nullptr;
    PG_CUDA_THROW(cudaMalloc(&p, bytes ? bytes : 16));
    return p;
}

static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
constexpr int kSlotAlign = 32;  // slot runs aligned to the GEMM K-block / 16 B vectors

// host f64 -> device dtype conversion (round to nearest even for bf16/f32)
static uint16_t f32_to_bf16_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // NaN
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}
static void convert_store(const double* src, size_t count, pg_dtype dt, void* dst) {
    if (dt == PG_F64) std::memcpy(dst, src, count * 8);
    else if (dt == PG_F32)
        for (size_t i = 0; i < count; ++i) static_cast<float*>(dst)[i] = (float)src[i];
    else
        for (size_t i = 0; i < count; ++i)
            static_cast<uint16_t*>(dst)[i] = f32_to_bf16_bits((float)src[i]);
}

}  // namespace pg

using namespace pg;

// ---------------------------------------------------------------- handles
struct pg_router_s {
    int r, n;
    double* theta;
    double* bias;
    bool owned;
};
struct pg_layer_s {
    int m, n, r, K;
    pg_dtype dt;
    void* bt;     // [r, ldb]
    int64_t ldb;  // >= n, 16-byte multiple
    void* a;      // [m, lda]
    int64_t lda;  // >= r, 16-byte multiple
    bool owned;
};
struct pg_agg_s {
    pg_layer layer;
    int m, n, P;
    pg_dtype dt;
    // reference-numbered structure (exec_engine.hpp:97-110)
    std::vector<uint32_t> shared_ids;
    std::vector<std::vector<uint32_t>> res_ids;
    std::vector<std::vector<uint8_t>> use_shared;
    std::vector<size_t> ref_offset;
    // device arena: slot runs aligned to kSlotAlign
    int s_pad;
    std::vector<int> dev_off, cnt_pad;
    int arena_cols;
    void* bt_arena;  // [arena_cols, ldb]
    int64_t ldb;
    void* a_arena;   // [m, lda] lda = arena_cols
    int64_t lda;
    uint8_t* masks;   // [P, s_pad]
    std::vector<char> mask_full;  // pattern p uses every shared expert: no activity mask needed
    int32_t* table;   // [P, 2] (run1_start, run1_len)
    size_t bytes;
};
struct pg_cache_s {
    int d;
    size_t capacity, size;
    double min_sim;
    double* emb;
    double* sim;
    double* bnd;
    double* out_f64;
    int32_t* out_i32;
    int* flag;
    double* pinned_f64;
    int32_t* pinned_i32;
};

#define PG_API_BEGIN try {
#define PG_API_END                                                \
    return PG_OK;                                                 \
    }                                                             \
    catch (const ::pg::Error& e) {                                \
        ::pg::set_error(e.code, e.msg);                           \
        return e.code;                                            \
    }                                                             \
    catch (const std::bad_alloc&) {                               \
        ::pg::set_error(PG_RUNTIME_ERROR, "host allocation failed"); \
        return PG_RUNTIME_ERROR;                                  \
    }

static void require(bool ok, int code, const char* msg) {
    if (!ok) throw Error{code, msg};
}

extern "C" {

const char* pg_last_error(void) { return t_err.c_str(); }
int pg_abi_version(void) { return 1; }
uint64_t pg_launch_count(void) { return g_launches.load(); }

// ------------------------------------------------------------ routing
int pg_mean_pool(const void* x, pg_dtype dt, pg_layout lay, size_t n, const int64_t* offs,
                 size_t P, double* h, pg_stream s) {
    PG_API_BEGIN
    require(x && h && offs && P > 0 && n > 0, PG_INVALID_ARGUMENT, "mean_pool: bad arguments");
    const cudaStream_t st = as_stream(s);
    Scratch od((P + 1) * 8, st);
    PG_CUDA_THROW(cudaMemcpyAsync(od.p, offs, (P + 1) * 8, cudaMemcpyHostToDevice, st));
    launch_mean_pool(x, dt, lay, (int)n, offs[P], od.as<int64_t>(), (int)P, h, st);
    PG_API_END
}

int pg_router_create(pg_router* out, size_t r, size_t n, const double* theta, const double* bias) {
    PG_API_BEGIN
    require(out && theta && bias && r > 0 && n > 0, PG_INVALID_ARGUMENT, "router: bad arguments");
    auto* R = new pg_router_s{(int)r, (int)n, nullptr, nullptr, true};
    R->theta = static_cast<double*>(dev_alloc(r * n * 8));
    R->bias = static_cast<double*>(dev_alloc(r * 8));
    PG_CUDA_THROW(cudaMemcpy(R->theta, theta, r * n * 8, cudaMemcpyHostToDevice));
    PG_CUDA_THROW(cudaMemcpy(R->bias, bias, r * 8, cudaMemcpyHostToDevice));
    *out = R;
    PG_API_END
}

int pg_router_create_device(pg_router* out, size_t r, size_t n, const double* theta,
                            const double* bias, int copy) {
    PG_API_BEGIN
    require(out && theta && bias && r > 0 && n > 0, PG_INVALID_ARGUMENT, "router: bad arguments");
    auto* R = new pg_router_s{(int)r, (int)n, const_cast<double*>(theta), const_cast<double*>(bias), false};
    if (copy) {
        R->theta = static_cast<double*>(dev_alloc(r * n * 8));
        R->bias = static_cast<double*>(dev_alloc(r * 8));
        PG_CUDA_THROW(cudaMemcpy(R->theta, theta, r * n * 8, cudaMemcpyDeviceToDevice));
        PG_CUDA_THROW(cudaMemcpy(R->bias, bias, r * 8, cudaMemcpyDeviceToDevice));
        R->owned = true;
    }
    *out = R;
    PG_API_END
}

int pg_router_destroy(pg_router R) {
    PG_API_BEGIN
    if (!R) return PG_OK;
    if (R->owned) {
        cudaFree(R->theta);
        cudaFree(R->bias);
    }
    delete R;
    PG_API_END
}

int pg_score(pg_router R, const double* h, size_t P, double* logits, int exact, pg_stream s) {
    PG_API_BEGIN
    require(R && h && logits && P > 0, PG_INVALID_ARGUMENT, "score: bad input length");
    Scratch hn(exact ? 0 : P * 8, as_stream(s));
    launch_score(R->theta, R->bias, R->r, R->n, h, (int)P, logits, nullptr, exact ? 1 : 0,
                 as_stream(s), hn.as<double>());
    PG_API_END
}

int pg_select_topk(const double* logits, size_t r, size_t P, size_t k, uint32_t* sel, pg_stream s) {
    PG_API_BEGIN
    require(k != 0 && k <= r, PG_INVALID_ARGUMENT, "select_topk: K out of range");
    require(logits && sel && P > 0, PG_INVALID_ARGUMENT, "select_topk: bad arguments");
    require((int)r <= max_select_rows(), PG_INVALID_ARGUMENT, "select_topk: too many experts for device top-k");
    launch_select_topk(logits, (int)r, (int)P, (int)k, sel, as_stream(s));
    PG_API_END
}

int pg_route_select(pg_router R, const void* x, pg_dtype dt, pg_layout lay, const int64_t* offs,
                    size_t P, size_t k, uint32_t* sel, double* logits_out, pg_stream s) {
    PG_API_BEGIN
    require(R && x && offs && sel && P > 0, PG_INVALID_ARGUMENT, "route_select: bad arguments");
    require(k != 0 && k <= (size_t)R->r, PG_INVALID_ARGUMENT, "select_topk: K out of range");
    require(R->r <= max_select_rows(), PG_INVALID_ARGUMENT, "select_topk: too many experts for device top-k");
    const cudaStream_t st = as_stream(s);
    const size_t r = R->r, n = R->n;
    // sub-buffers 256-byte aligned (the GEMV reads h / theta with 16-byte loads)
    const size_t o_h = round_up((P + 1) * 8, 256), o_z = o_h + round_up(P * n * 8, 256),
                 o_b = o_z + round_up(P * r * 8, 256), o_n = o_b + round_up(P * r * 8, 256);
    Scratch ws(o_n + P * 8, st);
    int64_t* od = ws.as<int64_t>();
    double* h = reinterpret_cast<double*>(ws.as<char>() + o_h);
    double* z = reinterpret_cast<double*>(ws.as<char>() + o_z);
    double* bnd = reinterpret_cast<double*>(ws.as<char>() + o_b);
    PG_CUDA_THROW(cudaMemcpyAsync(od, offs, (P + 1) * 8, cudaMemcpyHostToDevice, st));
    launch_mean_pool(x, dt, lay, (int)n, offs[P], od, (int)P, h, st);
    launch_score(R->theta, R->bias, (int)r, (int)n, h, (int)P, z, bnd, 0, st,
                 reinterpret_cast<double*>(ws.as<char>() + o_n));
    launch_route_select(z, bnd, R->theta, R->bias, h, (int)r, (int)n, (int)k, (int)P, sel,
                        logits_out, nullptr, st);
    PG_API_END
}

int pg_route_select_pooled(pg_router R, const double* h, size_t P, size_t k, uint32_t* sel, double* logits_out,
                           pg_stream s) {
    PG_API_BEGIN
    require(R && h && sel && P > 0, PG_INVALID_ARGUMENT, "route_select: bad arguments");
    require(k != 0 && k <= (size_t)R->r, PG_INVALID_ARGUMENT, "select_topk: K out of range");
    require(R->r <= max_select_rows(), PG_INVALID_ARGUMENT, "select_topk: too many experts for device top-k");
    const cudaStream_t st = as_stream(s);
    const size_t r = R->r, n = R->n;
    const size_t o_b = round_up(P * r * 8, 256), o_n = o_b + round_up(P * r * 8, 256);
    Scratch ws(o_n + P * 8, st);
    double* z = ws.as<double>();
    double* bnd = reinterpret_cast<double*>(ws.as<char>() + o_b);
    launch_score(R->theta, R->bias, (int)r, (int)n, h, (int)P, z, bnd, 0, st,
                 reinterpret_cast<double*>(ws.as<char>() + o_n));
    launch_route_select(z, bnd, R->theta, R->bias, h, (int)r, (int)n, (int)k, (int)P, sel, logits_out, nullptr,
                        st);
    PG_API_END
}

// ------------------------------------------------------------ cache
int pg_cosine(const double* a, const double* b, size_t d, double* out, pg_stream s) {
    PG_API_BEGIN
    require(a && b && out && d > 0, PG_INVALID_ARGUMENT, "cosine: length mismatch");
    launch_cosine_exact(a, b, (int)d, out, as_stream(s));
    PG_API_END
}

int pg_cache_create(pg_cache* out, size_t d, size_t capacity, double min_sim) {
    PG_API_BEGIN
    require(out && d > 0, PG_INVALID_ARGUMENT, "cache: bad arguments");
    require((int)d <= max_cache_dim(), PG_INVALID_ARGUMENT, "cache: d_model too large");
    auto* c = new pg_cache_s{};
    c->d = (int)d;
    c->capacity = capacity;
    c->size = 0;
    c->min_sim = min_sim;
    const size_t cap = std::max<size_t>(capacity, 1);
    c->emb = static_cast<double*>(dev_alloc(cap * d * 8));
    c->sim = static_cast<double*>(dev_alloc(cap * 8));
    c->bnd = static_cast<double*>(dev_alloc(cap * 8));
    c->out_f64 = static_cast<double*>(dev_alloc(16));
    c->out_i32 = static_cast<int32_t*>(dev_alloc(16));
    c->flag = static_cast<int*>(dev_alloc(16));
    PG_CUDA_THROW(cudaMallocHost(&c->pinned_f64, 16));
    PG_CUDA_THROW(cudaMallocHost(&c->pinned_i32, 16));
    *out = c;
    PG_API_END
}

int pg_cache_destroy(pg_cache c) {
    PG_API_BEGIN
    if (!c) return PG_OK;
    cudaFree(c->emb); cudaFree(c->sim); cudaFree(c->bnd);
    cudaFree(c->out_f64); cudaFree(c->out_i32); cudaFree(c->flag);
    cudaFreeHost(c->pinned_f64); cudaFreeHost(c->pinned_i32);
    delete c;
    PG_API_END
}

int pg_cache_size(pg_cache c, size_t* out) {
    PG_API_BEGIN
    require(c && out, PG_INVALID_ARGUMENT, "cache: bad arguments");
    *out = c->size;
    PG_API_END
}

int pg_cache_insert(pg_cache c, const double* emb, int on_dev, int* inserted, pg_stream s) {
    PG_API_BEGIN
    require(c && emb, PG_INVALID_ARGUMENT, "cache_insert: bad arguments");
    if (c->size >= c->capacity) {  // pattern_cache.hpp:121 -- refused, no eviction
        if (inserted) *inserted = 0;
        return PG_OK;
    }
    PG_CUDA_THROW(cudaMemcpyAsync(c->emb + c->size * c->d, emb, (size_t)c->d * 8,
                                  on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                  as_stream(s)));
    c->size += 1;
    if (inserted) *inserted = 1;
    PG_API_END
}

int pg_cache_load(pg_cache c, const double* emb, size_t N) {
    PG_API_BEGIN
    require(c && (emb || N == 0), PG_INVALID_ARGUMENT, "cache: bad arguments");
    require(N <= c->capacity, PG_INVALID_ARGUMENT, "cache: more entries than capacity");
    if (N) PG_CUDA_THROW(cudaMemcpy(c->emb, emb, N * c->d * 8, cudaMemcpyHostToDevice));
    c->size = N;
    PG_API_END
}

int pg_retrieve(pg_cache c, const double* q, int exact_sim, pg_retrieve_result* res,
                int32_t* entry_dev, int32_t* hit_dev, pg_stream s) {
    PG_API_BEGIN
    require(c && q, PG_INVALID_ARGUMENT, "retrieve: bad arguments");
    if (c->size == 0) throw Error{PG_RUNTIME_ERROR, "empty cache"};
    const cudaStream_t st = as_stream(s);
    launch_cosine_scan(c->emb, q, (int)c->size, c->d, c->sim, c->bnd, st);
    launch_retrieve_select(c->sim, c->bnd, c->emb, q, (int)c->size, c->d, c->min_sim, exact_sim,
                           c->out_f64, c->out_i32, entry_dev, hit_dev, st);
    if (res) {
        PG_CUDA_THROW(cudaMemcpyAsync(c->pinned_f64, c->out_f64, 8, cudaMemcpyDeviceToHost, st));
        PG_CUDA_THROW(cudaMemcpyAsync(c->pinned_i32, c->out_i32, 16, cudaMemcpyDeviceToHost, st));
        PG_CUDA_THROW(cudaStreamSynchronize(st));
        res->similarity = c->pinned_f64[0];
        res->entry = (size_t)c->pinned_i32[0];
        res->hit = c->pinned_i32[1];
        res->exact_similarity = c->pinned_i32[2];
    }
    PG_API_END
}

int pg_embed_normalize(const void* x, pg_dtype dt, pg_layout lay, size_t d, size_t T, double* emb,
                       pg_stream s) {
    PG_API_BEGIN
    require(x && emb && d > 0, PG_INVALID_ARGUMENT, "embed_prompt: bad arguments");
    require(T > 0, PG_INVALID_ARGUMENT, "embed_prompt: empty prompt");
    const cudaStream_t st = as_stream(s);
    Scratch ws(32, st);
    int64_t offs[2] = {0, (int64_t)T};
    PG_CUDA_THROW(cudaMemcpyAsync(ws.p, offs, 16, cudaMemcpyHostToDevice, st));
    launch_mean_pool(x, dt, lay, (int)d, (int64_t)T, ws.as<int64_t>(), 1, emb, st);
    int* flag = reinterpret_cast<int*>(ws.as<int64_t>() + 2);
    launch_embed_finish(emb, (int)d, flag, st);
    int hflag = 0;
    PG_CUDA_THROW(cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, st));
    PG_CUDA_THROW(cudaStreamSynchronize(st));
    if (hflag) throw Error{PG_RUNTIME_ERROR, "degenerate embedding"};
    PG_API_END
}

// ------------------------------------------------------------ layers
static int64_t padded_ld(size_t cols, pg_dtype dt) {
    const size_t per = 16 / dtype_size(dt);
    return (int64_t)round_up(cols, per);
}

int pg_layer_create(pg_layer* out, size_t m, size_t n, size_t r, size_t K, const double* A,
                    const double* B, pg_dtype dt) {
    PG_API_BEGIN
    require(out && A && B && m && n && r, PG_INVALID_ARGUMENT, "layer: bad arguments");
    require(K <= r, PG_INVALID_ARGUMENT, "layer: K > r_store");
    const size_t es = dtype_size(dt);
    const int64_t ldb = padded_ld(n, dt), lda = padded_ld(r, dt);
    // B (n x r) -> B^T (r x ldb); A (m x r) -> (m x lda)
    std::vector<double> bt((size_t)r * ldb, 0.0), ap((size_t)m * lda, 0.0);
    for (size_t j = 0; j < n; ++j)
        for (size_t e = 0; e < r; ++e) bt[e * ldb + j] = B[j * r + e];
    for (size_t i = 0; i < m; ++i)
        for (size_t e = 0; e < r; ++e) ap[i * lda + e] = A[i * r + e];
    std::vector<unsigned char> tb(bt.size() * es), ta(ap.size() * es);
    convert_store(bt.data(), bt.size(), dt, tb.data());
    convert_store(ap.data(), ap.size(), dt, ta.data());
    auto* L = new pg_layer_s{(int)m, (int)n, (int)r, (int)K, dt, nullptr, ldb, nullptr, lda, true};
    L->bt = dev_alloc(tb.size());
    L->a = dev_alloc(ta.size());
    PG_CUDA_THROW(cudaMemcpy(L->bt, tb.data(), tb.size(), cudaMemcpyHostToDevice));
    PG_CUDA_THROW(cudaMemcpy(L->a, ta.data(), ta.size(), cudaMemcpyHostToDevice));
    *out = L;
    PG_API_END
}

int pg_layer_create_device(pg_layer* out, size_t m, size_t n, size_t r, size_t K, const void* bt,
                           const void* a, pg_dtype dt, int copy) {
    PG_API_BEGIN
    require(out && bt && a && m && n && r, PG_INVALID_ARGUMENT, "layer: bad arguments");
    require(K <= r, PG_INVALID_ARGUMENT, "layer: K > r_store");
    const size_t es = dtype_size(dt);
    auto* L = new pg_layer_s{(int)m, (int)n, (int)r, (int)K, dt, const_cast<void*>(bt), (int64_t)n,
                             const_cast<void*>(a), (int64_t)r, false};
    const int64_t ldb = padded_ld(n, dt), lda = padded_ld(r, dt);
    if (copy || ldb != (int64_t)n || lda != (int64_t)r) {
        L->bt = dev_alloc((size_t)r * ldb * es);
        L->a = dev_alloc((size_t)m * lda * es);
        PG_CUDA_THROW(cudaMemset(L->bt, 0, (size_t)r * ldb * es));
        PG_CUDA_THROW(cudaMemset(L->a, 0, (size_t)m * lda * es));
        PG_CUDA_THROW(cudaMemcpy2D(L->bt, ldb * es, bt, n * es, n * es, r, cudaMemcpyDeviceToDevice));
        PG_CUDA_THROW(cudaMemcpy2D(L->a, lda * es, a, r * es, r * es, m, cudaMemcpyDeviceToDevice));
        L->ldb = ldb;
        L->lda = lda;
        L->owned = true;
    }
    *out = L;
    PG_API_END
}

int pg_layer_destroy(pg_layer L) {
    PG_API_BEGIN
    if (!L) return PG_OK;
    if (L->owned) {
        cudaFree(L->bt);
        cudaFree(L->a);
    }
    delete L;
    PG_API_END
}

int pg_layer_info(pg_layer L, size_t* m, size_t* n, size_t* r, size_t* K, pg_dtype* dt) {
    PG_API_BEGIN
    require(L, PG_INVALID_ARGUMENT, "layer: null");
    if (m) *m = L->m;
    if (n) *n = L->n;
    if (r) *r = L->r;
    if (K) *K = L->K;
    if (dt) *dt = L->dt;
    PG_API_END
}

static void check_sel_host(const uint32_t* sel, size_t k, size_t r) {  // rank_experts.hpp:30-37
    if (k == 0) throw Error{PG_INVALID_ARGUMENT, "selection must be non-empty"};
    for (size_t i = 1; i < k; ++i)
        if (sel[i] <= sel[i - 1])
            throw Error{PG_INVALID_ARGUMENT, "selection indices not strictly increasing"};
    if (sel[k - 1] >= r) throw Error{PG_OUT_OF_RANGE, "selection index beyond r_store"};
}

int pg_check_selection(pg_layer L, const uint32_t* sel, size_t k) {
    PG_API_BEGIN
    require(L, PG_INVALID_ARGUMENT, "layer: null");
    check_sel_host(sel, k, (size_t)L->r);
    PG_API_END
}

static void check_ydt(pg_dtype wdt, pg_dtype ydt) {
    if (!(ydt == wdt || ydt == PG_F32 || (wdt == PG_F64 && ydt == PG_F64)))
        throw Error{PG_INVALID_ARGUMENT, "forward: unsupported output dtype"};
    if (wdt == PG_F64 && ydt != PG_F64)
        throw Error{PG_INVALID_ARGUMENT, "forward: f64 layers produce f64 output"};
}

// Two-stage contraction over a slot map: decode GEMV when T is small and the
// operands fit shared memory, SIMT GEMM otherwise (bf16 large-T goes to the
// tensor-core path once enabled).
// Optional per-CTA phase timestamps (PG_CHAIN_DBG=1), read by pg_chain_debug_dump.
static unsigned long long* g_chain_dbg = nullptr;
static unsigned long long* chain_debug_buffer() {
    static const bool on = [] {
        const char* e = getenv("PG_CHAIN_DBG");
        return e && atoi(e);
    }();
    if (on && !g_chain_dbg) {
        PG_CUDA_THROW(cudaMalloc(&g_chain_dbg, 1024 * 16 * 8));
        PG_CUDA_THROW(cudaMemset(g_chain_dbg, 0, 1024 * 16 * 8));
    }
    return on ? g_chain_dbg : nullptr;
}

// One linear of a decode chain (T = 1).
struct LinSpec {
    const void* bt;
    int64_t ldb;
    const void* a;
    int64_t lda;
    SlotMap sm;
    int cap, n, m;
    void* y;
};

// Single-launch decode chain (decode.cu).  phases[0] = linears sharing x; when
// mlp is set, phase 0 is {up, gate} with the silu epilogue into act and phase
// 1 is {down} reading act.
// Decode-chain workspace per (device, stream, grid size): [barrier counter |
// epoch | z | act].  Grows outside graph capture only; reused by every launch
// on that stream with that grid.  Keyed by grid size because the monotone
// barrier counter and the launch epoch count in units of the grid size.
// pg_chain_workspace_release(stream) frees a stream's workspaces (call it
// before destroying a per-request stream).
static std::mutex g_ws_mu;
// `owner` separates workspaces whose launch epochs must advance independently
// of other chain launches on the same stream: the expert-sharded peer path keys
// its workspace by this rank's receive buffer, so its tags count only that
// PeerReduceLinear's launches (identical on every rank) and an unrelated chain
// launch on one rank cannot desynchronise the ranks' tags.
static std::map<std::tuple<int, cudaStream_t, int, const void*>, std::pair<char*, size_t>> g_ws;
static char* chain_workspace(cudaStream_t st, size_t bytes, int grid, const void* owner = nullptr) {
    int dev = 0;
    PG_CUDA_THROW(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto& w = g_ws[std::make_tuple(dev, st, grid, owner)];
    if (w.second < bytes) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        PG_CUDA_THROW(cudaStreamIsCapturing(st, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            throw Error{PG_RUNTIME_ERROR, "decode chain: workspace must be sized by a call before graph capture"};
        PG_CUDA_THROW(cudaStreamSynchronize(st));
        if (w.first) PG_CUDA_THROW(cudaFree(w.first));
        const size_t sz = round_up(bytes, 1 << 20);
        PG_CUDA_THROW(cudaMalloc(&w.first, sz));
        // on the launching stream: a user stream created non-blocking is not
        // ordered after the legacy default stream a plain cudaMemset runs on
        PG_CUDA_THROW(cudaMemsetAsync(w.first, 0, sz, st));
        w.second = sz;
    }
    return w.first;
}

static size_t chain_tab_bytes(size_t nphase) { return std::max<size_t>(1024, round_up(nphase * kMaxLin * kLinSBytes, 128)); }

// Chain feasibility: contiguous runs only (no gather list) and the largest
// streamed item (a B^T row, or an up/gate A-row pair) fits one ring stage.
static size_t chain_chunk_bytes(pg_dtype wdt, const std::vector<std::vector<LinSpec>>& phases, bool mlp,
                                size_t* xs_bytes, size_t* zs_bytes) {
    const size_t accs = wdt == PG_F64 ? 8 : 4, es = dtype_size(wdt);
    size_t xs = 16, zs = 16, item = 16;
    for (size_t p = 0; p < phases.size(); ++p) {
        const auto& ph = phases[p];
        size_t zsum = 0, pair = 0;
        for (const auto& l : ph) {
            if (l.sm.idx) return 0;
            xs = std::max(xs, round_up((size_t)l.n * es + 16, 128));
            zsum += round_up(l.cap, 4) * accs;
            item = std::max(item, (size_t)l.ldb * es);
            item = std::max(item, (size_t)l.cap * es);
            pair += (size_t)l.cap * es;
        }
        if (mlp && p % 2 == 0) item = std::max(item, pair);  // up/gate A-row pairs
        zs = std::max(zs, round_up(zsum, 128));
    }
    *xs_bytes = xs;
    *zs_bytes = zs;
    const size_t fixed = chain_tab_bytes(phases.size()) + xs + zs + kRingStages * (128 + 16) + 128;
    const size_t kMaxSmem = 227 * 1024;
    if (fixed + 2 * item > kMaxSmem) return 0;  // need >= 2 stages in flight
    static const int div_env = [] {  // experiments: size chunks for this many stages
        const char* e = getenv("PG_CHAIN_CHUNK_DIV");
        return e ? std::max(2, std::min(atoi(e), kRingStages)) : kRingStages;
    }();
    size_t ch = (kMaxSmem - fixed) / div_env / 128 * 128;
    return std::max(ch, round_up(item, 128));
}

static bool chain_ok(pg_dtype wdt, const std::vector<std::vector<LinSpec>>& phases, bool mlp) {
    size_t a, b;
    return chain_chunk_bytes(wdt, phases, mlp, &a, &b) != 0;
}

// Single-launch decode chain (decode.cu).  phases[0] = linears sharing x; when
// mlp is set, phase 0 is {up, gate} with the silu epilogue into act and phase
// 1 is {down} reading act.
struct PeerSpec {  // expert-sharded peer reduction (ChainParams::npeer)
    int rank = 0, npeer = 0, grid = 0;
    void* const* bufs = nullptr;
};

// Per-phase inputs of a chain: x (the phase input), act (MLP epilogue target,
// also the next phase's input), epilogue kind.  A chain of S MLP blocks has
// 2S phases: {up_s, gate_s} (epilogue 1 into act_s) and {down_s} (x = act_s,
// y_s); block s+1 reads y_s.
struct ChainIO {
    std::vector<const void*> x;
    std::vector<void*> act;
    std::vector<int> epi;
};

static void run_chain_io(pg_dtype wdt, const std::vector<std::vector<LinSpec>>& phases, ChainIO io, bool mlp,
                         pg_dtype ydt, cudaStream_t st, const PeerSpec* peer);

static void run_chain(pg_dtype wdt, const std::vector<std::vector<LinSpec>>& phases, const void* x,
                      bool mlp, void* act, pg_dtype ydt, cudaStream_t st, const PeerSpec* peer = nullptr) {
    ChainIO io;
    for (size_t p = 0; p < phases.size(); ++p) {
        io.x.push_back(p == 0 ? x : nullptr);  // null: the workspace act (MLP phase 1)
        io.act.push_back(act);
        io.epi.push_back((mlp && p == 0) ? 1 : 0);
    }
    run_chain_io(wdt, phases, io, mlp, ydt, st, peer);
}

static void run_chain_io(pg_dtype wdt, const std::vector<std::vector<LinSpec>>& phases, ChainIO io, bool mlp,
                         pg_dtype ydt, cudaStream_t st, const PeerSpec* peer) {
    const size_t accs = wdt == PG_F64 ? 8 : 4, es = dtype_size(wdt);
    if (phases.empty() || phases.size() > (size_t)kMaxPhase)
        throw Error{PG_INVALID_ARGUMENT, "decode chain: 1..16 phases"};
    ChainParams P = {};
    P.nphase = (int)phases.size();
    P.tab_bytes = (int)chain_tab_bytes(phases.size());
    size_t xs_bytes = 0, zs_bytes = 0;
    const size_t ch = chain_chunk_bytes(wdt, phases, mlp, &xs_bytes, &zs_bytes);
    if (!ch) throw Error{PG_INVALID_ARGUMENT, "decode chain: operands exceed shared memory"};
    P.xs_bytes = (int)xs_bytes;
    P.zs_bytes = (int)zs_bytes;
    P.chunk_bytes = (int)ch;
    // ring depth: measured on three boxes, the MLP launch is 7-9 % faster with
    // 7 of the 8 stages (fewer bytes in flight shorten its cross-CTA exchanges
    // more than they cost streaming); single-linear launches keep all 8
    static const int stages_env = [] {
        const char* e = getenv("PG_CHAIN_STAGES");
        return e ? std::max(2, std::min(atoi(e), kRingStages)) : 0;
    }();
    P.max_stages = stages_env ? stages_env : (mlp ? kRingStages - 1 : kRingStages);
    // producer throttle across the z exchange: after a stage-1 segment at most 3
    // chunks are issued until the consumers have the exchanged z (less HBM
    // traffic queued ahead of the exchange); measured -2 % per MLP step
    static const int throttle_env = [] {
        const char* e = getenv("PG_CHAIN_THROTTLE");
        return e ? atoi(e) : -2;
    }();
    P.throttle = throttle_env != -2 ? throttle_env : (mlp ? 3 : -1);
    // weights are streamed once per launch: L2 evict-first keeps them from
    // displacing the exchange words (measured -2 % per MLP step)
    static const int l2hint_env = [] {
        const char* e = getenv("PG_CHAIN_L2HINT");
        return e ? atoi(e) : 1;
    }();
    P.l2hint = l2hint_env;
    P.dbg = chain_debug_buffer();
    const size_t zw = wdt == PG_F64 ? 2 : 1;  // tagged exchange words per z value
    size_t zbytes = 256;
    for (auto& ph : phases)
        for (auto& l : ph) zbytes += round_up((size_t)l.cap * zw * 8, 256);
    // workspace act for MLP blocks given none (one per block: a block's act is
    // read by its down phase while the next block may already write its own)
    size_t act_bytes = 0;
    std::vector<size_t> act_off(phases.size(), (size_t)-1);
    for (size_t p = 0; p < phases.size(); ++p)
        if (io.epi[p] == 1 && !io.act[p]) {
            act_off[p] = act_bytes;
            act_bytes += round_up((size_t)phases[p][0].m * es, 256);
        }
    // Persistent per-stream workspace: [barrier counter | epoch | z words | act].
    // The barrier counter is monotone (every launch adds a multiple of the grid
    // size) and z words carry their launch's tag, so consecutive chain launches
    // need no memset between them and can overlap under programmatic dependent
    // launch.
    static const int grid_env = [] {  // experiments: decode-chain grid size (default: every SM)
        const char* e = getenv("PG_CHAIN_GRID");
        return e ? atoi(e) : 0;
    }();
    // MLP launches leave 4 SMs free: the next launch's first CTAs (programmatic
    // dependent launch) start streaming their weights during this launch's tail
    // (measured ~1 % per step on three boxes)
    int grid = grid_env ? grid_env : (mlp ? std::max(1, chain_grid() - 4) : 0);
    if (peer && peer->npeer > 0) grid = peer->grid;
    const int eff_grid = grid > 0 ? std::min(grid, chain_grid()) : chain_grid();
    char* base = chain_workspace(st, zbytes + act_bytes, eff_grid,
                                 (peer && peer->npeer > 0) ? peer->bufs[peer->rank] : nullptr);
    P.bar = reinterpret_cast<unsigned long long*>(base);
    P.epoch = reinterpret_cast<unsigned long long*>(base + 64);
    // measured: tagged z words win for the 2-phase MLP launch (30.5 vs 31.7 us
    // per step), the fenced barrier for single-linear launches (13.6 vs 20.8 us)
    static const int ztag_env = [] {
        const char* e = getenv("PG_CHAIN_ZTAG");
        return e ? atoi(e) : -1;
    }();
    // and for single-phase modules of >= 2 linears (q/k/v, up/gate): 13B q/k/v
    // 34.0 -> 30.0 us, 2-linear 25.6 -> 22.0; 7B q/k/v 20.5 -> 18.2, up/gate
    // 24.3 -> 21.8 (tools/experiments/exp_c5_qkvo.py)
    const bool multi = phases.size() == 1 && phases[0].size() >= 2;
    P.ztag = ztag_env >= 0 ? ztag_env : ((mlp || multi) ? 1 : 0);
    size_t off = 256;
    for (size_t p = 0; p < phases.size(); ++p)
        if (act_off[p] != (size_t)-1) io.act[p] = base + zbytes + act_off[p];
    for (size_t p = 0; p < phases.size(); ++p) {
        ChainPhase& Q = P.ph[p];
        Q.nlin = (int)phases[p].size();
        // a phase without an explicit x reads the previous phase's act
        Q.x = io.x[p] ? io.x[p] : (p > 0 ? io.act[p - 1] : nullptr);
        if (!Q.x) throw Error{PG_INVALID_ARGUMENT, "decode chain: phase without input"};
        Q.epilogue = io.epi[p];
        Q.ydt = ydt;
        Q.act = io.act[p];
        for (int l = 0; l < Q.nlin; ++l) {
            const LinSpec& S = phases[p][l];
            ChainLin& L = Q.lin[l];
            L.bt = S.bt; L.ldb = S.ldb; L.a = S.a; L.lda = S.lda; L.sm = S.sm; L.cap = S.cap;
            L.n = S.n; L.m = S.m; L.y = S.y;
            L.zpart = base + off;
            off += round_up((size_t)S.cap * zw * 8, 256);
        }
    }
    if (peer && peer->npeer > 0) {
        P.npeer = peer->npeer;
        P.prank = peer->rank;
        for (int r = 0; r < peer->npeer; ++r) P.peer_recv[r] = static_cast<unsigned long long*>(peer->bufs[r]);
        // words per (parity, rank): one linear's m rows, or an MLP block's up
        // and gate rows (reduced into act mid-launch) followed by down's rows
        if (mlp) {
            if (phases.size() != 2) throw Error{PG_INVALID_ARGUMENT, "decode chain: peer MLP is one block"};
            P.peer_words = 2 * phases[0][0].m + phases[1][0].m;
            P.peer_last_off = 2 * phases[0][0].m;
        } else {
            if (phases.size() != 1) throw Error{PG_INVALID_ARGUMENT, "decode chain: peer launch is one linear"};
            P.peer_words = phases[0][0].m;
            P.peer_last_off = 0;
        }
    }
    const size_t total = chain_tab_bytes(phases.size()) + xs_bytes + zs_bytes + kRingStages * (128 + 16) + 128 +
                         (size_t)kRingStages * ch;
    launch_chain(wdt, P, std::min(total, (size_t)227 * 1024), st, grid);
}

// ---- bf16 prefill on the tensor cores (umma.cu): stage 1 and stage 2 of every
// job are one grouped launch each.  Jobs whose slot map has a second run or an
// activity mask are first gathered into a contiguous [ns] arena (masked slots
// become zero rows, so their z is exactly 0).
struct PrefillJob {
    const void* bt;
    int64_t ldb;
    const void* a;
    int64_t lda;
    SlotMap sm;
    int n, m;
    const void* x;  // token-major [T, n] bf16
    int T;
    void* y;        // token-major [T, m]
    pg_dtype ydt;
};

static bool prefill_ok(int n, int T) { return T > 8 && n % 8 == 0; }

static void run_prefill(const std::vector<PrefillJob>& jobs, cudaStream_t st) {
    const size_t es = 2;
    // workspace: packed operands (when needed) + Z per job
    std::vector<size_t> zoff(jobs.size()), poff(jobs.size(), (size_t)-1);
    size_t bytes = 0;
    for (size_t j = 0; j < jobs.size(); ++j) {
        const PrefillJob& J = jobs[j];
        const int ns = J.sm.nslots();
        const bool pack = J.sm.idx || J.sm.run1_len || J.sm.mask;
        if (pack) {
            poff[j] = bytes;
            bytes += round_up((size_t)ns * 4, 256) + round_up((size_t)ns * J.ldb * es, 256) +
                     round_up((size_t)J.m * ns * es, 256);
        }
        zoff[j] = bytes;
        bytes += round_up((size_t)J.T * ns * es, 256);
    }
    Scratch ws(bytes, st);
    char* base = ws.as<char>();
    std::vector<UmmaSpec> s1, s2;
    for (size_t j = 0; j < jobs.size(); ++j) {
        const PrefillJob& J = jobs[j];
        const int ns = J.sm.nslots();
        const void* bt = J.bt;
        const void* a = J.a;
        int64_t lda = J.lda;
        if (poff[j] != (size_t)-1) {
            // gather list over the slot map: -1 for inactive (masked) slots
            std::vector<int32_t> idx(ns);
            if (J.sm.idx) {
                PG_CUDA_THROW(cudaMemcpyAsync(idx.data(), J.sm.idx, ns * 4, cudaMemcpyDeviceToHost, st));
                PG_CUDA_THROW(cudaStreamSynchronize(st));
            } else {
                std::vector<uint8_t> mask(J.sm.run0_len, 1);
                if (J.sm.mask) {
                    PG_CUDA_THROW(cudaMemcpyAsync(mask.data(), J.sm.mask, J.sm.run0_len, cudaMemcpyDeviceToHost, st));
                    PG_CUDA_THROW(cudaStreamSynchronize(st));
                }
                for (int s = 0; s < ns; ++s)
                    idx[s] = s < J.sm.run0_len ? (mask[s] ? s : -1) : J.sm.run1_start + (s - J.sm.run0_len);
            }
            char* p = base + poff[j];
            int32_t* didx = reinterpret_cast<int32_t*>(p);
            void* pb = p + round_up((size_t)ns * 4, 256);
            void* pa = static_cast<char*>(pb) + round_up((size_t)ns * J.ldb * es, 256);
            PG_CUDA_THROW(cudaMemcpyAsync(didx, idx.data(), ns * 4, cudaMemcpyHostToDevice, st));
            PG_CUDA_THROW(cudaStreamSynchronize(st));  // idx is host-owned
            launch_gather_rows(PG_BF16, J.bt, J.ldb, didx, ns, ns, J.n, pb, J.ldb, st);
            launch_gather_cols(PG_BF16, J.a, J.lda, didx, ns, ns, J.m, pa, ns, st);
            bt = pb;
            a = pa;
            lda = ns;
        }
        void* z = base + zoff[j];
        s1.push_back(UmmaSpec{J.x, J.n, bt, J.ldb, z, ns, J.T, ns, J.n, 1});
        s2.push_back(UmmaSpec{z, ns, a, lda, J.y, J.m, J.T, J.m, ns, J.ydt == PG_BF16 ? 1 : 0});
    }
    launch_umma(s1, st);
    launch_umma(s2, st);
}

static void run_forward(pg_dtype wdt, const void* bt, int64_t ldb, const void* a, int64_t lda,
                        SlotMap sm, int nslots_max, int n, int m, const void* x, int fm, int T,
                        void* y, pg_dtype ydt, cudaStream_t st) {
    if (T == 0) return;
    const size_t accs = wdt == PG_F64 ? 8 : 4;
    if (T == 1) {
        std::vector<std::vector<LinSpec>> ph = {{LinSpec{bt, ldb, a, lda, sm, nslots_max, n, m, y}}};
        if (chain_ok(wdt, ph, false)) {
            run_chain(wdt, ph, x, false, nullptr, ydt, st);
            return;
        }
    }
    if (wdt == PG_BF16 && prefill_ok(n, T) && !sm.dyn_pattern) {
        // tensor-core prefill; feature-major operands are transposed around it
        const void* xt = x;
        void* yt = y;
        Scratch tx(fm ? (size_t)T * n * 2 : 0, st), ty(fm ? (size_t)T * m * dtype_size(ydt) : 0, st);
        if (fm) {
            launch_transpose(PG_BF16, x, n, T, tx.p, st);  // [n, T] -> [T, n]
            xt = tx.p;
            yt = ty.p;
        }
        run_prefill({PrefillJob{bt, ldb, a, lda, sm, n, m, xt, T, yt, ydt}}, st);
        if (fm) launch_transpose(ydt, ty.p, T, m, y, st);  // [T, m] -> [m, T]
        return;
    }
    if (decode_tmax(T) && decode_smem_need(wdt, n, nslots_max, T) <= 200 * 1024) {
        Scratch z((size_t)nslots_max * T * accs, st);
        sm.cap = nslots_max;
        launch_decode(wdt, bt, ldb, a, lda, sm, n, m, x, fm, T, z.p, y, ydt, st);
        return;
    }
    Scratch ws(simt_ws_elems(n, m, nslots_max, T) * accs, st);
    launch_simt(wdt, bt, ldb, a, lda, sm, n, m, x, fm, T, ws.p, y, ydt, st);
}

int pg_masked_forward(pg_layer L, const uint32_t* sel, size_t k, int sel_on_dev, const void* x,
                      pg_layout lay, size_t T, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(L && sel && x && y, PG_INVALID_ARGUMENT, "masked_forward: bad X shape");
    if (!sel_on_dev) check_sel_host(sel, k, (size_t)L->r);
    else require(k > 0 && k <= (size_t)L->r, PG_INVALID_ARGUMENT, "selection must be non-empty");
    check_ydt(L->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const int fm = lay == PG_FEATURE_MAJOR && T > 1;
    const int ki = (int)k;
    Scratch idx(k * 4, st);
    PG_CUDA_THROW(cudaMemcpyAsync(idx.p, sel, k * 4, sel_on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (decode_tmax((int)T) && decode_smem_need(L->dt, L->n, ki, (int)T) <= 200 * 1024) {
        SlotMap sm;
        sm.idx = idx.as<int32_t>();
        sm.run0_len = ki;
        run_forward(L->dt, L->bt, L->ldb, L->a, L->lda, sm, ki, L->n, L->m, x, fm, (int)T, y, ydt, st);
        return PG_OK;
    }
    // large T: expert gather into a packed [K_pad] arena, then the GEMM path
    const int kp = (int)round_up(k, kSlotAlign);
    const size_t es = dtype_size(L->dt);
    Scratch pb((size_t)kp * L->ldb * es, st), pa((size_t)L->m * kp * es, st);
    launch_gather_rows(L->dt, L->bt, L->ldb, idx.as<int32_t>(), ki, kp, L->n, pb.p, L->ldb, st);
    launch_gather_cols(L->dt, L->a, L->lda, idx.as<int32_t>(), ki, kp, L->m, pa.p, kp, st);
    SlotMap sm;
    sm.run0_len = kp;
    run_forward(L->dt, pb.p, L->ldb, pa.p, kp, sm, kp, L->n, L->m, x, fm, (int)T, y, ydt, st);
    PG_API_END
}

// ------------------------------------------------------------ union-masked batches
// Heterogeneous decode batches (BASELINE config 4): every token t carries its
// prompt's selection S_p(t).  Rather than one pass over the weights per prompt,
// the union of the selections -- all r_store experts once a GPU serves more than
// a handful of patterns -- is read ONCE for the whole batch:
//   Z[T, r] = X[T, n] . B^T[r, n]^T, masked per row: Z[t, e] = 0 unless e in S_p(t)
//   Y[T, m] = Z[T, r] . A[m, r]^T
// which is masked_forward (rank_experts.hpp:52-72) for every token: the masked
// experts contribute exact zeros.  Both stages are tcgen05 GEMMs; the mask is
// applied in the stage-1 epilogue (per-row pattern id -> [P, ld] byte mask).
static size_t sel_mask_ld(int r) { return round_up((size_t)r + 32, 64); }

int pg_selection_mask_stride(pg_layer L, size_t* out) {
    PG_API_BEGIN
    require(L && out, PG_INVALID_ARGUMENT, "selection_mask_stride: bad arguments");
    *out = sel_mask_ld(L->r);
    PG_API_END
}

int pg_selection_masks(pg_layer L, const uint32_t* sels, const size_t* ks, size_t P, uint8_t* masks, pg_stream s) {
    PG_API_BEGIN
    require(L && sels && ks && masks && P > 0, PG_INVALID_ARGUMENT, "selection_masks: bad arguments");
    const size_t ld = sel_mask_ld(L->r);
    std::vector<uint8_t> h(P * ld, 0);
    size_t off = 0;
    for (size_t p = 0; p < P; ++p) {
        check_sel_host(sels + off, ks[p], (size_t)L->r);
        for (size_t q = 0; q < ks[p]; ++q) h[p * ld + sels[off + q]] = 1;
        off += ks[p];
    }
    const cudaStream_t st = as_stream(s);
    PG_CUDA_THROW(cudaMemcpyAsync(masks, h.data(), h.size(), cudaMemcpyHostToDevice, st));
    PG_CUDA_THROW(cudaStreamSynchronize(st));
    PG_API_END
}

int pg_masked_forward_union(pg_layer L, const uint8_t* masks, size_t P, const int32_t* tok_pat, size_t T,
                            const void* x, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(L && masks && tok_pat && x && y && P > 0 && T > 0, PG_INVALID_ARGUMENT,
            "masked_forward_union: bad arguments");
    require(L->dt == PG_BF16, PG_INVALID_ARGUMENT, "masked_forward_union: bf16 layers (tensor-core path)");
    require(L->n % 8 == 0, PG_INVALID_ARGUMENT, "masked_forward_union: n must be a multiple of 8");
    check_ydt(L->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const int rp = (int)round_up((size_t)L->r, 8);
    Scratch z((size_t)T * rp * 2, st);
    // stage 1 Z = mask(X . B^T), stage 2 Y = Z . A^T.  Per GEMM: the weights-on-M
    // kernel (union_wm.cu, T <= 256) where it wins, else tokens on M with narrow
    // expert tiles covering the SMs (launch_umma; K split across CTAs when long).
    // Either writes Z's padding columns [r, rp) as zeros.
    const WmSpec wa{L->bt, L->ldb, L->r, L->n, x, L->n, z.p, rp, 1, masks, (long long)sel_mask_ld(L->r)};
    const WmSpec wb{L->a, L->lda, L->m, L->r, z.p, rp, y, L->m, ydt == PG_BF16 ? 1 : 0};
    const bool use_a = union_wm_ok((int)T, {wa}), use_b = union_wm_ok((int)T, {wb});
    UmmaSpec s1{x, L->n, L->bt, L->ldb, z.p, rp, (int)T, rp, L->n, 1};
    s1.mask = masks;
    s1.mask_ld = (long long)sel_mask_ld(L->r);
    s1.row_pat = tok_pat;
    s1.b_rows = L->r;
    s1.a_hint = 2;  // the batch's tokens are re-read per N tile: keep them in L2
    s1.b_hint = 1;  // every weight byte is read once per batch: evict first
    UmmaSpec s2{z.p, rp, L->a, L->lda, y, L->m, (int)T, L->m, rp, ydt == PG_BF16 ? 1 : 0};
    s2.a_hint = 2;
    s2.b_hint = 1;
    Scratch ws(std::max(use_a ? 0 : umma_splitk_bytes(s1), use_b ? 0 : umma_splitk_bytes(s2)), st);
    if (use_a) launch_union_wm({wa}, (int)T, tok_pat, st);
    else if (!launch_umma_splitk(s1, ws.p, st)) launch_umma({s1}, st);
    if (use_b) launch_union_wm({wb}, (int)T, nullptr, st);
    else if (!launch_umma_splitk(s2, ws.p, st)) launch_umma({s2}, st);
    PG_API_END
}

int pg_module_forward_union(const pg_layer* Ls, const uint8_t* const* masks, const size_t* Ps, size_t nlin,
                            const int32_t* tok_pat, size_t T, const void* x, void* const* ys, pg_dtype ydt,
                            pg_stream s) {
    PG_API_BEGIN
    require(Ls && masks && Ps && tok_pat && x && ys && nlin >= 1 && nlin <= 32 && T > 0, PG_INVALID_ARGUMENT,
            "module_forward_union: bad arguments");
    std::vector<size_t> zoff(nlin);
    size_t zbytes = 0;
    for (size_t l = 0; l < nlin; ++l) {
        const pg_layer L = Ls[l];
        require(L && masks[l] && ys[l] && Ps[l] > 0, PG_INVALID_ARGUMENT, "module_forward_union: bad arguments");
        require(L->dt == PG_BF16 && L->n == Ls[0]->n && L->n % 8 == 0, PG_INVALID_ARGUMENT,
                "module_forward_union: bf16 linears sharing one input width (multiple of 8)");
        check_ydt(L->dt, ydt);
        zoff[l] = zbytes;
        zbytes += round_up((size_t)T * round_up((size_t)L->r, 8) * 2, 256);
    }
    const cudaStream_t st = as_stream(s);
    Scratch z(zbytes, st);
    // T <= 256: per stage, weights on M with the whole batch as N (union_wm.cu)
    // where that kernel wins, else the tokens-on-M grouped kernel
    std::vector<WmSpec> wm1, wm2;
    for (size_t l = 0; l < nlin; ++l) {
        const pg_layer L = Ls[l];
        const int rp = (int)round_up((size_t)L->r, 8);
        void* zl = z.as<char>() + zoff[l];
        wm1.push_back(WmSpec{L->bt, L->ldb, L->r, L->n, x, L->n, zl, rp, 1, masks[l], (long long)sel_mask_ld(L->r)});
        wm2.push_back(WmSpec{L->a, L->lda, L->m, L->r, zl, rp, ys[l], L->m, ydt == PG_BF16 ? 1 : 0});
    }
    const bool wa = union_wm_ok((int)T, wm1), wb = union_wm_ok((int)T, wm2);
    std::vector<UmmaSpec> s1, s2;
    for (size_t l = 0; l < nlin; ++l) {
        const pg_layer L = Ls[l];
        const int rp = (int)round_up((size_t)L->r, 8);
        void* zl = z.as<char>() + zoff[l];
        UmmaSpec a{x, L->n, L->bt, L->ldb, zl, rp, (int)T, rp, L->n, 1};
        a.mask = masks[l];
        a.mask_ld = (long long)sel_mask_ld(L->r);
        a.row_pat = tok_pat;
        a.b_rows = L->r;
        a.a_hint = 2;  // tokens re-read per N tile: keep; weights read once: evict first
        a.b_hint = 1;
        s1.push_back(a);
        UmmaSpec b{zl, rp, L->a, L->lda, ys[l], L->m, (int)T, L->m, rp, ydt == PG_BF16 ? 1 : 0};
        b.a_hint = 2;
        b.b_hint = 1;
        s2.push_back(b);
    }
    // the linears' first GEMMs share x: one grouped launch per stage (with
    // their K split across the SMs when that pays, see launch_umma_splitk)
    size_t w1 = 0, w2 = 0;
    for (const UmmaSpec& u : s1) w1 += wa ? 0 : umma_splitk_bytes(u);
    for (const UmmaSpec& u : s2) w2 += wb ? 0 : umma_splitk_bytes(u);
    Scratch ws(std::max(w1, w2), st);
    if (wa) launch_union_wm(wm1, (int)T, tok_pat, st);
    else if (!launch_umma_splitk_multi(s1, ws.p, st)) launch_umma(s1, st);
    if (wb) launch_union_wm(wm2, (int)T, nullptr, st);
    else if (!launch_umma_splitk_multi(s2, ws.p, st)) launch_umma(s2, st);
    PG_API_END
}

// ------------------------------------------------------------ union program
// A whole decode step of modules as one persistent launch (union_prog.cu).
// Each module adds two phases: stage 1 into a program-owned Z buffer (the
// selection mask in the epilogue), stage 2 from Z into the caller's outputs.
struct pg_union_prog_s {
    std::unique_ptr<pg::UnionProgram> prog;
    size_t T;
    std::vector<void*> z;  // per module: [T, r_pad] bf16 per linear, program-owned
    ~pg_union_prog_s() {
        for (void* p : z) cudaFree(p);
    }
};

int pg_union_prog_create(pg_union_prog* out, size_t T) {
    PG_API_BEGIN
    require(out && T >= 1 && T <= 256, PG_INVALID_ARGUMENT, "union_prog_create: 1 <= T <= 256");
    auto h = std::make_unique<pg_union_prog_s>();
    h->prog = std::make_unique<UnionProgram>((int)T);
    h->T = T;
    *out = h.release();
    PG_API_END
}

int pg_union_prog_add_module(pg_union_prog H, const pg_layer* Ls, const uint8_t* const* masks, const size_t* Ps,
                             size_t nlin, const void* x, void* const* ys, pg_dtype ydt, size_t tok_off,
                             int weights_reused) {
    PG_API_BEGIN
    require(H && Ls && masks && Ps && x && ys && nlin >= 1 && nlin <= 4, PG_INVALID_ARGUMENT,
            "union_prog_add_module: bad arguments (1..4 linears)");
    const size_t T = H->T;
    std::vector<size_t> zoff(nlin);
    size_t zbytes = 0;
    for (size_t l = 0; l < nlin; ++l) {
        const pg_layer L = Ls[l];
        require(L && masks[l] && ys[l] && Ps[l] > 0, PG_INVALID_ARGUMENT, "union_prog_add_module: bad arguments");
        require(L->dt == PG_BF16 && L->n == Ls[0]->n && L->n % 8 == 0, PG_INVALID_ARGUMENT,
                "union_prog_add_module: bf16 linears sharing one input width (multiple of 8)");
        check_ydt(L->dt, ydt);
        zoff[l] = zbytes;
        zbytes += round_up(T * round_up((size_t)L->r, 8) * 2, 256);
    }
    void* z = dev_alloc(zbytes);
    H->z.push_back(z);
    std::vector<WmSpec> s1, s2;
    for (size_t l = 0; l < nlin; ++l) {
        const pg_layer L = Ls[l];
        const int rp = (int)round_up((size_t)L->r, 8);
        void* zl = static_cast<char*>(z) + zoff[l];
        WmSpec a{L->bt, L->ldb, L->r, L->n, x, L->n, zl, rp, 1, masks[l], (long long)sel_mask_ld(L->r)};
        WmSpec b{L->a, L->lda, L->m, L->r, zl, rp, ys[l], L->m, ydt == PG_BF16 ? 1 : 0};
        a.tok_off = b.tok_off = (int)tok_off;
        a.w_hint = b.w_hint = weights_reused ? 0 : 1;
        s1.push_back(a);
        s2.push_back(b);
    }
    H->prog->add_phase(s1);
    H->prog->add_phase(s2);
    PG_API_END
}

int pg_union_prog_run(pg_union_prog H, const int32_t* tok_pat, pg_stream s) {
    PG_API_BEGIN
    require(H && tok_pat, PG_INVALID_ARGUMENT, "union_prog_run: bad arguments");
    H->prog->run(tok_pat, as_stream(s));
    PG_API_END
}

int pg_union_prog_info(pg_union_prog H, size_t* phases, size_t* grid) {
    PG_API_BEGIN
    require(H, PG_INVALID_ARGUMENT, "union_prog_info: bad arguments");
    if (phases) *phases = (size_t)H->prog->phases();
    if (grid) *grid = (size_t)H->prog->grid();
    PG_API_END
}

int pg_union_prog_debug(pg_union_prog H, uint64_t* out, size_t n, int* have) {
    PG_API_BEGIN
    require(H && out && have, PG_INVALID_ARGUMENT, "union_prog_debug: bad arguments");
    PG_CUDA_THROW(cudaDeviceSynchronize());
    *have = H->prog->debug_dump(reinterpret_cast<unsigned long long*>(out), n);
    PG_API_END
}

int pg_union_prog_destroy(pg_union_prog H) {
    PG_API_BEGIN
    delete H;
    PG_API_END
}

// ------------------------------------------------------------ aggregated layout
int pg_aggregate_layout(pg_agg* out, pg_layer L, const uint32_t* pats, const size_t* ks, size_t P,
                        double psi, pg_stream s) {
    PG_API_BEGIN
    require(out && L, PG_INVALID_ARGUMENT, "aggregate_layout: bad arguments");
    if (P == 0) throw Error{PG_INVALID_ARGUMENT, "aggregate_layout: no patterns"};
    if (psi <= 0 || psi > 1) throw Error{PG_INVALID_ARGUMENT, "aggregate_layout: psi out of range"};
    const size_t r = L->r;
    std::vector<size_t> freq(r, 0);
    size_t off = 0;
    for (size_t p = 0; p < P; ++p) {
        for (size_t q = 0; q < ks[p]; ++q) {
            const uint32_t e = pats[off + q];
            if (e >= r) throw Error{PG_OUT_OF_RANGE, "pattern references expert >= r_store"};
            freq[e] += 1;
        }
        off += ks[p];
    }
    auto g = std::make_unique<pg_agg_s>();
    g->layer = L;
    g->m = L->m;
    g->n = L->n;
    g->P = (int)P;
    g->dt = L->dt;
    for (size_t e = 0; e < r; ++e)
        if (double(freq[e]) >= psi * double(P)) g->shared_ids.push_back((uint32_t)e);
    const size_t sc = g->shared_ids.size();
    g->s_pad = (int)round_up(sc, kSlotAlign);
    g->res_ids.resize(P);
    g->use_shared.resize(P);
    g->ref_offset.resize(P);
    g->dev_off.resize(P);
    g->cnt_pad.resize(P);
    size_t arena_ref = sc;
    int arena_dev = g->s_pad;
    off = 0;
    for (size_t p = 0; p < P; ++p) {
        g->use_shared[p].assign(sc, 0);
        for (size_t q = 0; q < ks[p]; ++q) {
            const uint32_t e = pats[off + q];
            auto it = std::lower_bound(g->shared_ids.begin(), g->shared_ids.end(), e);
            if (it != g->shared_ids.end() && *it == e) g->use_shared[p][it - g->shared_ids.begin()] = 1;
            else g->res_ids[p].push_back(e);
        }
        g->ref_offset[p] = arena_ref;
        arena_ref += g->res_ids[p].size();
        g->dev_off[p] = arena_dev;
        g->cnt_pad[p] = (int)round_up(g->res_ids[p].size(), kSlotAlign);
        arena_dev += g->cnt_pad[p];
        off += ks[p];
    }
    g->arena_cols = arena_dev;
    // gather list over the device arena (-1 = zero padding)
    std::vector<int32_t> idx(arena_dev, -1);
    for (size_t j = 0; j < sc; ++j) idx[j] = (int32_t)g->shared_ids[j];
    for (size_t p = 0; p < P; ++p)
        for (size_t j = 0; j < g->res_ids[p].size(); ++j) idx[g->dev_off[p] + j] = (int32_t)g->res_ids[p][j];
    std::vector<uint8_t> masks((size_t)P * g->s_pad, 0);
    std::vector<int32_t> table(2 * P);
    g->mask_full.assign(P, 1);
    for (size_t p = 0; p < P; ++p) {
        for (size_t j = 0; j < sc; ++j) {
            masks[p * g->s_pad + j] = g->use_shared[p][j];
            if (!g->use_shared[p][j]) g->mask_full[p] = 0;
        }
        table[2 * p] = g->dev_off[p];
        table[2 * p + 1] = g->cnt_pad[p];
    }
    const size_t es = dtype_size(L->dt);
    g->ldb = L->ldb;
    g->lda = arena_dev;  // multiple of 32 elements -> 16-byte aligned rows
    g->bt_arena = dev_alloc((size_t)arena_dev * g->ldb * es);
    g->a_arena = dev_alloc((size_t)g->m * g->lda * es);
    g->masks = static_cast<uint8_t*>(dev_alloc(masks.size()));
    g->table = static_cast<int32_t*>(dev_alloc(table.size() * 4));
    g->bytes = (size_t)arena_dev * (g->ldb + g->m) * es;
    const cudaStream_t st = as_stream(s);
    PG_CUDA_THROW(cudaMemcpy(g->masks, masks.data(), masks.size(), cudaMemcpyHostToDevice));
    PG_CUDA_THROW(cudaMemcpy(g->table, table.data(), table.size() * 4, cudaMemcpyHostToDevice));
    Scratch di(idx.size() * 4, st);
    PG_CUDA_THROW(cudaMemcpyAsync(di.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, st));
    launch_gather_rows(L->dt, L->bt, L->ldb, di.as<int32_t>(), arena_dev, arena_dev, L->n, g->bt_arena,
                       g->ldb, st);
    launch_gather_cols(L->dt, L->a, L->lda, di.as<int32_t>(), arena_dev, arena_dev, L->m, g->a_arena,
                       g->lda, st);
    PG_CUDA_THROW(cudaStreamSynchronize(st));  // idx is host-owned until the copy lands
    *out = g.release();
    PG_API_END
}

int pg_agg_destroy(pg_agg g) {
    PG_API_BEGIN
    if (!g) return PG_OK;
    cudaFree(g->bt_arena); cudaFree(g->a_arena); cudaFree(g->masks); cudaFree(g->table);
    delete g;
    PG_API_END
}

int pg_agg_patterns(pg_agg g, size_t* n) {
    PG_API_BEGIN
    require(g && n, PG_INVALID_ARGUMENT, "agg: bad arguments");
    *n = g->P;
    PG_API_END
}

int pg_agg_shared(pg_agg g, size_t* count, uint32_t* ids) {
    PG_API_BEGIN
    require(g && count, PG_INVALID_ARGUMENT, "agg: bad arguments");
    *count = g->shared_ids.size();
    if (ids) std::copy(g->shared_ids.begin(), g->shared_ids.end(), ids);
    PG_API_END
}

int pg_agg_residual(pg_agg g, size_t p, size_t* count, uint32_t* ids, size_t* arena_offset,
                    uint8_t* use_shared) {
    PG_API_BEGIN
    require(g, PG_INVALID_ARGUMENT, "agg: bad arguments");
    if (p >= (size_t)g->P) throw Error{PG_OUT_OF_RANGE, "unknown pattern"};
    if (count) *count = g->res_ids[p].size();
    if (ids) std::copy(g->res_ids[p].begin(), g->res_ids[p].end(), ids);
    if (arena_offset) *arena_offset = g->ref_offset[p];
    if (use_shared) std::copy(g->use_shared[p].begin(), g->use_shared[p].end(), use_shared);
    PG_API_END
}

int pg_agg_trace(pg_agg g, size_t p, size_t* count, size_t* cols) {
    PG_API_BEGIN
    require(g && count, PG_INVALID_ARGUMENT, "agg: bad arguments");
    if (p >= (size_t)g->P) throw Error{PG_OUT_OF_RANGE, "unknown pattern"};
    // one coalesced shared-block read [0, s) plus the pattern's residual block
    // (exec_engine.hpp:201-213), reported in the reference's arena numbering
    const size_t sc = g->shared_ids.size(), rc = g->res_ids[p].size();
    *count = sc + rc;
    if (cols) {
        for (size_t j = 0; j < sc; ++j) cols[j] = j;
        for (size_t j = 0; j < rc; ++j) cols[sc + j] = g->ref_offset[p] + j;
    }
    PG_API_END
}

int pg_agg_bytes(pg_agg g, size_t* bytes) {
    PG_API_BEGIN
    require(g && bytes, PG_INVALID_ARGUMENT, "agg: bad arguments");
    *bytes = g->bytes;
    PG_API_END
}

static SlotMap agg_slotmap(pg_agg g, int p) {
    SlotMap sm;
    sm.run0_len = g->s_pad;
    sm.run1_start = g->dev_off[p];
    sm.run1_len = g->cnt_pad[p];
    // padding slots are zero rows / columns, so a pattern that uses every
    // shared expert needs no activity mask
    sm.mask = g->mask_full[p] ? nullptr : g->masks + (size_t)p * g->s_pad;
    return sm;
}

int pg_aggregated_forward(pg_agg g, size_t p, const int32_t* pdev, const void* x, pg_layout lay,
                          size_t T, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(g && x && y, PG_INVALID_ARGUMENT, "aggregated_forward: bad X shape");
    check_ydt(g->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const int fm = lay == PG_FEATURE_MAJOR && T > 1;
    int maxcnt = 0;
    for (int c : g->cnt_pad) maxcnt = std::max(maxcnt, c);
    if (pdev) {
        if (decode_tmax((int)T) && decode_smem_need(g->dt, g->n, g->s_pad + maxcnt, (int)T) <= 200 * 1024) {
            SlotMap sm;
            sm.run0_len = g->s_pad;
            sm.dyn_pattern = pdev;
            sm.dyn_table = g->table;
            sm.dyn_masks = g->masks;
            sm.dyn_mask_stride = g->s_pad;
            run_forward(g->dt, g->bt_arena, g->ldb, g->a_arena, g->lda, sm, g->s_pad + maxcnt, g->n,
                        g->m, x, fm, (int)T, y, ydt, st);
            return PG_OK;
        }
        int32_t hp = 0;
        PG_CUDA_THROW(cudaMemcpyAsync(&hp, pdev, 4, cudaMemcpyDeviceToHost, st));
        PG_CUDA_THROW(cudaStreamSynchronize(st));
        p = (size_t)hp;
    }
    if (p >= (size_t)g->P) throw Error{PG_OUT_OF_RANGE, "unknown pattern"};
    SlotMap sm = agg_slotmap(g, (int)p);
    run_forward(g->dt, g->bt_arena, g->ldb, g->a_arena, g->lda, sm, sm.nslots(), g->n, g->m, x, fm,
                (int)T, y, ydt, st);
    PG_API_END
}

int pg_aggregated_forward_batched(pg_agg g, const int32_t* pats, const int64_t* offs, size_t P,
                                  const void* x, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(g && pats && offs && x && y, PG_INVALID_ARGUMENT, "aggregated_forward: bad X shape");
    check_ydt(g->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const size_t es = dtype_size(g->dt), ys = dtype_size(ydt);
    std::vector<PrefillJob> jobs;  // bf16 prompts with T > 8: one grouped tensor-core launch per stage
    for (size_t q = 0; q < P; ++q) {
        const int p = pats[q];
        if (p < 0 || p >= g->P) throw Error{PG_OUT_OF_RANGE, "unknown pattern"};
        const int64_t t0 = offs[q], t1 = offs[q + 1];
        if (t1 <= t0) continue;
        SlotMap sm = agg_slotmap(g, p);
        const void* xq = static_cast<const char*>(x) + t0 * g->n * es;
        void* yq = static_cast<char*>(y) + t0 * g->m * ys;
        if (g->dt == PG_BF16 && prefill_ok(g->n, (int)(t1 - t0))) {
            jobs.push_back(PrefillJob{g->bt_arena, g->ldb, g->a_arena, g->lda, sm, g->n, g->m, xq, (int)(t1 - t0), yq, ydt});
            continue;
        }
        run_forward(g->dt, g->bt_arena, g->ldb, g->a_arena, g->lda, sm, sm.nslots(), g->n, g->m, xq, 0,
                    (int)(t1 - t0), yq, ydt, st);
    }
    if (!jobs.empty()) run_prefill(jobs, st);
    PG_API_END
}

int pg_silu_mul(const void* g, const void* u, pg_dtype in_dt, size_t count, void* act,
                pg_dtype act_dt, pg_stream s) {
    PG_API_BEGIN
    require(g && u && act, PG_INVALID_ARGUMENT, "silu_mul: null");
    require(in_dt == PG_F32 || in_dt == PG_F64, PG_INVALID_ARGUMENT, "silu_mul: inputs must be f32/f64");
    if (count) launch_silu_mul(g, u, in_dt, count, act, act_dt, as_stream(s));
    PG_API_END
}

static LinSpec agg_spec(pg_agg g, int p, const int32_t* pdev, void* y) {
    SlotMap sm;
    int cap;
    if (pdev) {
        sm.run0_len = g->s_pad;
        sm.dyn_pattern = pdev;
        sm.dyn_table = g->table;
        sm.dyn_masks = g->masks;
        sm.dyn_mask_stride = g->s_pad;
        int maxcnt = 0;
        for (int c : g->cnt_pad) maxcnt = std::max(maxcnt, c);
        cap = g->s_pad + maxcnt;
    } else {
        if (p < 0 || p >= g->P) throw Error{PG_OUT_OF_RANGE, "unknown pattern"};
        sm = agg_slotmap(g, p);
        cap = sm.nslots();
    }
    return LinSpec{g->bt_arena, g->ldb, g->a_arena, g->lda, sm, cap, g->n, g->m, y};
}

int pg_module_forward(const pg_agg* gs, size_t nlin, const size_t* patterns, const int32_t* pattern_dev,
                      const void* x, void* const* ys, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(gs && nlin >= 1 && nlin <= (size_t)kMaxLin && x && ys, PG_INVALID_ARGUMENT,
            "module_forward: 1..3 linears sharing one input");
    std::vector<LinSpec> ph;
    for (size_t l = 0; l < nlin; ++l) {
        require(gs[l] && gs[l]->dt == gs[0]->dt && gs[l]->n == gs[0]->n, PG_INVALID_ARGUMENT,
                "module_forward: linears must share dtype and input width");
        check_ydt(gs[l]->dt, ydt);
        ph.push_back(agg_spec(gs[l], pattern_dev ? 0 : (int)patterns[l], pattern_dev, ys[l]));
    }
    const cudaStream_t st = as_stream(s);
    if (chain_ok(gs[0]->dt, {ph}, false)) {
        run_chain(gs[0]->dt, {ph}, x, false, nullptr, ydt, st);
    } else {  // operands too wide for one launch: one chain per linear
        for (const LinSpec& L : ph) run_forward(gs[0]->dt, L.bt, L.ldb, L.a, L.lda, L.sm, L.cap, L.n, L.m, x, 0, 1,
                                                L.y, ydt, st);
    }
    PG_API_END
}

int pg_mlp_forward(pg_agg up, pg_agg gate, pg_agg down, const size_t* patterns, const int32_t* pattern_dev,
                   const void* x, void* act, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(up && gate && down && x && y, PG_INVALID_ARGUMENT, "mlp_forward: bad arguments");
    require(up->dt == gate->dt && up->dt == down->dt, PG_INVALID_ARGUMENT, "mlp_forward: mixed dtypes");
    require(up->m == gate->m && up->n == gate->n && down->n == up->m, PG_INVALID_ARGUMENT,
            "mlp_forward: shape mismatch (up/gate m x n, down n x m)");
    check_ydt(down->dt, ydt);
    const int p0 = pattern_dev ? 0 : (int)patterns[0], p1 = pattern_dev ? 0 : (int)patterns[1],
              p2 = pattern_dev ? 0 : (int)patterns[2];
    const cudaStream_t st = as_stream(s);
    const std::vector<std::vector<LinSpec>> ph = {
        {agg_spec(up, p0, pattern_dev, nullptr), agg_spec(gate, p1, pattern_dev, nullptr)},
        {agg_spec(down, p2, pattern_dev, y)}};
    if (chain_ok(up->dt, ph, true)) {
        run_chain(up->dt, ph, x, true, act, ydt, st);
    } else {  // too wide for one launch: up, gate, silu, down as separate chains
        const size_t accs = up->dt == PG_F64 ? 8 : 4, es = dtype_size(up->dt);
        const pg_dtype mid = up->dt == PG_F64 ? PG_F64 : PG_F32;
        Scratch ws(2 * round_up((size_t)up->m * accs, 256) + ((act == nullptr) ? (size_t)up->m * es : 0), st);
        char* u = ws.as<char>();
        char* g = u + round_up((size_t)up->m * accs, 256);
        void* a = act ? act : (void*)(g + round_up((size_t)up->m * accs, 256));
        for (int l = 0; l < 2; ++l) {
            const LinSpec& L = ph[0][l];
            run_forward(up->dt, L.bt, L.ldb, L.a, L.lda, L.sm, L.cap, L.n, L.m, x, 0, 1, l ? g : u, mid, st);
        }
        launch_silu_mul(g, u, mid, (size_t)up->m, a, up->dt, st);
        const LinSpec& D = ph[1][0];
        run_forward(up->dt, D.bt, D.ldb, D.a, D.lda, D.sm, D.cap, D.n, D.m, a, 0, 1, y, ydt, st);
    }
    PG_API_END
}

// A chain of S MLP blocks (x_{s+1} = y_s) through the decode chain, up to 8
// blocks per launch: the weight producer streams block s+1's rows through
// block s's last exchanges and the launch boundary disappears.
int pg_mlp_forward_chain(const pg_agg* ups, const pg_agg* gates, const pg_agg* downs, const size_t* patterns,
                         size_t S, const void* x, void* const* acts, void* const* ys, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(ups && gates && downs && patterns && x && ys && S >= 1, PG_INVALID_ARGUMENT,
            "mlp_forward_chain: bad arguments");
    const pg_dtype wdt = ups[0]->dt;
    for (size_t b = 0; b < S; ++b) {
        const pg_agg up = ups[b], gate = gates[b], down = downs[b];
        require(up && gate && down && ys[b], PG_INVALID_ARGUMENT, "mlp_forward_chain: bad arguments");
        require(up->dt == wdt && gate->dt == wdt && down->dt == wdt, PG_INVALID_ARGUMENT, "mlp_forward_chain: mixed dtypes");
        require(up->m == gate->m && up->n == gate->n && down->n == up->m && down->m == up->n, PG_INVALID_ARGUMENT,
                "mlp_forward_chain: shape mismatch (up/gate m x n, down n x m, blocks chained)");
    }
    check_ydt(wdt, ydt);
    require(S == 1 || ydt == wdt, PG_INVALID_ARGUMENT, "mlp_forward_chain: chained blocks need y in the weight dtype");
    const cudaStream_t st = as_stream(s);
    for (size_t b0 = 0; b0 < S; b0 += kMaxPhase / 2) {
        const size_t nb = std::min<size_t>(kMaxPhase / 2, S - b0);
        std::vector<std::vector<LinSpec>> ph;
        ChainIO io;
        for (size_t b = b0; b < b0 + nb; ++b) {
            const size_t* pt = patterns + 3 * b;
            ph.push_back({agg_spec(ups[b], (int)pt[0], nullptr, nullptr), agg_spec(gates[b], (int)pt[1], nullptr, nullptr)});
            ph.push_back({agg_spec(downs[b], (int)pt[2], nullptr, ys[b])});
            io.x.push_back(b == 0 ? x : ys[b - 1]);
            io.x.push_back(nullptr);
            void* a = acts ? acts[b] : nullptr;
            io.act.push_back(a);
            io.act.push_back(a);
            io.epi.push_back(1);
            io.epi.push_back(0);
        }
        require(chain_ok(wdt, ph, true), PG_INVALID_ARGUMENT, "mlp_forward_chain: block too wide for the decode chain");
        run_chain_io(wdt, ph, io, true, ydt, st, nullptr);
    }
    PG_API_END
}

// ------------------------------------------------------------ expert-sharded peer reduction
int pg_peer_buffer_bytes(size_t m, size_t npeer, size_t* bytes) {
    PG_API_BEGIN
    require(bytes && npeer >= 1 && npeer <= (size_t)kMaxPeers && m > 0, PG_INVALID_ARGUMENT,
            "peer_buffer_bytes: 1..8 ranks");
    *bytes = 2 * npeer * m * 8;
    PG_API_END
}

int pg_agg_forward_peer(pg_agg g, size_t pattern, const void* x, void* y, pg_dtype ydt, int rank, int npeer,
                        void* const* peer_bufs, int grid, pg_stream s) {
    PG_API_BEGIN
    require(g && x && y && peer_bufs && npeer >= 1 && npeer <= kMaxPeers && rank >= 0 && rank < npeer,
            PG_INVALID_ARGUMENT, "forward_peer: bad arguments");
    require(g->dt != PG_F64 && ydt != PG_F64, PG_INVALID_ARGUMENT, "forward_peer: bf16/f32 layouts");
    for (int r = 0; r < npeer; ++r) require(peer_bufs[r] != nullptr, PG_INVALID_ARGUMENT, "forward_peer: null buffer");
    check_ydt(g->dt, ydt);
    const std::vector<std::vector<LinSpec>> ph = {{agg_spec(g, (int)pattern, nullptr, y)}};
    require(chain_ok(g->dt, ph, false), PG_INVALID_ARGUMENT, "forward_peer: layer too wide for the decode chain");
    PeerSpec ps;
    ps.rank = rank;
    ps.npeer = npeer;
    ps.grid = grid;
    ps.bufs = peer_bufs;
    run_chain(g->dt, ph, x, false, nullptr, ydt, as_stream(s), &ps);
    PG_API_END
}

int pg_mlp_forward_peer(pg_agg up, pg_agg gate, pg_agg down, const size_t* patterns, const void* x, void* act,
                        void* y, pg_dtype ydt, int rank, int npeer, void* const* peer_bufs, int grid, pg_stream s) {
    PG_API_BEGIN
    require(up && gate && down && patterns && x && y && peer_bufs && npeer >= 1 && npeer <= kMaxPeers && rank >= 0 &&
                rank < npeer,
            PG_INVALID_ARGUMENT, "mlp_forward_peer: bad arguments");
    require(up->dt == gate->dt && up->dt == down->dt, PG_INVALID_ARGUMENT, "mlp_forward_peer: mixed dtypes");
    require(up->dt != PG_F64 && ydt != PG_F64, PG_INVALID_ARGUMENT, "mlp_forward_peer: bf16/f32 layouts");
    require(up->m == gate->m && up->n == gate->n && down->n == up->m, PG_INVALID_ARGUMENT,
            "mlp_forward_peer: shape mismatch (up/gate m x n, down n x m)");
    for (int r = 0; r < npeer; ++r) require(peer_bufs[r] != nullptr, PG_INVALID_ARGUMENT, "mlp_forward_peer: null buffer");
    check_ydt(down->dt, ydt);
    const std::vector<std::vector<LinSpec>> ph = {
        {agg_spec(up, (int)patterns[0], nullptr, nullptr), agg_spec(gate, (int)patterns[1], nullptr, nullptr)},
        {agg_spec(down, (int)patterns[2], nullptr, y)}};
    require(chain_ok(up->dt, ph, true), PG_INVALID_ARGUMENT, "mlp_forward_peer: block too wide for the decode chain");
    PeerSpec ps;
    ps.rank = rank;
    ps.npeer = npeer;
    ps.grid = grid;
    ps.bufs = peer_bufs;
    run_chain(up->dt, ph, x, true, act, ydt, as_stream(s), &ps);
    PG_API_END
}

int pg_ipc_get_handle(const void* dev_ptr, void* handle_out) {
    PG_API_BEGIN
    require(dev_ptr && handle_out, PG_INVALID_ARGUMENT, "ipc: bad arguments");
    cudaIpcMemHandle_t h;
    PG_CUDA_THROW(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    PG_API_END
}

int pg_ipc_open_handle(const void* handle, void** dev_ptr) {
    PG_API_BEGIN
    require(handle && dev_ptr, PG_INVALID_ARGUMENT, "ipc: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    PG_CUDA_THROW(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    PG_API_END
}

int pg_ipc_close(void* dev_ptr) {
    PG_API_BEGIN
    require(dev_ptr, PG_INVALID_ARGUMENT, "ipc: null");
    PG_CUDA_THROW(cudaIpcCloseMemHandle(dev_ptr));
    PG_API_END
}

int pg_copy_io(const void* src, void* dst, size_t bytes, pg_stream s) {
    PG_API_BEGIN
    require(src && dst, PG_INVALID_ARGUMENT, "copy_io: null buffer");
    launch_copy_io(src, dst, bytes, as_stream(s));
    PG_API_END
}

int pg_chain_workspace_release(pg_stream s) {
    PG_API_BEGIN
    cudaStream_t st = as_stream(s);
    int dev = 0;
    PG_CUDA_THROW(cudaGetDevice(&dev));
    PG_CUDA_THROW(cudaStreamSynchronize(st));
    union_wm_release(st);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
        if (std::get<0>(it->first) == dev && std::get<1>(it->first) == st) {
            if (it->second.first) PG_CUDA_THROW(cudaFree(it->second.first));
            it = g_ws.erase(it);
        } else {
            ++it;
        }
    }
    PG_API_END
}

int pg_chain_debug_dump(uint64_t* out_host, size_t n) {
    PG_API_BEGIN
    if (getenv("PG_WM_DBG") && out_host) {  // union batch kernel stamps instead (diagnostics only)
        union_wm_debug_dump(reinterpret_cast<unsigned long long*>(out_host), n);
        return PG_OK;
    }
    require(out_host && g_chain_dbg, PG_INVALID_ARGUMENT, "chain debug: set PG_CHAIN_DBG=1");
    PG_CUDA_THROW(cudaMemcpy(out_host, g_chain_dbg, std::min<size_t>(n, 1024 * 16) * 8, cudaMemcpyDeviceToHost));
    PG_API_END
}

int pg_fill_normal_device(void* out, pg_dtype dt, size_t count, uint64_t seed, double scale,
                          pg_stream s) {
    PG_API_BEGIN
    require(out, PG_INVALID_ARGUMENT, "fill: null");
    launch_fill_normal(out, dt, count, seed, scale, as_stream(s));
    PG_API_END
}

}  // extern "C"

extern "C" int pg_gemm_bf16(const void* a, int64_t lda, const void* b, int64_t ldb, void* out, int64_t ldo, size_t M,
                            size_t N, size_t K, int out_bf16, pg_stream s) {
    PG_API_BEGIN
    require(a && b && out, PG_INVALID_ARGUMENT, "gemm: null operand");
    require(K % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0, PG_INVALID_ARGUMENT, "gemm: rows must be 16-byte aligned");
    launch_umma({UmmaSpec{a, lda, b, ldb, out, ldo, (int)M, (int)N, (int)K, out_bf16}}, as_stream(s));
    PG_API_END
}

// ------------------------------------------------------------ routed prefill (device pack)
extern "C" int pg_pack_bytes(pg_layer L, size_t k, size_t n_prompts, size_t* bt_bytes, size_t* a_bytes) {
    PG_API_BEGIN
    require(L && bt_bytes && a_bytes && k >= 1 && k <= (size_t)L->r, PG_INVALID_ARGUMENT, "pack_bytes: bad arguments");
    const size_t kp = round_up(k, 8), es = dtype_size(L->dt);
    *bt_bytes = n_prompts * kp * (size_t)L->ldb * es;
    *a_bytes = n_prompts * (size_t)L->m * kp * es;
    PG_API_END
}

extern "C" int pg_pack_selected(pg_layer L, const int32_t* sel_dev, size_t k, size_t P, void* bt_out, void* a_out,
                                pg_stream s) {
    PG_API_BEGIN
    require(L && sel_dev && a_out && P > 0, PG_INVALID_ARGUMENT, "pack_selected: bad arguments");
    require(L->dt == PG_BF16, PG_INVALID_ARGUMENT, "pack_selected: bf16 layers (tensor-core prefill path)");
    if (k == 0 || k > (size_t)L->r) throw Error{PG_INVALID_ARGUMENT, "select_topk: K out of range"};
    launch_pack_selected(L->bt, L->ldb, L->a, L->lda, L->r, L->n, L->m, sel_dev, (int)k, (int)P, bt_out, a_out,
                         as_stream(s));
    PG_API_END
}

extern "C" int pg_prefill_packed(pg_layer L, const void* bt_packed, const void* a_packed, size_t k,
                                 const int64_t* offs, size_t P, const void* x, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(L && bt_packed && a_packed && offs && x && y && P > 0, PG_INVALID_ARGUMENT,
            "prefill_packed: bad arguments");
    require(L->dt == PG_BF16 && L->n % 8 == 0, PG_INVALID_ARGUMENT, "prefill_packed: bf16 layers, n % 8 == 0");
    if (k == 0 || k > (size_t)L->r) throw Error{PG_INVALID_ARGUMENT, "select_topk: K out of range"};
    check_ydt(L->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const int kp = (int)round_up(k, 8);
    const size_t ys = dtype_size(ydt);
    size_t zbytes = 0;
    for (size_t p = 0; p < P; ++p) zbytes += round_up((size_t)(offs[p + 1] - offs[p]) * kp * 2, 256);
    Scratch z(zbytes, st);
    std::vector<UmmaSpec> s1, s2;
    size_t zo = 0;
    for (size_t p = 0; p < P; ++p) {
        const int64_t t0 = offs[p], T = offs[p + 1] - offs[p];
        if (T <= 0) continue;
        const void* bt = static_cast<const char*>(bt_packed) + p * (size_t)kp * L->ldb * 2;
        const void* a = static_cast<const char*>(a_packed) + p * (size_t)L->m * kp * 2;
        const void* xq = static_cast<const char*>(x) + t0 * L->n * 2;
        void* yq = static_cast<char*>(y) + t0 * L->m * ys;
        if (!prefill_ok(L->n, (int)T)) {  // a few tokens: the gather GEMV path over the packed arena
            SlotMap sm;
            sm.run0_len = kp;
            sm.cap = kp;
            run_forward(PG_BF16, bt, L->ldb, a, kp, sm, kp, L->n, L->m, xq, 0, (int)T, yq, ydt, st);
            continue;
        }
        void* zq = z.as<char>() + zo;
        zo += round_up((size_t)T * kp * 2, 256);
        s1.push_back(UmmaSpec{xq, L->n, bt, L->ldb, zq, kp, (int)T, kp, L->n, 1});
        s2.push_back(UmmaSpec{zq, kp, a, kp, yq, L->m, (int)T, L->m, kp, ydt == PG_BF16 ? 1 : 0});
    }
    if (!s1.empty()) {
        launch_umma(s1, st);
        launch_umma(s2, st);
    }
    PG_API_END
}

extern "C" int pg_prefill_gathered(pg_layer L, const int32_t* sel_dev, const void* a_packed, size_t k,
                                   const int64_t* offs, size_t P, const void* x, void* y, pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(L && sel_dev && a_packed && offs && x && y && P > 0, PG_INVALID_ARGUMENT,
            "prefill_gathered: bad arguments");
    require(L->dt == PG_BF16 && L->n % 8 == 0, PG_INVALID_ARGUMENT, "prefill_gathered: bf16 layers, n % 8 == 0");
    if (k == 0 || k > (size_t)L->r) throw Error{PG_INVALID_ARGUMENT, "select_topk: K out of range"};
    check_ydt(L->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const int kp = (int)round_up(k, 8);
    const size_t ys = dtype_size(ydt);
    size_t zbytes = 0;
    for (size_t p = 0; p < P; ++p) {
        const int64_t T = offs[p + 1] - offs[p];
        require(T == 0 || T >= 256, PG_INVALID_ARGUMENT,
                "prefill_gathered: every prompt needs 0 or >= 256 tokens (CTA-pair tiles); pack B^T for shorter ones");
        zbytes += round_up((size_t)T * kp * 2, 256);
    }
    Scratch z(zbytes, st);
    std::vector<UmmaSpec> s1, s2;
    size_t zo = 0;
    for (size_t p = 0; p < P; ++p) {
        const int64_t t0 = offs[p], T = offs[p + 1] - offs[p];
        if (T <= 0) continue;
        const void* a = static_cast<const char*>(a_packed) + p * (size_t)L->m * kp * 2;
        const void* xq = static_cast<const char*>(x) + t0 * L->n * 2;
        void* yq = static_cast<char*>(y) + t0 * L->m * ys;
        void* zq = z.as<char>() + zo;
        zo += round_up((size_t)T * kp * 2, 256);
        // stage 1: Z = X . B^T[sel]^T, the selected rows gathered by the GEMM's TMA
        // (columns j >= k read zero rows -> zero Z padding for stage 2)
        UmmaSpec a1{xq, L->n, L->bt, L->ldb, zq, kp, (int)T, kp, L->n, 1};
        a1.b_idx = sel_dev + p * k;
        a1.b_idx_n = (int)k;
        a1.b_idx_rows = L->r;
        s1.push_back(a1);
        s2.push_back(UmmaSpec{zq, kp, a, kp, yq, L->m, (int)T, L->m, kp, ydt == PG_BF16 ? 1 : 0});
    }
    if (!s1.empty()) {
        launch_umma(s1, st);
        launch_umma(s2, st);
    }
    PG_API_END
}

extern "C" int pg_prefill_batched(const pg_agg* aggs, const int64_t* offs, size_t P, const void* x, void* y,
                                  pg_dtype ydt, pg_stream s) {
    PG_API_BEGIN
    require(aggs && offs && x && y && P > 0, PG_INVALID_ARGUMENT, "prefill_batched: bad arguments");
    const pg_agg g0 = aggs[0];
    require(g0 && g0->dt == PG_BF16, PG_INVALID_ARGUMENT, "prefill_batched: bf16 layouts only");
    check_ydt(g0->dt, ydt);
    const cudaStream_t st = as_stream(s);
    const size_t ys = dtype_size(ydt);
    std::vector<PrefillJob> jobs;
    for (size_t q = 0; q < P; ++q) {
        const pg_agg g = aggs[q];
        require(g && g->dt == PG_BF16 && g->n == g0->n && g->m == g0->m, PG_INVALID_ARGUMENT,
                "prefill_batched: layouts must share shape and dtype");
        const int64_t t0 = offs[q], t1 = offs[q + 1];
        if (t1 <= t0) continue;
        const void* xq = static_cast<const char*>(x) + t0 * g->n * 2;
        void* yq = static_cast<char*>(y) + t0 * g->m * ys;
        SlotMap sm = agg_slotmap(g, 0);
        if (prefill_ok(g->n, (int)(t1 - t0)))
            jobs.push_back(PrefillJob{g->bt_arena, g->ldb, g->a_arena, g->lda, sm, g->n, g->m, xq, (int)(t1 - t0), yq, ydt});
        else
            run_forward(g->dt, g->bt_arena, g->ldb, g->a_arena, g->lda, sm, sm.nslots(), g->n, g->m, xq, 0,
                        (int)(t1 - t0), yq, ydt, st);
    }
    if (!jobs.empty()) run_prefill(jobs, st);
    PG_API_END
}
