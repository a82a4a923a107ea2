// parse_gpu.hpp -- C++ drop-in mirror of the reference hot-path API on B200.
//
// Include AFTER the reference headers are on the include path
// (-I<reference>/proj/include); link libparse_gpu.so.  Every function keeps the
// reference's name, argument types and exception behaviour, in namespace
// parse::gpu, so a caller swaps `parse::masked_forward` for
// `parse::gpu::masked_forward` (or a provider for parse::gpu::GpuProvider):
//
//   reference (proj/include/parse/...)           here
//   router.hpp:80  mean_pool(const Matd&)         gpu::mean_pool          bit-exact
//   router.hpp:41  score(RouterParams, h)         gpu::score              bit-exact
//   router.hpp:49  select_topk(logits, K)         gpu::select_topk        bit-exact
//   model.hpp:102  select_topk(score(mean_pool))  gpu::route              bit-exact (fused)
//   pattern_cache.hpp:38  cosine                  gpu::cosine             bit-exact
//   pattern_cache.hpp:104 retrieve(const PatternCache&, emb)  gpu::retrieve / gpu::DeviceCache::retrieve
//   pattern_cache.hpp:120 cache_insert(PatternCache&, entry)  gpu::cache_insert / gpu::DeviceCache::insert
//   pattern_cache.hpp:50  embed_prompt(core, prov, tokens)    gpu::embed_prompt (pooling on device, bit-exact)
//   rank_experts.hpp:52   masked_forward          gpu::masked_forward     f64: <= 1e-10 rel
//   exec_engine.hpp:112   aggregate_layout<T>     gpu::aggregate_layout<T>  (same shared/residual split)
//   exec_engine.hpp:193   aggregated_forward<T>   gpu::aggregated_forward<T>
//   exec_engine.hpp:239   scattered_forward<T>    gpu::scattered_forward<T>
//   exec_engine.hpp:275   ExecEngine<T>::build/forward/storage_overhead  gpu::ExecEngine<T>
//   exec_engine.hpp:322   ExecProvider            gpu::ExecProvider
//   toy_lm.hpp:68  ProjectionProvider             gpu::GpuProvider (RoutingProvider semantics;
//                                                 f64 / f32 / bf16 resident storage)
//   pattern_cache.hpp:67  route_prompt            gpu::route_prompt (GpuProvider prefill)
//   retrieve-or-route serving composition         gpu::select_for_prompt (hit: cached S; miss: route + insert)
//   (also: gpu::DeviceAggregatedLayer, the round-1 f64 layout wrapper)
//
// Host-memory convenience: each call copies its operands to the device and the
// result back (synchronous).  Serving code keeps handles resident and uses the
// C-ABI (parse_gpu.h) with device pointers and streams directly.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "parse/exec_engine.hpp"
#include "parse/model.hpp"
#include "parse/pattern_cache.hpp"
#include "parse/rank_experts.hpp"
#include "parse/router.hpp"
#include "parse_gpu.h"

namespace parse {
namespace gpu {

inline void check(int code) {
    if (code == PG_OK) return;
    const std::string msg = pg_last_error();
    switch (code) {
        case PG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case PG_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

// RAII device buffer
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t count) : n(count) { cuda(cudaMalloc(&p, (count ? count : 1) * sizeof(T))); }
    DevBuf(const T* host, size_t count) : DevBuf(count) {
        if (count) cuda(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
    }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    std::vector<T> host() const {
        std::vector<T> h(n);
        if (n) cuda(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
        return h;
    }
};

// ---------------------------------------------------------------- router
inline std::vector<double> mean_pool(const Matd& x) {
    DevBuf<double> xd(x.data(), x.rows() * x.cols()), h(x.rows());
    const int64_t offs[2] = {0, (int64_t)x.cols()};
    check(pg_mean_pool(xd.p, PG_F64, PG_FEATURE_MAJOR, x.rows(), offs, 1, h.p, nullptr));
    return h.host();
}

struct DeviceRouter {
    pg_router h = nullptr;
    size_t r = 0, n = 0;
    explicit DeviceRouter(const RouterParams& p) : r(p.theta.rows()), n(p.theta.cols()) {
        check(pg_router_create(&h, r, n, p.theta.data(), p.bias.data()));
    }
    ~DeviceRouter() { pg_router_destroy(h); }
    DeviceRouter(const DeviceRouter&) = delete;
    DeviceRouter& operator=(const DeviceRouter&) = delete;
};

inline std::vector<double> score(const RouterParams& r, const std::vector<double>& h) {
    if (h.size() != r.theta.cols()) throw std::invalid_argument("score: bad input length");
    DeviceRouter dr(r);
    DevBuf<double> hd(h.data(), h.size()), z(r.theta.rows());
    check(pg_score(dr.h, hd.p, 1, z.p, /*exact=*/1, nullptr));
    return z.host();
}

inline RankSelection select_topk(const std::vector<double>& logits, std::size_t k) {
    DevBuf<double> zd(logits.data(), logits.size());
    DevBuf<uint32_t> sel(k ? k : 1);
    check(pg_select_topk(zd.p, logits.size(), 1, k, sel.p, nullptr));
    RankSelection s;
    s.indices = sel.host();
    s.indices.resize(k);
    return s;
}

// select_topk(score(r, mean_pool(x)), k) -- RoutingProvider's routing step
inline RankSelection route(const DeviceRouter& r, const Matd& x, std::size_t k) {
    DevBuf<double> xd(x.data(), x.rows() * x.cols());
    DevBuf<uint32_t> sel(k ? k : 1);
    const int64_t offs[2] = {0, (int64_t)x.cols()};
    check(pg_route_select(r.h, xd.p, PG_F64, PG_FEATURE_MAJOR, offs, 1, k, sel.p, nullptr, nullptr));
    RankSelection s;
    s.indices = sel.host();
    s.indices.resize(k);
    return s;
}

// ---------------------------------------------------------------- cache
inline double cosine(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) throw std::invalid_argument("cosine: length mismatch");
    DevBuf<double> ad(a.data(), a.size()), bd(b.data(), b.size()), out(1);
    check(pg_cosine(ad.p, bd.p, a.size(), out.p, nullptr));
    return out.host()[0];
}

// Device mirror of a PatternCache's embeddings; patterns stay host-side and
// RetrieveResult::pattern points into the source cache (pattern_cache.hpp:96).
// Built from a const cache it serves retrieve only; from a mutable one it also
// runs the miss-path insertion on both copies.
class DeviceCache {
public:
    explicit DeviceCache(const PatternCache& cache) : cc_(&cache) { load(); }
    explicit DeviceCache(PatternCache& cache) : cc_(&cache), mc_(&cache) { load(); }
    ~DeviceCache() { pg_cache_destroy(h_); }
    DeviceCache(const DeviceCache&) = delete;
    DeviceCache& operator=(const DeviceCache&) = delete;

    RetrieveResult retrieve(const PromptEmbedding& emb) const {
        if (cc_->entries.empty()) throw std::runtime_error("empty cache");
        DevBuf<double> q(emb.vec.data(), emb.vec.size());
        pg_retrieve_result r{};
        check(pg_retrieve(h_, q.p, /*exact_similarity=*/1, &r, nullptr, nullptr, nullptr));
        RetrieveResult out;
        out.entry = r.entry;
        out.similarity = r.similarity;
        out.hit = r.hit != 0;
        out.pattern = &cc_->entries[r.entry].pattern;
        return out;
    }
    // cache_insert (pattern_cache.hpp:120-124): refused once at capacity
    bool insert(CacheEntry entry) {
        if (!mc_) throw std::logic_error("DeviceCache: built from a const PatternCache");
        int ins = 0;
        check(pg_cache_insert(h_, entry.embedding.vec.data(), 0, &ins, nullptr));
        if (ins) mc_->entries.push_back(std::move(entry));
        return ins != 0;
    }
    const PatternCache& cache() const { return *cc_; }

private:
    void load() {
        check(pg_cache_create(&h_, cc_->d_model, cc_->capacity, cc_->min_similarity));
        std::vector<double> emb;
        for (const auto& e : cc_->entries) emb.insert(emb.end(), e.embedding.vec.begin(), e.embedding.vec.end());
        check(pg_cache_load(h_, emb.data(), cc_->entries.size()));
    }
    const PatternCache* cc_ = nullptr;
    PatternCache* mc_ = nullptr;
    pg_cache h_ = nullptr;
};

// retrieve (pattern_cache.hpp:104-117), reference signature
inline RetrieveResult retrieve(const PatternCache& cache, const PromptEmbedding& emb) {
    if (cache.entries.empty()) throw std::runtime_error("empty cache");
    DeviceCache dc(cache);
    return dc.retrieve(emb);
}

// cache_insert (pattern_cache.hpp:120-124), reference signature: the capacity
// rule on the host list (the device copy, if any, is updated through
// DeviceCache::insert)
inline bool cache_insert(PatternCache& cache, CacheEntry entry) {
    if (cache.entries.size() >= cache.capacity) return false;
    cache.entries.push_back(std::move(entry));
    return true;
}
inline bool cache_insert(DeviceCache& cache, CacheEntry entry) { return cache.insert(std::move(entry)); }

// ---------------------------------------------------------------- layers
template <typename T> struct DType;
template <> struct DType<double> { static constexpr pg_dtype v = PG_F64; };
template <> struct DType<float> { static constexpr pg_dtype v = PG_F32; };

inline uint16_t f32_to_bf16(float f) {  // round to nearest even (NaN kept quiet)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// A FactorizedLayer resident on the device in f64, f32 or bf16 storage.
class DeviceLayer {
public:
    DeviceLayer(const FactorizedLayer& l, pg_dtype storage = PG_F64) : m_(l.m), n_(l.n), dt_(storage) {
        check(pg_layer_create(&h_, l.m, l.n, l.r_store, l.K, l.A.data(), l.B.data(), storage));
    }
    ~DeviceLayer() { pg_layer_destroy(h_); }
    DeviceLayer(const DeviceLayer&) = delete;
    DeviceLayer& operator=(const DeviceLayer&) = delete;
    pg_layer handle() const { return h_; }
    size_t m() const { return m_; }
    size_t n() const { return n_; }
    pg_dtype dtype() const { return dt_; }

    // masked_forward (rank_experts.hpp:52-72) in the storage dtype's arithmetic
    // (f64 -> f64; f32 -> f32; bf16 storage -> f32 accumulation), y as double
    Matd forward(const RankSelection& sel, const Matd& x) const {
        if (x.rows() != n_) throw std::invalid_argument("masked_forward: bad X shape");
        const size_t T = x.cols(), nx = x.rows() * T;
        Matd out(m_, T);
        if (dt_ == PG_F64) {
            DevBuf<double> xd(x.data(), nx), y(m_ * T);
            check(pg_masked_forward(h_, sel.indices.data(), sel.indices.size(), 0, xd.p, PG_FEATURE_MAJOR, T, y.p,
                                    PG_F64, nullptr));
            const std::vector<double> hy = y.host();
            std::copy(hy.begin(), hy.end(), out.data());
            return out;
        }
        std::vector<float> xf(nx);
        for (size_t i = 0; i < nx; ++i) xf[i] = float(x.data()[i]);
        DevBuf<float> y(m_ * T);
        if (dt_ == PG_F32) {
            DevBuf<float> xd(xf.data(), nx);
            check(pg_masked_forward(h_, sel.indices.data(), sel.indices.size(), 0, xd.p, PG_FEATURE_MAJOR, T, y.p,
                                    PG_F32, nullptr));
        } else {
            std::vector<uint16_t> xb(nx);
            for (size_t i = 0; i < nx; ++i) xb[i] = f32_to_bf16(xf[i]);
            DevBuf<uint16_t> xd(xb.data(), nx);
            check(pg_masked_forward(h_, sel.indices.data(), sel.indices.size(), 0, xd.p, PG_FEATURE_MAJOR, T, y.p,
                                    PG_F32, nullptr));
        }
        const std::vector<float> hy = y.host();
        for (size_t i = 0; i < hy.size(); ++i) out.data()[i] = hy[i];
        return out;
    }

    template <typename T>
    Mat<T> forward_t(const RankSelection& sel, const Mat<T>& x) const {
        if (DType<T>::v != dt_) throw std::invalid_argument("DeviceLayer: storage dtype differs from T");
        if (x.rows() != n_) throw std::invalid_argument("masked_forward: bad X shape");
        DevBuf<T> xd(x.data(), x.rows() * x.cols()), y(m_ * x.cols());
        check(pg_masked_forward(h_, sel.indices.data(), sel.indices.size(), 0, xd.p, PG_FEATURE_MAJOR, x.cols(), y.p,
                                DType<T>::v, nullptr));
        Mat<T> out(m_, x.cols());
        const std::vector<T> hy = y.host();
        std::copy(hy.begin(), hy.end(), out.data());
        return out;
    }

private:
    pg_layer h_ = nullptr;
    size_t m_, n_;
    pg_dtype dt_;
};

inline Matd masked_forward(const FactorizedLayer& layer, const RankSelection& sel, const Matd& x) {
    DeviceLayer dl(layer, PG_F64);
    return dl.forward(sel, x);
}

// aggregate_layout + aggregated_forward (exec_engine.hpp:112-236), f64 storage
// (round-1 wrapper, kept for existing callers; see AggregatedLayer<T> below)
class DeviceAggregatedLayer {
public:
    DeviceAggregatedLayer(const FactorizedLayer& layer, const std::vector<RankSelection>& patterns, double psi)
        : layer_(layer, PG_F64), m_(layer.m), n_(layer.n) {
        std::vector<uint32_t> flat;
        std::vector<size_t> ks;
        for (const auto& p : patterns) {
            flat.insert(flat.end(), p.indices.begin(), p.indices.end());
            ks.push_back(p.indices.size());
        }
        check(pg_aggregate_layout(&h_, layer_.handle(), flat.data(), ks.data(), patterns.size(), psi, nullptr));
    }
    ~DeviceAggregatedLayer() { pg_agg_destroy(h_); }
    DeviceAggregatedLayer(const DeviceAggregatedLayer&) = delete;
    DeviceAggregatedLayer& operator=(const DeviceAggregatedLayer&) = delete;

    std::vector<uint32_t> shared_ids() const {
        size_t c = 0;
        check(pg_agg_shared(h_, &c, nullptr));
        std::vector<uint32_t> v(c);
        check(pg_agg_shared(h_, &c, v.data()));
        return v;
    }
    Matd forward(std::size_t pattern_id, const Matd& x, AccessTrace* trace = nullptr) const {
        if (x.rows() != n_) throw std::invalid_argument("aggregated_forward: bad X shape");
        if (trace) {
            size_t c = 0;
            check(pg_agg_trace(h_, pattern_id, &c, nullptr));
            std::vector<size_t> cols(c);
            check(pg_agg_trace(h_, pattern_id, &c, cols.data()));
            trace->a_cols.insert(trace->a_cols.end(), cols.begin(), cols.end());
            trace->b_cols.insert(trace->b_cols.end(), cols.begin(), cols.end());
        }
        DevBuf<double> xd(x.data(), x.rows() * x.cols()), y(m_ * x.cols());
        check(pg_aggregated_forward(h_, pattern_id, nullptr, xd.p, PG_FEATURE_MAJOR, x.cols(), y.p, PG_F64, nullptr));
        Matd out(m_, x.cols());
        std::vector<double> hy = y.host();
        std::copy(hy.begin(), hy.end(), out.data());
        return out;
    }

private:
    DeviceLayer layer_;
    pg_agg h_ = nullptr;
    size_t m_, n_;
};

// ---- AggregatedLayer<T> (exec_engine.hpp:97-110) on the device: the same
// reference-numbered structure (shared ids, per-pattern residual ids,
// use_shared, arena_offset) as host metadata; the arena itself lives in HBM.
template <typename T>
struct AggregatedLayer {
    std::size_t m = 0, n = 0, r_store = 0;
    std::vector<std::uint32_t> shared_ids;
    struct Residual {
        std::vector<std::uint32_t> ids;
        std::vector<std::uint8_t> use_shared;
        std::size_t arena_offset = 0;
    };
    std::vector<Residual> residuals;
    double psi = 0.9;
    std::shared_ptr<DeviceLayer> layer;  // full factors, storage dtype of T
    std::shared_ptr<pg_agg_s> arena;     // packed [shared | residual_0 | ...] arena
};

template <typename T>
AggregatedLayer<T> aggregate_layout(const FactorizedLayer& layer, const std::vector<RankSelection>& patterns,
                                    double psi, std::shared_ptr<DeviceLayer> dev = nullptr) {
    AggregatedLayer<T> g;
    g.m = layer.m;
    g.n = layer.n;
    g.r_store = layer.r_store;
    g.psi = psi;
    g.layer = dev ? dev : std::make_shared<DeviceLayer>(layer, DType<T>::v);
    std::vector<uint32_t> flat;
    std::vector<size_t> ks;
    for (const auto& p : patterns) {
        flat.insert(flat.end(), p.indices.begin(), p.indices.end());
        ks.push_back(p.indices.size());
    }
    pg_agg h = nullptr;
    check(pg_aggregate_layout(&h, g.layer->handle(), flat.data(), ks.data(), patterns.size(), psi, nullptr));
    g.arena = std::shared_ptr<pg_agg_s>(h, [](pg_agg a) { pg_agg_destroy(a); });
    size_t c = 0;
    check(pg_agg_shared(h, &c, nullptr));
    g.shared_ids.resize(c);
    check(pg_agg_shared(h, &c, g.shared_ids.data()));
    g.residuals.resize(patterns.size());
    for (size_t p = 0; p < patterns.size(); ++p) {
        auto& R = g.residuals[p];
        size_t rc = 0, off = 0;
        check(pg_agg_residual(h, p, &rc, nullptr, nullptr, nullptr));
        R.ids.resize(rc);
        R.use_shared.resize(g.shared_ids.size());
        check(pg_agg_residual(h, p, &rc, R.ids.data(), &off, R.use_shared.data()));
        R.arena_offset = off;
    }
    return g;
}

template <typename T>
Mat<T> aggregated_forward(const AggregatedLayer<T>& g, std::size_t pattern_id, const Mat<T>& x,
                          AccessTrace* trace = nullptr) {
    if (pattern_id >= g.residuals.size()) throw std::out_of_range("unknown pattern");
    if (x.rows() != g.n) throw std::invalid_argument("aggregated_forward: bad X shape");
    if (trace) {
        size_t c = 0;
        check(pg_agg_trace(g.arena.get(), pattern_id, &c, nullptr));
        std::vector<size_t> cols(c);
        check(pg_agg_trace(g.arena.get(), pattern_id, &c, cols.data()));
        trace->a_cols.insert(trace->a_cols.end(), cols.begin(), cols.end());
        trace->b_cols.insert(trace->b_cols.end(), cols.begin(), cols.end());
    }
    DevBuf<T> xd(x.data(), x.rows() * x.cols()), y(g.m * x.cols());
    check(pg_aggregated_forward(g.arena.get(), pattern_id, nullptr, xd.p, PG_FEATURE_MAJOR, x.cols(), y.p,
                                DType<T>::v, nullptr));
    Mat<T> out(g.m, x.cols());
    const std::vector<T> hy = y.host();
    std::copy(hy.begin(), hy.end(), out.data());
    return out;
}

// scattered_forward (exec_engine.hpp:239-252): the selected columns of the full
// factors in S order (host matrices in, result out; uploads the factors)
template <typename T>
Mat<T> scattered_forward(const Mat<T>& a_full, const Mat<T>& b_full, const RankSelection& sel, const Mat<T>& x,
                         AccessTrace* trace = nullptr) {
    if (a_full.cols() != b_full.cols()) throw std::invalid_argument("scattered_forward: factor mismatch");
    FactorizedLayer fl;
    fl.m = a_full.rows();
    fl.n = b_full.rows();
    fl.r_store = a_full.cols();
    fl.K = sel.indices.size();
    fl.A = a_full.template cast<double>();
    fl.B = b_full.template cast<double>();
    DeviceLayer dl(fl, DType<T>::v);
    if (trace)
        for (std::uint32_t e : sel.indices) {
            trace->a_cols.push_back(e);
            trace->b_cols.push_back(e);
        }
    return dl.forward_t<T>(sel, x);
}

// ExecEngine<T> (exec_engine.hpp:275-319): per tensor the full factors and the
// aggregated layout, resident on the device; forward dispatches on the
// aggregated / scattered variants exactly like the reference.
template <typename T>
struct ExecEngine {
    struct Tensor {
        std::shared_ptr<DeviceLayer> full;
        AggregatedLayer<T> agg;
    };
    std::map<std::string, Tensor> tensors;
    std::vector<SelectionMap> patterns;
    double psi = 0.9;

    static ExecEngine build(const FactorizedModel& fm, std::vector<SelectionMap> pats, double psi_val) {
        ExecEngine eng;
        eng.psi = psi_val;
        eng.patterns = std::move(pats);
        for (const auto& [id, layer] : fm.layers) {
            Tensor t;
            t.full = std::make_shared<DeviceLayer>(layer, DType<T>::v);
            std::vector<RankSelection> sels;
            for (const auto& p : eng.patterns) sels.push_back(p.at(id));
            t.agg = aggregate_layout<T>(layer, sels, psi_val, t.full);
            eng.tensors[id] = std::move(t);
        }
        return eng;
    }

    Mat<T> forward(const std::string& id, std::size_t pattern_id, const Mat<T>& x, ExecVariant v,
                   AccessTrace* trace = nullptr) const {
        const Tensor& t = tensors.at(id);
        if (variant_aggregated(v)) return aggregated_forward(t.agg, pattern_id, x, trace);
        const RankSelection& sel = patterns.at(pattern_id).at(id);
        if (trace)
            for (std::uint32_t e : sel.indices) {
                trace->a_cols.push_back(e);
                trace->b_cols.push_back(e);
            }
        return t.full->template forward_t<T>(sel, x);
    }

    double storage_overhead() const {
        double dup = 0, base = 0;
        for (const auto& [id, t] : tensors) {
            base += double(t.agg.r_store) * double(t.agg.m + t.agg.n);
            for (const auto& r : t.agg.residuals) dup += double(r.ids.size()) * double(t.agg.m + t.agg.n);
        }
        return dup / base;
    }
};

// ExecProvider (exec_engine.hpp:322-348): plan-driven full-LM serving (f64)
class ExecProvider : public ProjectionProvider {
public:
    ExecProvider(const ExecEngine<double>& eng, std::size_t pattern_id, ExecVariant v)
        : eng_(eng), pattern_(pattern_id), variant_(v) {}
    Matd apply(std::size_t b, const char* p, const Matd& x) const {
        ++launches_;
        return eng_.forward(tensor_id(b, p), pattern_, x, variant_);
    }
    void qkv(std::size_t b, const Matd& hn, Matd& q, Matd& k, Matd& v) const override {
        q = apply(b, "q", hn);
        k = apply(b, "k", hn);
        v = apply(b, "v", hn);
    }
    Matd o_proj(std::size_t b, const Matd& x) const override { return apply(b, "o", x); }
    void upgate(std::size_t b, const Matd& hn, Matd& up, Matd& gate) const override {
        up = apply(b, "up", hn);
        gate = apply(b, "gate", hn);
    }
    Matd down_proj(std::size_t b, const Matd& x) const override { return apply(b, "down", x); }
    std::size_t launches() const { return launches_; }

private:
    const ExecEngine<double>& eng_;
    std::size_t pattern_;
    ExecVariant variant_;
    mutable std::size_t launches_ = 0;
};

// embed_prompt (pattern_cache.hpp:50-65): the block-0 forward through `prov`
// (the reference's forward_lm with any ProjectionProvider -- e.g. a GpuProvider
// or the static-prefix FactorizedProvider), then mean-pool + L2-normalise on
// the device (pg_embed_normalize: bit-exact pooling).
inline PromptEmbedding embed_prompt(const LmCore& core, const ProjectionProvider& prov,
                                    const std::vector<std::uint8_t>& tokens, const std::string& source = "") {
    if (tokens.empty()) throw std::invalid_argument("embed_prompt: empty prompt");
    std::vector<Matd> blocks;
    Capture cap;
    cap.block_outputs = true;
    cap.blocks = &blocks;
    KVCacheState kvc(core.cfg.n_blocks);
    forward_lm(core, prov, tokens, kvc, &cap);
    const Matd& b0 = blocks.front();
    DevBuf<double> xd(b0.data(), b0.rows() * b0.cols()), e(b0.rows());
    check(pg_embed_normalize(xd.p, PG_F64, PG_FEATURE_MAJOR, b0.rows(), b0.cols(), e.p, nullptr));
    return {e.host(), source};
}

// ---------------------------------------------------------------- provider
// RoutingProvider semantics (model.hpp:90-126) on the GPU: route once per
// tensor id from the first call's input, reuse the frozen selection after.
// `storage`: f64 (reference arithmetic), f32 or bf16 (f32 accumulation) device
// copies of every layer, resident for the provider's lifetime.
class GpuProvider : public ProjectionProvider {
public:
    explicit GpuProvider(const FactorizedModel& m, pg_dtype storage = PG_F64) : m_(m) {
        if (m.routers.empty()) throw std::runtime_error("model has no trained routers");
        for (const auto& [id, l] : m.layers) {
            layers_.emplace(id, std::make_unique<DeviceLayer>(l, storage));
            routers_.emplace(id, std::make_unique<DeviceRouter>(m.routers.at(id)));
        }
    }
    Matd apply(std::size_t b, const char* p, const Matd& x) const {
        const std::string id = tensor_id(b, p);
        auto it = selections_.find(id);
        if (it == selections_.end())
            it = selections_.emplace(id, route(*routers_.at(id), x, m_.layers.at(id).K)).first;
        return layers_.at(id)->forward(it->second, x);
    }
    void qkv(std::size_t b, const Matd& hn, Matd& q, Matd& k, Matd& v) const override {
        q = apply(b, "q", hn);
        k = apply(b, "k", hn);
        v = apply(b, "v", hn);
    }
    Matd o_proj(std::size_t b, const Matd& x) const override { return apply(b, "o", x); }
    void upgate(std::size_t b, const Matd& hn, Matd& up, Matd& gate) const override {
        up = apply(b, "up", hn);
        gate = apply(b, "gate", hn);
    }
    Matd down_proj(std::size_t b, const Matd& x) const override { return apply(b, "down", x); }
    const SelectionMap& selections() const { return selections_; }

private:
    const FactorizedModel& m_;
    std::map<std::string, std::unique_ptr<DeviceLayer>> layers_;
    std::map<std::string, std::unique_ptr<DeviceRouter>> routers_;
    mutable SelectionMap selections_;
};

// ---------------------------------------------------------------- serving composition
// route_prompt (pattern_cache.hpp:67-73) on the GPU: the prompt's prefill
// through GpuProvider (bit-exact routing), its frozen selections returned
inline SelectionMap route_prompt(const FactorizedModel& fm, const std::vector<std::uint8_t>& tokens) {
    GpuProvider prov(fm);
    KVCacheState kvc(fm.core.cfg.n_blocks);
    forward_lm(fm.core, prov, tokens, kvc);
    return prov.selections();
}

struct PromptSelection {
    SelectionMap pattern;      // the subsets the prompt is served with (prefill + every decode step)
    RetrieveResult retrieved;  // retrieve's answer (similarity -2 when the cache was empty)
    bool routed = false;       // miss: routed online
    bool inserted = false;     // miss: cache_insert accepted the routed pattern
};

// Retrieve-or-route (the north star's "S chosen by the router or by a
// pattern-cache lookup"): embed with the static-prefix model
// (pattern_cache.hpp:84), retrieve (:104-117); hit -> the entry's pattern;
// miss -> route_prompt + cache_insert (:120-124, refused at capacity).
inline PromptSelection select_for_prompt(const FactorizedModel& fm, DeviceCache& cache,
                                         const std::vector<std::uint8_t>& tokens) {
    const FactorizedProvider emb_prov(fm);
    PromptEmbedding emb = gpu::embed_prompt(fm.core, emb_prov, tokens);
    PromptSelection out;
    if (!cache.cache().entries.empty()) {
        out.retrieved = cache.retrieve(emb);
        if (out.retrieved.hit) {
            out.pattern = *out.retrieved.pattern;
            return out;
        }
    }
    out.routed = true;
    out.pattern = gpu::route_prompt(fm, tokens);
    CacheEntry e;
    e.embedding = std::move(emb);
    e.pattern = out.pattern;
    out.inserted = cache.insert(std::move(e));
    return out;
}

}  // namespace gpu
}  // namespace parse
