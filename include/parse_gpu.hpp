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
//   pattern_cache.hpp:104 retrieve                gpu::DeviceCache::retrieve / gpu::retrieve
//   pattern_cache.hpp:120 cache_insert            gpu::DeviceCache::insert
//   rank_experts.hpp:52   masked_forward          gpu::masked_forward     f64: <= 1e-10 rel
//   exec_engine.hpp:113/194 aggregate_layout / aggregated_forward  gpu::DeviceAggregatedLayer
//   toy_lm.hpp:68  ProjectionProvider             gpu::GpuProvider (RoutingProvider semantics)
//
// Host-memory convenience: each call copies its operands to the device and the
// result back (synchronous).  Serving code keeps handles resident and uses the
// C-ABI (parse_gpu.h) with device pointers and streams directly.
#pragma once

#include <cuda_runtime.h>

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
class DeviceCache {
public:
    explicit DeviceCache(PatternCache& cache) : cache_(cache) {
        check(pg_cache_create(&h_, cache.d_model, cache.capacity, cache.min_similarity));
        std::vector<double> emb;
        for (const auto& e : cache.entries) emb.insert(emb.end(), e.embedding.vec.begin(), e.embedding.vec.end());
        check(pg_cache_load(h_, emb.data(), cache.entries.size()));
    }
    ~DeviceCache() { pg_cache_destroy(h_); }
    DeviceCache(const DeviceCache&) = delete;
    DeviceCache& operator=(const DeviceCache&) = delete;

    RetrieveResult retrieve(const PromptEmbedding& emb) const {
        if (cache_.entries.empty()) throw std::runtime_error("empty cache");
        DevBuf<double> q(emb.vec.data(), emb.vec.size());
        pg_retrieve_result r{};
        check(pg_retrieve(h_, q.p, 0, &r, nullptr, nullptr, nullptr));
        RetrieveResult out;
        out.entry = r.entry;
        out.similarity = r.similarity;
        out.hit = r.hit != 0;
        out.pattern = &cache_.entries[r.entry].pattern;
        return out;
    }
    // cache_insert (pattern_cache.hpp:120-124): refused once at capacity
    bool insert(CacheEntry entry) {
        int ins = 0;
        check(pg_cache_insert(h_, entry.embedding.vec.data(), 0, &ins, nullptr));
        if (ins) cache_.entries.push_back(std::move(entry));
        return ins != 0;
    }

private:
    PatternCache& cache_;
    pg_cache h_ = nullptr;
};

inline RetrieveResult retrieve(PatternCache& cache, const PromptEmbedding& emb) {
    if (cache.entries.empty()) throw std::runtime_error("empty cache");
    DeviceCache dc(cache);
    return dc.retrieve(emb);
}

// ---------------------------------------------------------------- layers
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

    // masked_forward with f64 storage (rank_experts.hpp:52-72)
    Matd forward(const RankSelection& sel, const Matd& x) const {
        if (x.rows() != n_) throw std::invalid_argument("masked_forward: bad X shape");
        DevBuf<double> xd(x.data(), x.rows() * x.cols()), y(m_ * x.cols());
        check(pg_masked_forward(h_, sel.indices.data(), sel.indices.size(), 0, xd.p, PG_FEATURE_MAJOR,
                                x.cols(), y.p, PG_F64, nullptr));
        Matd out(m_, x.cols());
        std::vector<double> hy = y.host();
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

// ---------------------------------------------------------------- provider
// RoutingProvider semantics (model.hpp:90-126) on the GPU: route once per
// tensor id from the first call's input, reuse the frozen selection after.
class GpuProvider : public ProjectionProvider {
public:
    explicit GpuProvider(const FactorizedModel& m) : m_(m) {
        if (m.routers.empty()) throw std::runtime_error("model has no trained routers");
        for (const auto& [id, l] : m.layers) {
            layers_.emplace(id, std::make_unique<DeviceLayer>(l, PG_F64));
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

}  // namespace gpu
}  // namespace parse
