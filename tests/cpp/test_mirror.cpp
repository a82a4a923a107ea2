// test_mirror.cpp -- the C++ drop-in boundary (include/parse_gpu.hpp) exercised
// through the reference's OWN types and model code, compiled against the
// reference headers (tests/cpp/build.py) and run on the GPU by
// tests/test_gpu_cpp_mirror.py.
//
//  1. unit parity of parse::gpu::{mean_pool, score, select_topk, cosine,
//     retrieve, masked_forward, DeviceAggregatedLayer} vs parse::*;
//  2. drop-in: forward_lm (toy_lm.hpp:201) with parse::gpu::GpuProvider vs the
//     reference RoutingProvider (model.hpp:90-126) on a compressed toy model
//     with random routers: identical selections, logits within 1e-9, and the
//     frozen selection reused by decode_step (toy_lm.hpp:274).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "parse/corpus.hpp"
#include "parse_gpu.hpp"

using namespace parse;

static int g_fail = 0;
#define EXPECT(cond, what)                                                   \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__);      \
            ++g_fail;                                                        \
        } else {                                                             \
            std::printf("ok   %s\n", what);                                  \
        }                                                                    \
    } while (0)

static Matd random_mat(std::size_t m, std::size_t n, std::uint64_t seed) {
    Matd a(m, n);
    Rng rng(seed);
    for (double& v : a.raw()) v = rng.gaussian();
    return a;
}

static double max_rel(const Matd& a, const Matd& b) {
    double d = 0, s = 1e-300;
    for (std::size_t i = 0; i < a.raw().size(); ++i) {
        d = std::max(d, std::abs(a.raw()[i] - b.raw()[i]));
        s = std::max(s, std::abs(b.raw()[i]));
    }
    return d / s;
}

int main() {
    // ---- 1. unit parity
    {
        const Matd x = random_mat(96, 17, 1);
        EXPECT(gpu::mean_pool(x) == mean_pool(x), "mean_pool bit-exact");
        RouterParams r = make_router(64, 96);
        r.theta = random_mat(64, 96, 2);
        for (std::size_t i = 0; i < 64; ++i) r.bias[i] = 0.01 * double(i % 5);
        const auto h = mean_pool(x);
        EXPECT(gpu::score(r, h) == score(r, h), "score bit-exact");
        const auto z = score(r, h);
        for (std::size_t k : {std::size_t(1), std::size_t(20), std::size_t(64)})
            EXPECT(gpu::select_topk(z, k).indices == select_topk(z, k).indices, "select_topk bit-exact");
        EXPECT(gpu::select_topk({1, 2, 2, 1, 2}, 2).indices == (std::vector<std::uint32_t>{1, 2}),
               "select_topk lower-index ties (test_router.cpp:78)");
        bool threw = false;
        try {
            gpu::select_topk({1, 2, 3}, 0);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw, "select_topk K=0 throws invalid_argument");
        gpu::DeviceRouter dr(r);
        EXPECT(gpu::route(dr, x, 20).indices == select_topk(score(r, mean_pool(x)), 20).indices,
               "fused route == select_topk(score(mean_pool))");
        const std::vector<double> a = random_mat(1, 200, 3).raw(), b = random_mat(1, 200, 4).raw();
        EXPECT(gpu::cosine(a, b) == cosine(a, b), "cosine bit-exact");
    }
    {
        PatternCache cache;
        cache.min_similarity = 0.9;
        cache.capacity = 3;
        cache.d_model = 2;
        CacheEntry e1, e2;
        e1.embedding.vec = {1, 0};
        e1.pattern["t"] = RankSelection{{0}};
        e2.embedding.vec = {0, 1};
        e2.pattern["t"] = RankSelection{{1}};
        cache.entries = {e1, e2};
        gpu::DeviceCache dc(cache);
        const RetrieveResult r = dc.retrieve(PromptEmbedding{{0.995, 0.0998}, ""});
        const RetrieveResult w = retrieve(cache, PromptEmbedding{{0.995, 0.0998}, ""});
        EXPECT(r.entry == w.entry && r.hit == w.hit && r.pattern == w.pattern, "retrieve entry/hit/pattern");
        const RetrieveResult f = dc.retrieve(PromptEmbedding{{0.707, 0.707}, ""});
        EXPECT(!f.hit && f.pattern != nullptr, "retrieve below threshold misses");
        EXPECT(dc.insert(e1) && !dc.insert(e1) && cache.entries.size() == 3, "cache_insert capacity rule");
    }
    {
        FactorizedLayer fl;
        fl.m = 40; fl.n = 30; fl.r_store = 24; fl.K = 12;
        fl.A = random_mat(40, 24, 5);
        fl.B = random_mat(30, 24, 6);
        const Matd x = random_mat(30, 7, 7);
        const RankSelection sel{{0, 2, 3, 7, 8, 11, 13, 17, 19, 20, 22, 23}};
        EXPECT(max_rel(gpu::masked_forward(fl, sel, x), masked_forward(fl, sel, x)) <= 1e-12,
               "masked_forward f64 within 1e-12");
        bool threw = false;
        try {
            gpu::masked_forward(fl, RankSelection{{0, 24}}, x);
        } catch (const std::out_of_range&) {
            threw = true;
        }
        EXPECT(threw, "selection beyond r_store throws out_of_range");
        const std::vector<RankSelection> pats = {RankSelection{{0, 1}}, RankSelection{{0, 1}}, RankSelection{{0, 2}}};
        gpu::DeviceAggregatedLayer g(fl, pats, 0.9);
        const auto ref = aggregate_layout<double>(fl, pats, 0.9);
        EXPECT(g.shared_ids() == ref.shared_ids, "aggregate_layout shared ids (test_exec_engine.cpp:97)");
        for (std::size_t p = 0; p < pats.size(); ++p) {
            AccessTrace tr;
            const Matd y = g.forward(p, x, &tr);
            EXPECT(max_rel(y, aggregated_forward(ref, p, x)) <= 1e-12, "aggregated_forward f64 within 1e-12");
            EXPECT(maximal_runs(tr.a_cols).size() <= 2, "aggregated trace <= 2 contiguous runs");
        }
    }
    // ---- 2. drop-in through forward_lm
    {
        ToyLMConfig cfg;
        cfg.n_blocks = 2;
        cfg.d_model = 16;
        cfg.n_heads = 2;
        cfg.n_kv_heads = 2;
        cfg.d_ff = 24;
        cfg.max_seq = 128;
        cfg.seed = 91;
        const DenseModel dense = init_dense_model(cfg);
        const auto calib = sample_calibration({DomainKind::markov_text, 1, 0}, 8, 24, 3);
        CompressionConfig cc;
        cc.ratio = 0.3;
        FactorizedModel fm = compress_model(dense, calib, cc);
        std::uint64_t seed = 100;
        for (const auto& [id, layer] : fm.layers) {
            RouterParams p = make_router(layer.r_store, layer.n);
            p.theta = random_mat(layer.r_store, layer.n, ++seed);
            fm.routers[id] = std::move(p);
        }
        const auto toks = sample_calibration({DomainKind::markov_text, 5, 0}, 1, 12, 9)[0];
        RoutingProvider ref(fm);
        gpu::GpuProvider dev(fm);
        KVCacheState kv1(cfg.n_blocks), kv2(cfg.n_blocks);
        const Matd l1 = forward_lm(fm.core, ref, toks, kv1);
        const Matd l2 = forward_lm(fm.core, dev, toks, kv2);
        bool same_sel = ref.selections().size() == dev.selections().size();
        for (const auto& [id, s] : ref.selections()) same_sel = same_sel && dev.selections().at(id).indices == s.indices;
        EXPECT(same_sel, "GpuProvider routes every tensor id exactly like RoutingProvider");
        EXPECT(max_rel(l2, l1) <= 1e-9, "prefill logits through forward_lm within 1e-9");
        const auto d1 = decode_step(fm.core, ref, kv1, 7);
        const auto d2 = decode_step(fm.core, dev, kv2, 7);
        double dm = 0, ds = 1e-300;
        for (std::size_t i = 0; i < d1.size(); ++i) {
            dm = std::max(dm, std::abs(d1[i] - d2[i]));
            ds = std::max(ds, std::abs(d1[i]));
        }
        EXPECT(dm / ds <= 1e-9, "decode_step logits within 1e-9 (frozen selection reused)");
        bool still = true;
        for (const auto& [id, s] : ref.selections()) still = still && dev.selections().at(id).indices == s.indices;
        EXPECT(still, "decode never re-routes");
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "PASSED", g_fail);
    return g_fail ? 1 : 0;
}
