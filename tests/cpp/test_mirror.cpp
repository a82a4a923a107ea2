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
//     frozen selection reused by decode_step (toy_lm.hpp:274);
//  3. the reference's exec-engine test cases (test_exec_engine.cpp:128-226)
//     against parse::gpu::{aggregate_layout<T>, aggregated_forward<T>,
//     scattered_forward<T>, ExecEngine<T>, ExecProvider};
//  4. embed_prompt, retrieve(const PatternCache&), cache_insert, and the f32 /
//     bf16 resident GpuProvider through forward_lm.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

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

// the reference test's toy model (test_exec_engine.cpp:12-27 configuration)
static FactorizedModel small_model() {
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
    return compress_model(dense, calib, cc);
}

// prefix-biased random K-subsets per tensor (the reference test's generator rule)
static std::vector<SelectionMap> patterns_for(const FactorizedModel& fm, std::size_t count, std::uint64_t seed) {
    Rng rng(seed);
    std::vector<SelectionMap> pats(count);
    for (auto& p : pats)
        for (const auto& [id, layer] : fm.layers) {
            std::vector<std::uint32_t> pool(layer.r_store);
            std::iota(pool.begin(), pool.end(), 0u);
            RankSelection sel;
            for (std::size_t i = 0; i < layer.K; ++i) {
                const std::size_t pick = rng.below(2) ? 0 : rng.below(pool.size());
                sel.indices.push_back(pool[pick]);
                pool.erase(pool.begin() + std::ptrdiff_t(pick));
            }
            std::sort(sel.indices.begin(), sel.indices.end());
            p[id] = std::move(sel);
        }
    return pats;
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
    // ---- 3. exec engine on the device (test_exec_engine.cpp:128-226)
    {
        const FactorizedModel fm = small_model();
        const auto pats = patterns_for(fm, 4, 17);
        const auto eng = gpu::ExecEngine<double>::build(fm, pats, 0.5);
        const auto ref_eng = ExecEngine<double>::build(fm, pats, 0.5);
        bool same_layout = true;
        for (const auto& [id, t] : ref_eng.tensors) {
            const auto& g = eng.tensors.at(id).agg;
            same_layout = same_layout && g.shared_ids == t.agg.shared_ids;
            for (std::size_t p = 0; p < pats.size(); ++p)
                same_layout = same_layout && g.residuals[p].ids == t.agg.residuals[p].ids &&
                              g.residuals[p].use_shared == t.agg.residuals[p].use_shared &&
                              g.residuals[p].arena_offset == t.agg.residuals[p].arena_offset;
        }
        EXPECT(same_layout, "ExecEngine<double>::build: shared / residual / use_shared / arena_offset as the reference");
        Rng rng(19);
        double worst = 0;
        bool agg_pair = true, scat_pair = true;
        for (const auto& [id, layer] : fm.layers) {
            Matd x(layer.n, 6);
            for (double& v : x.raw()) v = rng.gaussian();
            for (std::size_t pid = 0; pid < pats.size(); ++pid) {
                const Matd ref = masked_forward(layer, pats[pid].at(id), x);
                const Matd a1 = eng.forward(id, pid, x, ExecVariant::aggregated_only);
                const Matd a2 = eng.forward(id, pid, x, ExecVariant::aggregated_fused);
                const Matd s1 = eng.forward(id, pid, x, ExecVariant::scattered_unfused);
                const Matd s2 = eng.forward(id, pid, x, ExecVariant::fused_only);
                for (const Matd* m : {&a1, &a2, &s1, &s2}) worst = std::max(worst, max_rel(*m, ref));
                agg_pair = agg_pair && a1.raw() == a2.raw();
                scat_pair = scat_pair && s1.raw() == s2.raw();
                const Matd sf = gpu::scattered_forward(ref_eng.tensors.at(id).a_full, ref_eng.tensors.at(id).b_full,
                                                       pats[pid].at(id), x);
                scat_pair = scat_pair && sf.raw() == s1.raw();
            }
        }
        std::printf("     four variants vs masked_forward: max rel %.3e\n", worst);
        EXPECT(worst <= 1e-12, "all four variants vs masked_forward, f64 <= 1e-12 (test_exec_engine.cpp:128-146)");
        EXPECT(agg_pair && scat_pair, "aggregated variants bit-identical to each other, scattered likewise");

        const auto pats3 = patterns_for(fm, 3, 23);
        const auto engf = gpu::ExecEngine<float>::build(fm, pats3, 0.5);
        Rng rf(29);
        bool close = true;
        for (const auto& [id, layer] : fm.layers) {
            Matd x(layer.n, 4);
            for (double& v : x.raw()) v = rf.gaussian();
            const Matf xf = x.cast<float>();
            for (std::size_t pid = 0; pid < pats3.size(); ++pid) {
                const Matd ref = masked_forward(layer, pats3[pid].at(id), x);
                const Matf got = engf.forward(id, pid, xf, ExecVariant::aggregated_fused);
                for (std::size_t i = 0; i < ref.raw().size(); ++i)
                    close = close && std::abs(double(got.raw()[i]) - ref.raw()[i]) < 1e-5 * (1.0 + std::abs(ref.raw()[i]));
            }
        }
        EXPECT(close, "float engine within 1e-5 (1 + |ref|) of the double reference (:148-165)");

        bool runs = true;
        Rng rt(37);
        for (const auto& [id, layer] : fm.layers) {
            Matd x(layer.n, 2);
            for (double& v : x.raw()) v = rt.gaussian();
            for (std::size_t pid = 0; pid < pats.size(); ++pid) {
                AccessTrace tr, sc;
                eng.forward(id, pid, x, ExecVariant::aggregated_fused, &tr);
                const auto& agg = eng.tensors.at(id).agg;
                runs = runs && tr.a_cols.size() == agg.shared_ids.size() + agg.residuals[pid].ids.size();
                runs = runs && maximal_runs(tr.a_cols).size() <= 2 && maximal_runs(tr.b_cols).size() <= 2;
                eng.forward(id, pid, x, ExecVariant::scattered_unfused, &sc);
                const std::vector<std::size_t> want(pats[pid].at(id).indices.begin(), pats[pid].at(id).indices.end());
                runs = runs && sc.a_cols == want;
            }
        }
        EXPECT(runs, "aggregated trace <= 2 contiguous runs, scattered trace = S (:167-193)");

        auto one = patterns_for(fm, 1, 41);
        const std::vector<SelectionMap> same = {one[0], one[0], one[0]};
        const auto varied = patterns_for(fm, 4, 43);
        EXPECT(gpu::ExecEngine<double>::build(fm, same, 0.9).storage_overhead() == 0.0 &&
                   gpu::ExecEngine<double>::build(fm, varied, 0.9).storage_overhead() ==
                       ExecEngine<double>::build(fm, varied, 0.9).storage_overhead(),
               "storage_overhead as the reference (:195-208)");

        const auto p2 = patterns_for(fm, 2, 47);
        const auto eng2 = gpu::ExecEngine<double>::build(fm, p2, 0.5);
        const auto toks = sample_calibration({DomainKind::markov_text, 5, 0}, 1, 12, 9)[0];
        double lm_worst = 0;
        for (std::size_t pid = 0; pid < p2.size(); ++pid) {
            const FactorizedProvider ref_prov(fm, &p2[pid]);
            KVCacheState kv1(fm.core.cfg.n_blocks);
            const Matd ref = forward_lm(fm.core, ref_prov, toks, kv1);
            for (ExecVariant v : {ExecVariant::scattered_unfused, ExecVariant::aggregated_fused}) {
                const gpu::ExecProvider prov(eng2, pid, v);
                KVCacheState kv2(fm.core.cfg.n_blocks);
                lm_worst = std::max(lm_worst, max_rel(forward_lm(fm.core, prov, toks, kv2), ref));
            }
        }
        std::printf("     ExecProvider full LM vs FactorizedProvider: max rel %.3e\n", lm_worst);
        EXPECT(lm_worst <= 1e-9, "ExecProvider serves the full LM like the masked provider, <= 1e-9 (:210-226)");

        bool threw = false;
        try {
            gpu::aggregated_forward(eng.tensors.begin()->second.agg, 99, Matd(16, 1));
        } catch (const std::out_of_range&) {
            threw = true;
        }
        EXPECT(threw, "aggregated_forward unknown pattern -> out_of_range");
    }
    // ---- 4. embed_prompt, const retrieve, cache_insert, f32 / bf16 GpuProvider
    {
        FactorizedModel fm = small_model();
        const FactorizedProvider static_prov(fm);  // the embedding model (pattern_cache.hpp:84)
        PatternCache cache;
        cache.d_model = fm.core.cfg.d_model;
        cache.capacity = 3;
        cache.min_similarity = 0.8;
        const auto prompts = sample_calibration({DomainKind::markov_text, 5, 0}, 4, 16, 11);
        bool emb_exact = true;
        for (std::size_t i = 0; i < 3; ++i) {
            const PromptEmbedding ref = embed_prompt(fm.core, static_prov, prompts[i]);
            const PromptEmbedding got = gpu::embed_prompt(fm.core, static_prov, prompts[i]);
            emb_exact = emb_exact && got.vec == ref.vec;
            CacheEntry e;
            e.embedding = got;
            e.pattern = patterns_for(fm, 1, 60 + i)[0];
            EXPECT(gpu::cache_insert(cache, e), "cache_insert below capacity");
        }
        EXPECT(emb_exact, "embed_prompt: device pooling bit-identical to the reference");
        CacheEntry extra;
        extra.embedding = gpu::embed_prompt(fm.core, static_prov, prompts[3]);
        EXPECT(!gpu::cache_insert(cache, extra) && cache.entries.size() == 3, "cache_insert refused at capacity");
        const PatternCache& cc = cache;
        bool rr = true;
        for (std::size_t i = 0; i < 4; ++i) {
            const PromptEmbedding q = embed_prompt(fm.core, static_prov, prompts[i]);
            const RetrieveResult a = gpu::retrieve(cc, q), b = retrieve(cc, q);
            rr = rr && a.entry == b.entry && a.hit == b.hit && a.pattern == b.pattern && a.similarity == b.similarity;
        }
        EXPECT(rr, "retrieve(const PatternCache&): entry, hit, pattern pointer, similarity as the reference");

        std::uint64_t seed = 300;
        for (const auto& [id, layer] : fm.layers) {
            RouterParams p = make_router(layer.r_store, layer.n);
            p.theta = random_mat(layer.r_store, layer.n, ++seed);
            fm.routers[id] = std::move(p);
        }
        const auto toks = sample_calibration({DomainKind::markov_text, 5, 0}, 1, 12, 9)[0];
        RoutingProvider ref(fm);
        KVCacheState kv0(fm.core.cfg.n_blocks);
        const Matd l0 = forward_lm(fm.core, ref, toks, kv0);
        for (pg_dtype dt : {PG_F32, PG_BF16}) {
            gpu::GpuProvider dev(fm, dt);
            KVCacheState kv(fm.core.cfg.n_blocks);
            const Matd l = forward_lm(fm.core, dev, toks, kv);
            bool sel_same = true;
            for (const auto& [id, s] : ref.selections()) sel_same = sel_same && dev.selections().at(id).indices == s.indices;
            const double e = max_rel(l, l0);
            std::printf("     GpuProvider %s storage: logits max rel %.3e\n", dt == PG_F32 ? "f32" : "bf16", e);
            EXPECT(sel_same && e <= (dt == PG_F32 ? 1e-4 : 5e-2),
                   dt == PG_F32 ? "f32 GpuProvider: same routes, logits <= 1e-4"
                                : "bf16 GpuProvider: same routes, logits <= 5e-2");
        }
    }
    // ---- 5. retrieve-or-route composition vs the reference build_cache / route_prompt
    {
        FactorizedModel fm = small_model();
        std::uint64_t seed = 500;
        for (const auto& [id, layer] : fm.layers) {
            RouterParams p = make_router(layer.r_store, layer.n);
            p.theta = random_mat(layer.r_store, layer.n, ++seed);
            fm.routers[id] = std::move(p);
        }
        const auto prompts = sample_calibration({DomainKind::markov_text, 5, 0}, 5, 16, 21);
        const std::vector<std::vector<std::uint8_t>> first(prompts.begin(), prompts.begin() + 3);
        PatternCache cache = build_cache(fm, first, 0.99999, 4);  // reference: embeddings + routed patterns
        gpu::DeviceCache dc(cache);
        const auto s1 = gpu::select_for_prompt(fm, dc, prompts[1]);
        bool same_pat = s1.pattern.size() == cache.entries[1].pattern.size();
        for (const auto& [id, sel] : cache.entries[1].pattern)
            same_pat = same_pat && s1.pattern.count(id) && s1.pattern.at(id).indices == sel.indices;
        EXPECT(!s1.routed && s1.retrieved.hit && s1.retrieved.entry == 1 && same_pat,
               "select_for_prompt: cached prompt hits its own entry and serves its pattern");
        const RetrieveResult want = retrieve(cache, embed_prompt(fm.core, FactorizedProvider(fm), prompts[3]));
        const auto s3 = gpu::select_for_prompt(fm, dc, prompts[3]);
        bool same_route = s3.pattern.size() == fm.layers.size();
        const SelectionMap ref_route = route_prompt(fm, prompts[3]);
        for (const auto& [id, sel] : ref_route) same_route = same_route && s3.pattern.at(id).indices == sel.indices;
        EXPECT(!want.hit && s3.routed && same_route && s3.inserted && cache.entries.size() == 4,
               "select_for_prompt: a miss routes exactly like route_prompt and is inserted");
        const auto s4 = gpu::select_for_prompt(fm, dc, prompts[4]);
        EXPECT(s4.routed && !s4.inserted && cache.entries.size() == 4, "select_for_prompt: at capacity, not inserted");
        const auto s3b = gpu::select_for_prompt(fm, dc, prompts[3]);
        EXPECT(!s3b.routed && s3b.retrieved.entry == 3, "select_for_prompt: the routed prompt now hits its entry");
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "PASSED", g_fail);
    return g_fail ? 1 : 0;
}
