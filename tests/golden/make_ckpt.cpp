// Golden checkpoint fixtures written by the REFERENCE's own serializers
// (checkpoint.hpp:135-163 save_factorized, pattern_cache.hpp:267-292
// save_cache), plus the reference's routed outputs on them, for the loader
// parity tests (tests/test_loaders.py).  Built and run by make_ckpt.py in this
// container only (needs /root/reference); the outputs are committed.
#include <cstdio>
#include <filesystem>
#include <fstream>

#include "parse/checkpoint.hpp"
#include "parse/model.hpp"
#include "parse/pattern_cache.hpp"
#include "parse/rank_experts.hpp"
#include "parse/rng.hpp"
#include "parse/router.hpp"

using namespace parse;

static Matd gauss(Rng& r, std::size_t rows, std::size_t cols, double s) {
    Matd m(rows, cols);
    for (auto& v : m.raw()) v = s * r.gaussian();
    return m;
}

int main(int argc, char** argv) {
    const std::filesystem::path out = argc > 1 ? argv[1] : "ckpt";
    Rng rng(20260517);
    FactorizedModel fm;
    fm.core.cfg.n_blocks = 1;
    fm.core.cfg.d_model = 32;
    fm.core.cfg.n_heads = 2;
    fm.core.cfg.n_kv_heads = 2;
    fm.core.cfg.d_ff = 48;
    fm.core.cfg.vocab = 8;
    fm.core.cfg.max_seq = 8;
    fm.core.cfg.seed = 7;
    const std::size_t d = 32, ff = 48;
    fm.core.embed = gauss(rng, 8, d, 1.0);
    fm.core.head = gauss(rng, 8, d, 1.0);
    fm.core.g_final.assign(d, 1.0);
    fm.core.g_attn.assign(1, std::vector<double>(d, 1.0));
    fm.core.g_mlp.assign(1, std::vector<double>(d, 1.0));
    fm.cfg.ratio = 0.6;
    fm.seed = 11;
    struct Shape { const char* p; std::size_t m, n; };
    const Shape shapes[] = {{"q", d, d}, {"k", d, d}, {"v", d, d}, {"o", d, d},
                            {"up", ff, d}, {"gate", ff, d}, {"down", d, ff}};
    std::ofstream exp(out / "expected.txt");
    std::filesystem::create_directories(out);
    std::ofstream expb(out / "expected_y.f64", std::ios::binary);
    std::ofstream expx(out / "x.f64", std::ios::binary);
    for (const auto& s : shapes) {
        const std::string id = tensor_id(0, s.p);
        FactorizedLayer l;
        l.layer_id = id;
        l.m = s.m;
        l.n = s.n;
        l.r_store = std::min(s.m, s.n);
        l.K = l.r_store / 2;
        l.A = gauss(rng, s.m, l.r_store, 0.5);
        l.B = gauss(rng, s.n, l.r_store, 0.5);
        l.sigma.assign(l.r_store, 1.0);
        l.whitened = false;
        RouterParams r;
        r.theta = gauss(rng, l.r_store, s.n, 1.0);
        r.bias.resize(l.r_store);
        for (auto& b : r.bias) b = 0.1 * rng.gaussian();
        // reference routing + value path on a fixed input (T = 5, feature-major)
        const Matd x = gauss(rng, s.n, 5, 1.0);
        const RankSelection sel = select_topk(score(r, mean_pool(x)), l.K);
        const Matd y = masked_forward(l, sel, x);
        exp << id << " " << l.K;
        for (auto e : sel.indices) exp << " " << e;
        exp << "\n";
        expx.write(reinterpret_cast<const char*>(x.raw().data()), std::streamsize(x.raw().size() * 8));
        expb.write(reinterpret_cast<const char*>(y.raw().data()), std::streamsize(y.raw().size() * 8));
        fm.layers[id] = l;
        fm.routers[id] = r;
    }
    save_factorized(out / "factorized", fm);
    // the reference's prompt embedding (block-0 output of the static-prefix
    // model, mean-pooled and normalised; pattern_cache.hpp:50-65, :84)
    {
        const std::vector<std::uint8_t> toks = {1, 5, 2, 7, 3, 0, 6};
        FactorizedProvider emb_prov(fm);
        const PromptEmbedding pe = embed_prompt(fm.core, emb_prov, toks, "golden");
        std::ofstream ef(out / "embed.f64", std::ios::binary);
        ef.write(reinterpret_cast<const char*>(pe.vec.data()), std::streamsize(pe.vec.size() * 8));
        std::ofstream tf(out / "embed_tokens.txt");
        for (auto t : toks) tf << int(t) << " ";
        tf << "\n";
    }
    // pattern cache: 6 entries, unit-norm embeddings, per-tensor selections
    PatternCache cache;
    cache.d_model = d;
    cache.capacity = 6;
    cache.min_similarity = 0.8;
    for (int e = 0; e < 6; ++e) {
        CacheEntry ce;
        ce.embedding.vec.resize(d);
        double nn = 0;
        for (auto& v : ce.embedding.vec) { v = rng.gaussian(); nn += v * v; }
        for (auto& v : ce.embedding.vec) v /= std::sqrt(nn);
        ce.embedding.source = "prompt-" + std::to_string(e);
        for (const auto& s : shapes) {
            const std::string id = tensor_id(0, s.p);
            const auto& l = fm.layers[id];
            std::vector<double> z(l.r_store);
            for (auto& v : z) v = rng.gaussian();
            ce.pattern[id] = select_topk(z, l.K);
        }
        cache.entries.push_back(ce);
    }
    save_cache(out / "cache", cache);
    // a query near entry 3 and its reference retrieval
    std::vector<double> q = cache.entries[3].embedding.vec;
    for (auto& v : q) v += 0.02 * rng.gaussian();
    double nq = 0;
    for (auto v : q) nq += v * v;
    for (auto& v : q) v /= std::sqrt(nq);
    const RetrieveResult rr = retrieve(cache, PromptEmbedding{q, "query"});
    std::ofstream qf(out / "query.f64", std::ios::binary);
    qf.write(reinterpret_cast<const char*>(q.data()), std::streamsize(q.size() * 8));
    std::FILE* f = std::fopen((out / "retrieve.txt").c_str(), "w");
    std::fprintf(f, "%zu %d %.17g\n", rr.entry, rr.hit ? 1 : 0, rr.similarity);
    std::fclose(f);
    return 0;
}
