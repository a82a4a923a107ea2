// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" wrapper that compiles the UNMODIFIED reference headers where
// they lie (-I/root/reference/proj/include) into oracle/_ref/libparse_ref.so,
// so tests and bench.py's reference arm can call the reference's own hot-path
// routines through ctypes.  No reference source is copied into this repo; this
// file only marshals plain arrays into the reference's types (parse::Matd,
// parse::RankSelection, parse::FactorizedLayer, parse::PatternCache, ...) and
// calls:
//   mean_pool / score / select_topk       include/parse/router.hpp:80,41,49
//   cosine / retrieve / embed pooling     include/parse/pattern_cache.hpp:38,104,60-64
//   check_selection / masked_forward      include/parse/rank_experts.hpp:30,52
//   aggregate_layout / aggregated_forward / scattered_forward
//                                         include/parse/exec_engine.hpp:113,194,240
//   maximal_runs                          include/parse/exec_engine.hpp:77
// Built by oracle/build.py with -O2 -ffp-contract=off (the reference's own
// CMake Release flags plus the FMA guard SURVEY.md §8c asks for).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "parse/exec_engine.hpp"
#include "parse/pattern_cache.hpp"
#include "parse/rank_experts.hpp"
#include "parse/router.hpp"

using namespace parse;

namespace {

int code_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const std::runtime_error&) {
        return 3;
    } catch (...) {
        return 9;
    }
}

Matd to_mat(const double* p, std::size_t r, std::size_t c) {
    Matd m(r, c);
    if (r * c) std::memcpy(m.data(), p, r * c * sizeof(double));
    return m;
}

FactorizedLayer make_layer(const double* A, const double* B, std::size_t m, std::size_t n,
                           std::size_t r) {
    FactorizedLayer fl;
    fl.layer_id = "ref";
    fl.m = m;
    fl.n = n;
    fl.r_store = r;
    fl.K = r;
    fl.A = to_mat(A, m, r);
    fl.B = to_mat(B, n, r);
    return fl;
}

std::vector<RankSelection> split_patterns(const std::uint32_t* pats, const std::size_t* ks,
                                          std::size_t P) {
    std::vector<RankSelection> out(P);
    std::size_t off = 0;
    for (std::size_t p = 0; p < P; ++p) {
        out[p].indices.assign(pats + off, pats + off + ks[p]);
        off += ks[p];
    }
    return out;
}

struct RefAgg {
    int elem;
    AggregatedLayer<float> f;
    AggregatedLayer<double> d;
};

}  // namespace

extern "C" {

void ref_mean_pool(const double* x, std::size_t n, std::size_t T, double* h) {
    std::vector<double> v = mean_pool(to_mat(x, n, T));
    std::memcpy(h, v.data(), n * sizeof(double));
}

void ref_score(const double* theta, const double* bias, std::size_t r, std::size_t n,
               const double* h, double* z) {
    RouterParams p;
    p.theta = to_mat(theta, r, n);
    p.bias.assign(bias, bias + r);
    std::vector<double> out = score(p, std::vector<double>(h, h + n));
    std::memcpy(z, out.data(), r * sizeof(double));
}

int ref_select_topk(const double* logits, std::size_t r, std::size_t k, std::uint32_t* out) {
    try {
        RankSelection s = select_topk(std::vector<double>(logits, logits + r), k);
        std::memcpy(out, s.indices.data(), k * sizeof(std::uint32_t));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

double ref_cosine(const double* a, const double* b, std::size_t d) {
    return cosine(std::vector<double>(a, a + d), std::vector<double>(b, b + d));
}

struct ref_retrieve_result {
    std::size_t entry;
    double similarity;
    int hit;
};

int ref_retrieve(const double* emb, std::size_t N, std::size_t d, double min_similarity,
                 const double* query, ref_retrieve_result* out) {
    PatternCache cache;
    cache.min_similarity = min_similarity;
    cache.capacity = N;
    cache.d_model = d;
    cache.entries.resize(N);
    for (std::size_t i = 0; i < N; ++i)
        cache.entries[i].embedding.vec.assign(emb + i * d, emb + (i + 1) * d);
    PromptEmbedding q;
    q.vec.assign(query, query + d);
    try {
        RetrieveResult r = retrieve(cache, q);
        out->entry = r.entry;
        out->similarity = r.similarity;
        out->hit = r.hit ? 1 : 0;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// embed_prompt's pooling half (pattern_cache.hpp:60-64), verbatim semantics:
// mean_pool(block output) then divide by vec_norm.
int ref_embed_normalize(const double* x, std::size_t d, std::size_t T, double* out) {
    std::vector<double> v = mean_pool(to_mat(x, d, T));
    const double nrm = vec_norm(v);
    if (nrm < 1e-12) return 3;
    for (double& e : v) e /= nrm;
    std::memcpy(out, v.data(), d * sizeof(double));
    return 0;
}

int ref_check_selection(const std::uint32_t* sel, std::size_t k, std::size_t r_store) {
    FactorizedLayer fl;
    fl.r_store = r_store;
    RankSelection s;
    s.indices.assign(sel, sel + k);
    try {
        check_selection(fl, s);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_masked_forward(const double* A, const double* B, std::size_t m, std::size_t n,
                       std::size_t r, const std::uint32_t* sel, std::size_t k, const double* x,
                       std::size_t T, double* out) {
    try {
        FactorizedLayer fl = make_layer(A, B, m, n, r);
        RankSelection s;
        s.indices.assign(sel, sel + k);
        Matd y = masked_forward(fl, s, to_mat(x, n, T));
        std::memcpy(out, y.data(), m * T * sizeof(double));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

void* ref_aggregate_layout(const double* A, const double* B, std::size_t m, std::size_t n,
                           std::size_t r, const std::uint32_t* pats, const std::size_t* ks,
                           std::size_t P, double psi, int elem, int* err) {
    *err = 0;
    try {
        FactorizedLayer fl = make_layer(A, B, m, n, r);
        auto sels = split_patterns(pats, ks, P);
        auto* g = new RefAgg;
        g->elem = elem;
        if (elem == 4) g->f = aggregate_layout<float>(fl, sels, psi);
        else g->d = aggregate_layout<double>(fl, sels, psi);
        return g;
    } catch (...) {
        *err = code_of(std::current_exception());
        return nullptr;
    }
}

void ref_agg_free(void* g) { delete static_cast<RefAgg*>(g); }

std::size_t ref_agg_shared_count(void* gp) {
    auto* g = static_cast<RefAgg*>(gp);
    return g->elem == 4 ? g->f.shared_ids.size() : g->d.shared_ids.size();
}
void ref_agg_shared_ids(void* gp, std::uint32_t* out) {
    auto* g = static_cast<RefAgg*>(gp);
    const auto& v = g->elem == 4 ? g->f.shared_ids : g->d.shared_ids;
    std::memcpy(out, v.data(), v.size() * sizeof(std::uint32_t));
}
std::size_t ref_agg_residual_count(void* gp, std::size_t p) {
    auto* g = static_cast<RefAgg*>(gp);
    return g->elem == 4 ? g->f.residuals[p].ids.size() : g->d.residuals[p].ids.size();
}
void ref_agg_residual_ids(void* gp, std::size_t p, std::uint32_t* out) {
    auto* g = static_cast<RefAgg*>(gp);
    const auto& v = g->elem == 4 ? g->f.residuals[p].ids : g->d.residuals[p].ids;
    std::memcpy(out, v.data(), v.size() * sizeof(std::uint32_t));
}
std::size_t ref_agg_arena_offset(void* gp, std::size_t p) {
    auto* g = static_cast<RefAgg*>(gp);
    return g->elem == 4 ? g->f.residuals[p].arena_offset : g->d.residuals[p].arena_offset;
}
void ref_agg_use_shared(void* gp, std::size_t p, std::uint8_t* out) {
    auto* g = static_cast<RefAgg*>(gp);
    const auto& v = g->elem == 4 ? g->f.residuals[p].use_shared : g->d.residuals[p].use_shared;
    std::memcpy(out, v.data(), v.size());
}

int ref_aggregated_forward_f32(void* gp, std::size_t pid, const float* x, std::size_t T,
                               float* out) {
    auto* g = static_cast<RefAgg*>(gp);
    try {
        Matf xm(g->f.n, T);
        std::memcpy(xm.data(), x, g->f.n * T * sizeof(float));
        Matf y = aggregated_forward(g->f, pid, xm);
        std::memcpy(out, y.data(), g->f.m * T * sizeof(float));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_aggregated_forward_f64(void* gp, std::size_t pid, const double* x, std::size_t T,
                               double* out) {
    auto* g = static_cast<RefAgg*>(gp);
    try {
        Matd y = aggregated_forward(g->d, pid, to_mat(x, g->d.n, T));
        std::memcpy(out, y.data(), g->d.m * T * sizeof(double));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

void ref_scattered_forward_f32(const float* A, const float* B, std::size_t m, std::size_t n,
                               std::size_t r, const std::uint32_t* sel, std::size_t k,
                               const float* x, std::size_t T, float* out) {
    Matf a(m, r), b(n, r), xm(n, T);
    std::memcpy(a.data(), A, m * r * sizeof(float));
    std::memcpy(b.data(), B, n * r * sizeof(float));
    std::memcpy(xm.data(), x, n * T * sizeof(float));
    RankSelection s;
    s.indices.assign(sel, sel + k);
    Matf y = scattered_forward(a, b, s, xm);
    std::memcpy(out, y.data(), m * T * sizeof(float));
}

std::size_t ref_maximal_runs(const std::size_t* cols, std::size_t count, std::size_t* starts,
                             std::size_t* lens) {
    auto runs = maximal_runs(std::vector<std::size_t>(cols, cols + count));
    for (std::size_t i = 0; i < runs.size(); ++i) {
        starts[i] = runs[i].start;
        lens[i] = runs[i].len;
    }
    return runs.size();
}

std::size_t ref_store_rank(std::size_t k, std::size_t r_max, double mult) {
    return store_rank(k, r_max, mult);
}

std::size_t ref_single_layer_k(std::size_t m, std::size_t n, double ratio) {
    std::vector<double> spectrum(std::min(m, n), 1.0);
    return allocate_budgets({spectrum}, {{m, n}}, ratio)[0];
}

// router.hpp:318-400 train_router_matrix on caller data: nseq sequences,
// sequence s has T[s] tokens, x_s (n x T_s) and y_s (m x T_s) concatenated
// row-major; outputs the returned (best-epoch) router and both loss curves.
int ref_train_router(const double* A, const double* B, std::size_t m, std::size_t n, std::size_t r, std::size_t K,
                     std::size_t nseq, const std::size_t* T, const double* xs, const double* ys, double lr,
                     std::size_t epochs, std::size_t batch, double warmup, double wd, std::uint64_t seed,
                     double tau, double* theta_out, double* bias_out, double* epoch_loss, double* frozen_loss) {
    try {
        FactorizedLayer fl = make_layer(A, B, m, n, r);
        fl.K = K;
        std::vector<RouterSeqStats> seqs;
        std::size_t ox = 0, oy = 0;
        for (std::size_t s = 0; s < nseq; ++s) {
            seqs.push_back(precompute_router_stats(fl, to_mat(xs + ox, n, T[s]), to_mat(ys + oy, m, T[s])));
            ox += n * T[s];
            oy += m * T[s];
        }
        RouterTrainConfig cfg;
        cfg.learning_rate = lr;
        cfg.epochs = epochs;
        cfg.batch_size = batch;
        cfg.warmup_frac = warmup;
        cfg.weight_decay = wd;
        cfg.seed = seed;
        RouterTrainResult res = train_router_matrix(fl, seqs, cfg, tau);
        std::memcpy(theta_out, res.params.theta.data(), r * n * sizeof(double));
        std::memcpy(bias_out, res.params.bias.data(), r * sizeof(double));
        std::memcpy(epoch_loss, res.epoch_loss.data(), epochs * sizeof(double));
        std::memcpy(frozen_loss, res.frozen_loss.data(), epochs * sizeof(double));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

void ref_fill_gaussian(std::uint64_t seed, double* out, std::size_t count) {
    Rng rng(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = rng.gaussian();
}

}  // extern "C"
