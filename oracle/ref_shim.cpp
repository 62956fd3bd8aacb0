// TEST INFRASTRUCTURE ONLY -- not part of the product path.
//
// C-ABI shim over the UNMODIFIED reference library (entropy-embed, compiled from
// /root/reference/proj/src/*.cpp where the sources lie; see oracle/Makefile).  The
// shim adds no arithmetic of its own: every function forwards to a public symbol of
// the reference (file:line cited at each wrapper).  The result, oracle/_ref/
// libgempe_ref.so, is used by tests/ as the ground truth, by tools/make_golden.py to
// generate tests/golden/*, and by bench.py as the `cpu_baseline` / `--impl reference`
// arm.  Nothing under paper_2011_03479_b200/ may load it.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "entropy_embed/engine.hpp"
#include "entropy_embed/errors.hpp"
#include "entropy_embed/graph.hpp"
#include "entropy_embed/hash_set.hpp"
#include "entropy_embed/histogram.hpp"
#include "entropy_embed/io.hpp"
#include "entropy_embed/metrics.hpp"
#include "entropy_embed/piecewise.hpp"
#include "entropy_embed/rng.hpp"
#include "entropy_embed/sampler.hpp"
#include "entropy_embed/sigmoid.hpp"
#include "entropy_embed/slope.hpp"

namespace ee = entropy_embed;

namespace {

thread_local std::string g_error;

// Exit-code convention of proj/tools/embed_main.cpp:214-230.
int classify(const std::exception& e) {
  g_error = e.what();
  if (dynamic_cast<const ee::divergence_error*>(&e)) return 3;
  if (dynamic_cast<const ee::config_error*>(&e)) return 1;
  return 2;
}

ee::Graph make_graph(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                     const std::uint32_t* dst) {
  ee::Graph g;
  g.n = n;
  g.src.assign(src, src + m);
  g.dst.assign(dst, dst + m);
  return g;
}

struct RefEngine {
  ee::Graph original;
  std::unique_ptr<ee::EmbeddingEngine> engine;
  ee::IterationCapture capture;
  std::uint64_t seed = 0;
};

struct RefHash {
  ee::EdgeHashSet hs;
};

ee::DistanceHistogram make_hist(const std::uint64_t* edge, const std::uint64_t* nonedge,
                                double nonedge_weight) {
  // DistanceHistogram has no counter setter (histogram.hpp:24-29): replay record().
  ee::DistanceHistogram h;
  for (int b = 0; b < h.bins(); ++b) {
    const double mid = h.bin_mid(b);
    for (std::uint64_t c = 0; c < edge[b]; ++c) h.record(mid, true);
    for (std::uint64_t c = 0; c < nonedge[b]; ++c) h.record(mid, false);
  }
  h.nonedge_weight = nonedge_weight;
  return h;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---- rng.hpp:17-34, 99-108 ----------------------------------------------------------
std::uint64_t ref_splitmix64(std::uint64_t z) { return ee::splitmix64(z); }
std::uint64_t ref_mix_seed(std::uint64_t s, std::uint64_t c) { return ee::mix_seed(s, c); }
std::uint32_t ref_expand_seed32(std::uint64_t s, std::uint64_t a, std::uint64_t b,
                                std::uint64_t c) {
  return ee::expand_seed32(s, a, b, c);
}
std::uint32_t ref_lane_uniform_index(std::uint32_t w, std::uint32_t n) {
  return ee::lane_uniform_index(w, n);
}
// hash_set.hpp:14-17
std::uint32_t ref_pair_hash(std::uint32_t i, std::uint32_t j, std::uint32_t n,
                            std::uint32_t size) {
  return ee::pair_hash(i, j, n, size);
}

// ---- graph.cpp:182-206, engine.cpp:116-124 -------------------------------------------
int ref_random_relabel(std::uint32_t n, std::uint64_t seed, std::uint32_t* forward) {
  ee::Graph g;
  g.n = n;
  auto [out, perm] = ee::random_relabel(g, seed);
  std::copy(perm.forward.begin(), perm.forward.end(), forward);
  return 0;
}
int ref_init_embedding(std::uint32_t n, std::uint32_t dim, std::uint64_t seed, float* out) {
  ee::Embedding e = ee::init_embedding(n, dim, seed);
  std::copy(e.coords.begin(), e.coords.end(), out);
  return 0;
}

// ---- hash_set.cpp:9-34, hash_set.hpp:28-30 --------------------------------------------
void* ref_hash_build(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                     const std::uint32_t* dst, int bits_override) {
  try {
    auto* h = new RefHash;
    std::optional<int> bits;
    if (bits_override > 0) bits = bits_override;
    h->hs = ee::EdgeHashSet::build(make_graph(n, m, src, dst), bits);
    return h;
  } catch (const std::exception& e) {
    classify(e);
    return nullptr;
  }
}
void ref_hash_free(void* h) { delete static_cast<RefHash*>(h); }
std::uint32_t ref_hash_size(void* h) { return static_cast<RefHash*>(h)->hs.size(); }
int ref_hash_bits(void* h) { return static_cast<RefHash*>(h)->hs.bits(); }
std::uint64_t ref_hash_occupied(void* h) { return static_cast<RefHash*>(h)->hs.occupied_cells(); }
void ref_hash_probe(void* h, const std::uint32_t* i, const std::uint32_t* j, std::uint64_t cnt,
                    std::uint8_t* out) {
  const auto& hs = static_cast<RefHash*>(h)->hs;
  for (std::uint64_t t = 0; t < cnt; ++t) out[t] = hs.maybe_edge(i[t], j[t]) ? 1 : 0;
}

// sampler.cpp:7-31 with one LaneRng lane per anchor; states are in/out.
int ref_sample_non_edges(void* h, std::uint32_t n, const std::uint32_t* anchors,
                         std::uint32_t* states, std::uint64_t cnt, std::uint32_t* out,
                         std::uint64_t* draws) {
  try {
    const auto& hs = static_cast<RefHash*>(h)->hs;
    ee::LaneRng rng;
    rng.state.assign(states, states + cnt);
    std::uint64_t dc = 0;
    ee::sample_non_edges(std::span<const std::uint32_t>(anchors, cnt), rng, hs, n,
                         std::span<std::uint32_t>(out, cnt), &dc);
    std::copy(rng.state.begin(), rng.state.end(), states);
    if (draws) *draws = dc;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// ---- sigmoid.hpp:88-101, piecewise.hpp:72-84, piecewise.cpp:182-195 ---------------------
// table: 0 = erf, 1 = exp_neg, 2 = gauss/erfc ratio.  Layout: knots[17], a[16], b[16], c[16], lo, hi.
int ref_fastmath_table(int table, double* out67) {
  static const ee::FastMath fm = ee::FastMath::build();
  const ee::PiecewiseQuad& q =
      table == 0 ? fm.erf_table : (table == 1 ? fm.exp_neg_table : fm.gauss_erfc_table);
  double* p = out67;
  for (double k : q.knots) *p++ = k;
  for (double v : q.a) *p++ = v;
  for (double v : q.b) *p++ = v;
  for (double v : q.c) *p++ = v;
  *p++ = q.lo;
  *p++ = q.hi;
  return q.odd_mirror ? 1 : 0;
}
double ref_gauss_erfc_ratio(double x, int fast) {
  static const ee::FastMath fm = ee::FastMath::build();
  return fast ? fm.gauss_erfc_ratio(x) : ee::detail::gauss_over_erfc(x);
}
void ref_parabola(double delta, double mu, double sigma, int is_edge, int fast, double* d_target,
                  double* w) {
  static const ee::FastMath fm = ee::FastMath::build();
  const ee::SigmoidParams p{mu, sigma};
  const ee::Parabola pb = fast ? ee::parabola_params_fast(delta, p, is_edge != 0, fm)
                               : ee::parabola_params(delta, p, is_edge != 0);
  *d_target = pb.d_target;
  *w = pb.w;
}
double ref_description_length(double delta, double mu, double sigma, int is_edge) {
  return ee::description_length(delta, {mu, sigma}, is_edge != 0);
}

// ---- slope.cpp:27-38, 75-125 ---------------------------------------------------------------
int ref_optimize_sigma(const std::uint64_t* edge, const std::uint64_t* nonedge,
                       double nonedge_weight, double mu, double* sigma, int* steps) {
  try {
    const ee::DistanceHistogram h = make_hist(edge, nonedge, nonedge_weight);
    const ee::SigmaSearchResult r = ee::optimize_sigma_detail(h, mu);
    *sigma = r.sigma;
    if (steps) *steps = r.bisection_steps;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}
double ref_histogram_objective(const std::uint64_t* edge, const std::uint64_t* nonedge,
                               double nonedge_weight, double mu, double sigma) {
  return ee::histogram_objective(make_hist(edge, nonedge, nonedge_weight), {mu, sigma});
}
double ref_histogram_objective_dsigma(const std::uint64_t* edge, const std::uint64_t* nonedge,
                                      double nonedge_weight, double mu, double sigma) {
  return ee::histogram_objective_dsigma(make_hist(edge, nonedge, nonedge_weight), {mu, sigma});
}

// ---- engine.hpp:112-134, engine.cpp:143-388 ----------------------------------------------------
void* ref_engine_create(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                        const std::uint32_t* dst, std::uint32_t dim, std::uint32_t lane_width,
                        std::uint32_t workers, int fast_math, int hash_bits, int relabel_period,
                        int max_iters, double convergence_tol, int convergence_window,
                        std::uint64_t seed) {
  try {
    auto eng = std::make_unique<RefEngine>();
    eng->original = make_graph(n, m, src, dst);
    eng->seed = seed;
    ee::IterationConfig cfg;
    cfg.max_iters = max_iters;
    cfg.lane_width = lane_width;
    cfg.workers = workers;
    cfg.convergence_tol = convergence_tol;
    cfg.convergence_window = convergence_window;
    cfg.relabel_period = relabel_period;
    cfg.fast_math = fast_math != 0;
    if (hash_bits > 0) cfg.hash_bits = hash_bits;
    eng->engine = std::make_unique<ee::EmbeddingEngine>(eng->original, dim, cfg, seed);
    eng->engine->set_capture(&eng->capture);
    return eng.release();
  } catch (const std::exception& e) {
    classify(e);
    return nullptr;
  }
}
void ref_engine_free(void* h) { delete static_cast<RefEngine*>(h); }
int ref_engine_degenerate(void* h) { return static_cast<RefEngine*>(h)->engine->degenerate(); }
int ref_engine_iteration(void* h) { return static_cast<RefEngine*>(h)->engine->iteration(); }
double ref_engine_sigma(void* h) { return static_cast<RefEngine*>(h)->engine->params().sigma; }
std::uint32_t ref_engine_hash_size(void* h) {
  return static_cast<RefEngine*>(h)->engine->hash_set().size();
}
void ref_engine_work_graph(void* h, std::uint32_t* src, std::uint32_t* dst) {
  const ee::Graph& g = static_cast<RefEngine*>(h)->engine->work_graph();
  std::copy(g.src.begin(), g.src.end(), src);
  std::copy(g.dst.begin(), g.dst.end(), dst);
}
void ref_engine_work_coords(void* h, float* out) {
  const ee::Embedding& e = static_cast<RefEngine*>(h)->engine->work_coords();
  std::copy(e.coords.begin(), e.coords.end(), out);
}
void ref_engine_probe(void* h, const std::uint32_t* i, const std::uint32_t* j, std::uint64_t cnt,
                      std::uint8_t* out) {
  const auto& hs = static_cast<RefEngine*>(h)->engine->hash_set();
  for (std::uint64_t t = 0; t < cnt; ++t) out[t] = hs.maybe_edge(i[t], j[t]) ? 1 : 0;
}
// One run_single_iteration (engine.cpp:278-325).  y/z may be null (skips the capture copy-out).
int ref_engine_iterate(void* h, double* pe_estimate, double* sigma, double* y, double* z) {
  auto* eng = static_cast<RefEngine*>(h);
  try {
    const ee::IterationStats st = eng->engine->run_single_iteration();
    if (pe_estimate) *pe_estimate = st.pe_estimate;
    if (sigma) *sigma = st.sigma;
    if (y) std::copy(eng->capture.y.begin(), eng->capture.y.end(), y);
    if (z) std::copy(eng->capture.z.begin(), eng->capture.z.end(), z);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}
void ref_engine_set_capture(void* h, int on) {
  auto* eng = static_cast<RefEngine*>(h);
  eng->engine->set_capture(on ? &eng->capture : nullptr);
}
// EmbeddingEngine::run (engine.cpp:339-382): embedding in ORIGINAL indexing.
int ref_engine_run(void* h, float* embedding, double* pe_trace, int pe_cap, int* iterations,
                   int* converged, int* degenerate, double* final_sigma,
                   std::uint32_t* relabel_forward, std::uint64_t* hist_edge,
                   std::uint64_t* hist_nonedge, double* nonedge_weight) {
  auto* eng = static_cast<RefEngine*>(h);
  try {
    const ee::EmbedResult r = eng->engine->run();
    if (embedding) std::copy(r.embedding.coords.begin(), r.embedding.coords.end(), embedding);
    if (pe_trace) {
      for (int i = 0; i < pe_cap && i < static_cast<int>(r.pe_trace.size()); ++i) {
        pe_trace[i] = r.pe_trace[i];
      }
    }
    if (iterations) *iterations = r.iterations;
    if (converged) *converged = r.converged;
    if (degenerate) *degenerate = r.degenerate;
    if (final_sigma) *final_sigma = r.final_sigma;
    if (relabel_forward) {
      std::copy(r.relabel.forward.begin(), r.relabel.forward.end(), relabel_forward);
    }
    if (hist_edge && hist_nonedge && !r.degenerate) {
      for (int b = 0; b < r.last_histogram.bins(); ++b) {
        hist_edge[b] = r.last_histogram.edge_count(b);
        hist_nonedge[b] = r.last_histogram.nonedge_count(b);
      }
      if (nonedge_weight) *nonedge_weight = r.last_histogram.nonedge_weight;
    }
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// metrics.cpp:139 pe_exact (guarded at 1e8 pairs) -- scoring only.
int ref_pe_exact(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                 const std::uint32_t* dst, std::uint32_t dim, const float* coords, double* pe) {
  try {
    ee::Embedding e;
    e.n = n;
    e.dim = dim;
    e.coords.assign(coords, coords + static_cast<std::size_t>(n) * dim);
    *pe = ee::pe_exact(make_graph(n, m, src, dst), e).pe;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// metrics.cpp:166 pe_sampled -- scoring only.
int ref_pe_sampled(std::uint32_t n, std::uint64_t m, const std::uint32_t* src, const std::uint32_t* dst,
                   std::uint32_t dim, const float* coords, int samples_per_edge, std::uint64_t seed, double* pe) {
  try {
    ee::Embedding e;
    e.n = n;
    e.dim = dim;
    e.coords.assign(coords, coords + static_cast<std::size_t>(n) * dim);
    *pe = ee::pe_sampled(make_graph(n, m, src, dst), e, samples_per_edge, seed).pe;
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// ---- graph.cpp:75-170, io.cpp:17-46 (text formats) ---------------------------------------------------------
// Returns 0 and fills n / m (call again with arrays sized n / m to receive them), 2 on data_error, 5 on
// parse_error with *line set.
int ref_load_edge_list(const char* text, std::uint64_t len, std::uint32_t* n, std::uint64_t* m, std::uint32_t* src,
                       std::uint32_t* dst, std::uint64_t* labels, std::uint64_t* line) {
  try {
    std::istringstream in(std::string(text, len));
    std::vector<std::uint64_t> raw;
    const ee::Graph g = ee::load_edge_list(in, &raw);
    *n = g.n;
    *m = g.edge_count();
    if (src) std::copy(g.src.begin(), g.src.end(), src);
    if (dst) std::copy(g.dst.begin(), g.dst.end(), dst);
    if (labels) std::copy(raw.begin(), raw.end(), labels);
    return 0;
  } catch (const ee::parse_error& e) {
    g_error = e.what();
    if (line) *line = e.line();
    return 5;
  } catch (const std::exception& e) {
    return classify(e);
  }
}
// write_embedding_tsv into a caller buffer; returns the text length (or -1 when cap is too small / on error)
long ref_write_embedding_tsv(std::uint32_t n, std::uint32_t dim, const float* coords, const std::uint64_t* labels,
                             const std::uint32_t* perm_forward, char* out, long cap) {
  try {
    ee::Embedding e;
    e.n = n;
    e.dim = dim;
    e.coords.assign(coords, coords + static_cast<std::size_t>(n) * dim);
    std::vector<std::uint64_t> lab;
    if (labels) lab.assign(labels, labels + n);
    ee::Permutation perm;
    if (perm_forward) perm.forward.assign(perm_forward, perm_forward + n);
    std::ostringstream os;
    ee::write_embedding_tsv(e, lab, os, perm_forward ? &perm : nullptr);
    const std::string s = os.str();
    if (static_cast<long>(s.size()) > cap) return -1;
    std::memcpy(out, s.data(), s.size());
    return static_cast<long>(s.size());
  } catch (const std::exception& e) {
    classify(e);
    return -1;
  }
}
long ref_save_graph_snapshot(std::uint32_t n, std::uint64_t m, const std::uint32_t* src, const std::uint32_t* dst,
                             char* out, long cap) {
  std::ostringstream os(std::ios::binary);
  ee::save_graph_snapshot(make_graph(n, m, src, dst), os);
  const std::string s = os.str();
  if (static_cast<long>(s.size()) > cap) return -1;
  std::memcpy(out, s.data(), s.size());
  return static_cast<long>(s.size());
}

}  // extern "C"
