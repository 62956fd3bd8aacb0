// gempe.hpp -- header-only C++ facade over the C-ABI (gempe.h) with the reference's names and signatures
// (/root/reference/proj/include/entropy_embed/{graph,engine,errors}.hpp), so that code written against
// entropy_embed::embed / EmbeddingEngine compiles against the GPU path by switching the include:
//
//     #include <gempe.hpp>
//     namespace entropy_embed = gempe;          // Graph, Embedding, IterationConfig, EmbeddingEngine, embed, errors
//
// Link with -lgempe_b200.  Everything numerical runs in the library on the GPU; this header only converts types
// and maps return codes back to the reference's exception taxonomy.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gempe.h"

namespace gempe {

// ---- errors.hpp:10-47 -------------------------------------------------------------------------------
class parse_error : public std::runtime_error {
 public:
  parse_error(std::string msg, std::size_t line) : std::runtime_error(std::move(msg)), line_(line) {}
  std::size_t line() const noexcept { return line_; }

 private:
  std::size_t line_;
};
class data_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class near_complete_graph_error : public data_error {
 public:
  using data_error::data_error;
};
class config_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class divergence_error : public std::runtime_error {
 public:
  divergence_error(std::string msg, int iteration) : std::runtime_error(std::move(msg)), iteration_(iteration) {}
  int iteration() const noexcept { return iteration_; }

 private:
  int iteration_;
};
class cuda_error : public std::runtime_error {  // no reference analogue: there is no CPU fallback
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc, const std::string& msg, int iteration = 0) {
  switch (rc) {
    case GEMPE_OK: return;
    case GEMPE_ERR_CONFIG: throw config_error(msg);
    case GEMPE_ERR_DIVERGENCE: throw divergence_error(msg, iteration);
    case GEMPE_ERR_DATA:
      if (msg.find("near-complete") != std::string::npos) throw near_complete_graph_error(msg);
      throw data_error(msg);
    default: throw cuda_error(msg);
  }
}
}  // namespace detail

// ---- graph.hpp:12-29 ---------------------------------------------------------------------------------
struct Graph {
  std::uint32_t n = 0;
  std::vector<std::uint32_t> src;
  std::vector<std::uint32_t> dst;
  std::uint64_t edge_count() const { return src.size(); }
  std::uint64_t pair_count() const { return static_cast<std::uint64_t>(n) * (n > 0 ? n - 1 : 0) / 2; }
};
struct Permutation {
  std::vector<std::uint32_t> forward;  // original -> relabeled
  std::vector<std::uint32_t> inverse;  // relabeled -> original
};

// looks_like_snapshot ? load_graph_snapshot : load_edge_list (graph.hpp:35-45, embed_main.cpp:150-153)
inline Graph load_graph_file(const std::string& path, std::vector<std::uint64_t>* raw_labels = nullptr) {
  gempe_graph g{};
  std::uint64_t line = 0;
  const int rc = gempe_load_graph_file(path.c_str(), &g, &line);
  if (rc != GEMPE_OK) {
    const std::string msg = gempe_last_error(nullptr);
    if (rc == GEMPE_ERR_DATA && line) throw parse_error(msg, static_cast<std::size_t>(line));
    detail::check(rc, msg);
  }
  Graph out;
  out.n = g.n;
  out.src.assign(g.src, g.src + g.m);
  out.dst.assign(g.dst, g.dst + g.m);
  if (raw_labels) {
    raw_labels->clear();
    if (g.raw_labels) raw_labels->assign(g.raw_labels, g.raw_labels + g.n);
  }
  gempe_graph_free(&g);
  return out;
}

// ---- engine.hpp:18-38, 87-107 ---------------------------------------------------------------------------
struct Embedding {
  std::uint32_t n = 0;
  std::uint32_t dim = 0;
  std::vector<float> coords;
  float* row(std::uint32_t v) { return coords.data() + static_cast<std::size_t>(v) * dim; }
  const float* row(std::uint32_t v) const { return coords.data() + static_cast<std::size_t>(v) * dim; }
};

struct IterationConfig {
  int max_iters = 100;
  std::uint32_t lane_width = 16;  // accepted for source compatibility; sample streams never depended on it
  std::uint32_t workers = 0;      // accepted for source compatibility; unused on the GPU
  double convergence_tol = 1e-4;
  int convergence_window = 5;
  int relabel_period = 0;
  bool fast_math = true;
  std::optional<int> hash_bits;
  // extensions (defaults = reference behaviour)
  std::uint32_t negatives_per_vertex = 0;  // > 0: BASELINE sampling, k draws per vertex instead of 2 per edge
  int device = 0;
  bool deterministic = false;
  std::vector<int> devices;  // more than one entry: vertices sharded over these GPUs of the process (gempe_group)
};

struct IterationStats {
  double pe_estimate = 0.0;
  double sigma = 0.0;
};
struct IterationCapture {
  std::vector<double> y;
  std::vector<double> z;
};
struct TallySnapshot {  // DistanceHistogram's observable content (histogram.hpp)
  std::vector<std::uint64_t> edge, nonedge;
  double nonedge_weight = 1.0;
};
struct EmbedResult {
  Embedding embedding;  // original vertex indexing
  std::vector<double> pe_trace;
  double final_sigma = 1.0;
  bool converged = false;
  bool degenerate = false;
  int iterations = 0;
  Permutation relabel;
  TallySnapshot last_histogram;
};

// engine.hpp:112-134
class EmbeddingEngine {
 public:
  EmbeddingEngine(const Graph& g, std::uint32_t dim, const IterationConfig& cfg, std::uint64_t seed)
      : n_(g.n), m_(g.edge_count()), dim_(dim), max_iters_(cfg.max_iters) {
    if (cfg.hash_bits && (*cfg.hash_bits < 1 || *cfg.hash_bits > 31)) {
      throw config_error("hash table bits must be in [1,31]");
    }
    gempe_iteration_config c;
    gempe_default_iteration_config(&c);
    c.max_iters = cfg.max_iters;
    c.lane_width = cfg.lane_width;
    c.workers = cfg.workers;
    c.convergence_tol = cfg.convergence_tol;
    c.convergence_window = cfg.convergence_window;
    c.relabel_period = cfg.relabel_period;
    c.fast_math = cfg.fast_math ? 1 : 0;
    c.hash_bits = cfg.hash_bits.value_or(0);
    c.neg_mode = cfg.negatives_per_vertex ? GEMPE_NEG_PER_VERTEX_K : GEMPE_NEG_PER_EDGE_2;
    c.negatives = cfg.negatives_per_vertex;
    c.device = cfg.device;
    c.deterministic = cfg.deterministic ? 1 : 0;
    const int rc = gempe_engine_create_multi(&handle_, g.n, g.edge_count(), g.src.data(), g.dst.data(), dim, &c, seed,
                                             cfg.devices.empty() ? nullptr : cfg.devices.data(),
                                             static_cast<int>(cfg.devices.size()));
    detail::check(rc, gempe_last_error(nullptr));  // two statements: the message must be read AFTER the call
  }
  ~EmbeddingEngine() { gempe_engine_destroy(handle_); }
  EmbeddingEngine(const EmbeddingEngine&) = delete;
  EmbeddingEngine& operator=(const EmbeddingEngine&) = delete;

  bool degenerate() const { return gempe_engine_degenerate(handle_) != 0; }
  int iteration() const { return gempe_engine_iteration(handle_); }
  const std::vector<double>& pe_trace() const { return pe_trace_; }
  void set_capture(IterationCapture* capture) {
    capture_ = capture;
    gempe_set_capture(gempe_engine_context(handle_), capture ? 1 : 0);
  }

  IterationStats run_single_iteration() {
    IterationStats st;
    const int rc = gempe_engine_run_single_iteration(handle_, &st.pe_estimate, &st.sigma);
    detail::check(rc, gempe_engine_last_error(handle_), iteration() + 1);
    pe_trace_.push_back(st.pe_estimate);
    if (capture_) {
      capture_->y.resize(static_cast<std::size_t>(n_) * dim_);
      capture_->z.resize(n_);
      gempe_get_yz(gempe_engine_context(handle_), capture_->y.data(), capture_->z.data());
    }
    return st;
  }

  EmbedResult run() {
    EmbedResult r;
    r.embedding.n = n_;
    r.embedding.dim = dim_;
    r.embedding.coords.resize(static_cast<std::size_t>(n_) * dim_);
    r.pe_trace.resize(static_cast<std::size_t>(max_iters_ > 0 ? max_iters_ : 0));
    r.relabel.forward.resize(n_);
    r.last_histogram.edge.assign(GEMPE_HIST_BINS, 0);
    r.last_histogram.nonedge.assign(GEMPE_HIST_BINS, 0);
    gempe_embed_result out{};
    out.embedding = r.embedding.coords.data();
    out.pe_trace = r.pe_trace.data();
    out.pe_trace_cap = static_cast<std::int32_t>(r.pe_trace.size());
    out.relabel_forward = r.relabel.forward.data();
    out.last_hist_edge = r.last_histogram.edge.data();
    out.last_hist_nonedge = r.last_histogram.nonedge.data();
    const int rc = gempe_engine_run(handle_, &out);
    detail::check(rc, gempe_engine_last_error(handle_), iteration());
    r.pe_trace.resize(static_cast<std::size_t>(out.pe_trace_len));
    pe_trace_ = r.pe_trace;
    r.final_sigma = out.final_sigma;
    r.converged = out.converged != 0;
    r.degenerate = out.degenerate != 0;
    r.iterations = out.iterations;
    r.last_histogram.nonedge_weight = out.last_nonedge_weight;
    r.relabel.inverse.resize(n_);
    if (r.degenerate) {
      r.relabel.inverse = r.relabel.forward;  // engine.cpp:344-345
    } else {
      for (std::uint32_t v = 0; v < n_; ++v) r.relabel.inverse[r.relabel.forward[v]] = v;
    }
    return r;
  }

  // EmbeddingEngine::work_graph() / work_coords() (test hooks)
  Graph work_graph() const {
    Graph g;
    g.n = n_;
    g.src.resize(m_);
    g.dst.resize(m_);
    gempe_get_work_graph(gempe_engine_context(handle_), g.src.data(), g.dst.data(), nullptr);
    return g;
  }
  Embedding work_coords() const {
    Embedding e;
    e.n = n_;
    e.dim = dim_;
    e.coords.resize(static_cast<std::size_t>(n_) * dim_);
    if (n_) gempe_get_coords(gempe_engine_context(handle_), e.coords.data());
    return e;
  }
  double sigma() const { return gempe_engine_sigma(handle_); }

  // metrics.hpp:11-27: pe_sampled of the engine's current embedding, computed on the device
  struct PEReport {
    double pe = 0.0, mu_star = 0.0, sigma_star = 0.0, h_basic = 0.0, compression_ratio = 0.0, grid_pe = 0.0;
  };
  PEReport pe_sampled(int samples_per_edge, std::uint64_t seed) {
    gempe_pe_report r{};
    const int rc = gempe_pe_sampled(gempe_engine_context(handle_), samples_per_edge, seed, &r);
    detail::check(rc, gempe_last_error(gempe_engine_context(handle_)));
    return PEReport{r.pe, r.mu_star, r.sigma_star, r.h_basic, r.compression_ratio, r.grid_pe};
  }

 private:
  gempe_engine* handle_ = nullptr;
  std::uint32_t n_;
  std::uint64_t m_;
  std::uint32_t dim_;
  int max_iters_;
  std::vector<double> pe_trace_;
  IterationCapture* capture_ = nullptr;
};

// engine.hpp:170-171
inline EmbedResult embed(const Graph& g, std::uint32_t dim, const IterationConfig& cfg, std::uint64_t seed) {
  EmbeddingEngine engine(g, dim, cfg, seed);
  return engine.run();
}

// BASELINE.json's convenience form: embed(dim, iterations, negatives, seed)
inline EmbedResult embed(const Graph& g, std::uint32_t dim, int iterations, std::uint32_t negatives, std::uint64_t seed) {
  IterationConfig cfg;
  cfg.max_iters = iterations;
  cfg.negatives_per_vertex = negatives;
  return embed(g, dim, cfg, seed);
}

// io.hpp:17: write_embedding_tsv to a file
inline void write_embedding_tsv(const Embedding& emb, const std::vector<std::uint64_t>& labels, const std::string& path,
                                const Permutation* perm = nullptr) {
  if (!labels.empty() && labels.size() != emb.n) throw data_error("label count does not match embedding rows");
  const int rc = gempe_write_embedding_tsv(path.c_str(), emb.n, emb.dim, emb.coords.data(),
                                           labels.empty() ? nullptr : labels.data(), perm ? perm->forward.data() : nullptr);
  detail::check(rc, gempe_last_error(nullptr));
}

}  // namespace gempe
