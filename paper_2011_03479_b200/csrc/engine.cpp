// Run-level facade over the device context: the host half of EmbeddingEngine
// (/root/reference/proj/src/engine.cpp:278-388) -- sigma search on the round's tallies, PE trace, best-PE
// snapshot, convergence window, periodic re-relabel, map-back to original ids.  The Jacobi round itself
// is gempe_iterate (context.cpp); nothing here touches coordinates on the host except the final export.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <thread>

#include "context.hpp"

using namespace gempe;

struct gempe_engine {
  gempe_ctx* ctx = nullptr;      // the engine's context; rank 0 of `group` (and owned by it) when the engine is sharded
  gempe_group* group = nullptr;  // several GPUs (gempe_engine_create_multi)
  gempe_iteration_config cfg{};
  std::uint64_t seed = 0;
  std::uint32_t n = 0, dim = 0;
  std::uint64_t m = 0;
  double mu = kDefaultMu, sigma = 1.0;  // SigmoidParams defaults (sigmoid.hpp:18-21)
  int iter = 0;
  std::vector<double> pe_trace;
  Tallies last_hist;
  bool have_hist = false;
  bool sigma_seeded = false;
  bool queued_converged = false, queued_best = false;  // outcome of a run queued on the device (run_queued)
  double best_pe = std::numeric_limits<double>::infinity();
  DeviceBuffer<float> best_x;               // device snapshot, WORK indexing of the moment it was taken
  std::vector<std::uint32_t> best_to_work;
  std::string error;

  ~gempe_engine() {
    if (group) gempe_group_destroy(group);
    else gempe_destroy(ctx);
  }
};

namespace {

template <typename Fn>
int guarded(gempe_engine* e, Fn&& fn) {
  try {
    fn();
    return GEMPE_OK;
  } catch (const divergence_error& ex) {
    e->error = ex.what();
    return GEMPE_ERR_DIVERGENCE;
  } catch (const config_error& ex) {
    e->error = ex.what();
    return GEMPE_ERR_CONFIG;
  } catch (const cuda_error& ex) {
    e->error = ex.what();
    return GEMPE_ERR_CUDA;
  } catch (const std::exception& ex) {
    e->error = ex.what();
    return GEMPE_ERR_DATA;
  }
}

void rethrow_message(int rc, const std::string& msg);
void rethrow(gempe_ctx* c, int rc) {
  if (rc == GEMPE_OK) return;
  rethrow_message(rc, gempe_last_error(c));
}
void rethrow(gempe_group* g, int rc) {
  if (rc == GEMPE_OK) return;
  rethrow_message(rc, gempe_group_last_error(g));
}
void rethrow_message(int rc, const std::string& msg) {
  switch (rc) {
    case GEMPE_ERR_CONFIG: throw config_error(msg);
    case GEMPE_ERR_DIVERGENCE: throw divergence_error(msg, 0);
    case GEMPE_ERR_CUDA: throw cuda_error(msg);
    default: throw data_error(msg);
  }
}

// original-indexed export of a work-indexed device layout (engine.cpp:327-337, 376-381): rows gathered on the
// device, one transfer into the caller's buffer
void map_back(gempe_engine* e, const float* x_dev, const std::vector<std::uint32_t>& to_work, float* out) {
  gempe_ctx* c = e->ctx;
  if (e->n == 0) return;
  PhaseTimer timer;
  DeviceBuffer<std::uint32_t> d_map;
  DeviceBuffer<float> own;
  d_map.upload(to_work);
  // the rows are packed (un-relabelled, pitch dim) into the round's OUTPUT buffer, which holds nothing once the round is
  // over and is rewritten by the next one -- no half-gigabyte allocation per export.  A group's buffers are written by
  // peers, and the snapshot may itself live there: those cases get a buffer of their own.
  const std::size_t floats = static_cast<std::size_t>(e->n) * e->dim;
  float* packed = c->x[c->cur ^ 1].get();
  if (e->group || x_dev == packed || c->x[c->cur ^ 1].size() < floats) {
    own.allocate(floats);
    packed = own.get();
  }
  c->launches += launch_permute_rows(x_dev, c->ld, packed, e->dim, e->dim, e->n, d_map.get(), false, c->stream);
  cuda_check(cudaStreamSynchronize(c->stream), "map_back");
  timer.lap("export: un-relabel (device)");
  download_to_pageable(out, packed, floats * sizeof(float), c->stream);
  timer.lap("export: download");
}

void single_iteration(gempe_engine* e, double* pe_out, double* sigma_out) {
  gempe_ctx* c = e->ctx;
  if (c->degenerate) throw config_error("cannot iterate a degenerate graph");
  if (e->cfg.relabel_period > 0 && e->iter > 0 && e->iter % e->cfg.relabel_period == 0) {  // engine.cpp:281-283
    const std::uint64_t relabel_seed = mix_seed(mix_seed(e->seed, 0xA11BE11), static_cast<std::uint64_t>(e->iter));
    if (e->group) rethrow(e->group, gempe_group_relabel(e->group, relabel_seed));
    else rethrow(c, gempe_relabel(c, relabel_seed));
  }
  Tallies t;
  double pe = 0.0;
  const std::uint64_t pairs = static_cast<std::uint64_t>(e->n) * (e->n > 0 ? e->n - 1 : 0) / 2;
  if (e->cfg.host_sigma) {
    if (e->group) {
      rethrow(e->group, gempe_group_iterate(e->group, e->mu, e->sigma, static_cast<std::uint64_t>(e->iter), t.edge.data(),
                                            t.nonedge.data()));
    } else {
      rethrow(c, gempe_iterate(c, e->mu, e->sigma, static_cast<std::uint64_t>(e->iter), t.edge.data(), t.nonedge.data()));
    }
    const std::uint64_t samples = t.nonedge_total();
    t.nonedge_weight = samples > 0 ? static_cast<double>(pairs - e->m) / static_cast<double>(samples) : 1.0;
    // growth-capped sigma update (engine.cpp:302-307)
    e->sigma = std::min(optimize_sigma(t, e->mu).sigma, e->sigma * 1.5);
    pe = histogram_objective(t, e->mu, e->sigma) / static_cast<double>(pairs);
  } else {
    // sigma search, growth cap and PE estimate on the device (sigma_update_kernel)
    if (!e->sigma_seeded) {
      if (e->group) rethrow(e->group, gempe_group_set_sigma(e->group, e->mu, e->sigma));
      else rethrow(c, gempe_set_sigma(c, e->mu, e->sigma));
      e->sigma_seeded = true;
    }
    if (e->group) {  // every rank searches sigma on its own device from the summed tallies
      rethrow(e->group, gempe_group_iterate_auto(e->group, static_cast<std::uint64_t>(e->iter), &e->sigma, &pe,
                                                 &t.nonedge_weight, t.edge.data(), t.nonedge.data()));
    } else {
      rethrow(c, gempe_iterate_auto(c, static_cast<std::uint64_t>(e->iter), &e->sigma, &pe, &t.nonedge_weight,
                                    t.edge.data(), t.nonedge.data()));
    }
  }
  e->pe_trace.push_back(pe);
  e->last_hist = t;
  e->have_hist = true;
  ++e->iter;
  if (pe < e->best_pe) {  // engine.cpp:316-319, kept on the device
    e->best_pe = pe;
    const std::size_t count = static_cast<std::size_t>(c->n_pad) * c->ld;
    if (e->best_x.size() != count) e->best_x.allocate(count);
    cuda_check(cudaMemcpyAsync(e->best_x.get(), c->x[c->cur].get(), count * sizeof(float), cudaMemcpyDeviceToDevice,
                               c->stream), "best snapshot");
    e->best_to_work = c->to_work;
  }
  if (pe_out) *pe_out = pe;
  if (sigma_out) *sigma_out = e->sigma;
}

// EmbeddingEngine::run (engine.cpp:349-373) with the loop on the device: whole iterations are queued in batches, the
// device keeps the PE trace, the best-PE snapshot and the convergence window, the host looks every `batch` rounds (and at
// every re-relabel boundary, which needs the host).  Returns false when the run has to fall back to the host loop.
bool run_queued(gempe_engine* e, int batch, bool use_graph) {
  gempe_ctx* c = e->ctx;
  const int max_iters = e->cfg.max_iters;
  if (e->iter != 0 || max_iters <= 0) return false;  // a run that continues manual steps keeps the host loop
  const std::uint32_t max_rounds = static_cast<std::uint32_t>(max_iters);
  rethrow(c, gempe_run_begin(c, e->mu, e->sigma, 0, e->cfg.convergence_window, e->cfg.convergence_tol, max_rounds));
  e->sigma_seeded = true;
  const int period = e->cfg.relabel_period;
  gempe_run_status st{};
  std::uint64_t improved_seen = 0;
  std::vector<double> trace(max_rounds);
  while (true) {
    std::uint64_t stop_at = max_rounds;
    if (period > 0) stop_at = std::min<std::uint64_t>(stop_at, (static_cast<std::uint64_t>(e->iter) / period + 1) * period);
    const std::uint64_t todo = stop_at - static_cast<std::uint64_t>(e->iter);
    // a graph always replays `batch` rounds (the surplus ones are no-ops); plain launches queue only what is left
    const std::uint32_t rounds = use_graph ? static_cast<std::uint32_t>(batch)
                                           : static_cast<std::uint32_t>(std::min<std::uint64_t>(batch, todo));
    rethrow(c, gempe_run_enqueue(c, rounds, stop_at, use_graph ? 1 : 0));
    rethrow(c, gempe_run_poll(c, &st, trace.data(), nullptr, max_rounds, e->last_hist.edge.data(), e->last_hist.nonedge.data()));
    e->iter = static_cast<int>(st.rounds_done);
    if (st.improved_at != improved_seen) {  // the snapshot on the device was taken under the current relabelling
      improved_seen = st.improved_at;
      e->best_to_work = c->to_work;
    }
    if (st.converged || e->iter >= max_iters) break;
    if (period > 0 && e->iter > 0 && e->iter % period == 0) {  // engine.cpp:281-283
      rethrow(c, gempe_relabel(c, mix_seed(mix_seed(e->seed, 0xA11BE11), static_cast<std::uint64_t>(e->iter))));
      rethrow(c, gempe_run_rebase(c));
    }
  }
  e->pe_trace.assign(trace.begin(), trace.begin() + e->iter);
  e->sigma = st.sigma;
  e->best_pe = st.best_pe;
  e->last_hist.nonedge_weight = st.last_nonedge_weight;
  e->have_hist = e->iter > 0;
  e->queued_converged = st.converged != 0;
  e->queued_best = st.improved_at > 0;
  return true;
}

}  // namespace

extern "C" {

void gempe_default_iteration_config(gempe_iteration_config* cfg) {
  std::memset(cfg, 0, sizeof *cfg);
  cfg->max_iters = 100;
  cfg->lane_width = 16;
  cfg->workers = 0;
  cfg->convergence_tol = 1e-4;
  cfg->convergence_window = 5;
  cfg->relabel_period = 0;
  cfg->fast_math = 1;
  cfg->hash_bits = 0;
  cfg->neg_mode = GEMPE_NEG_PER_EDGE_2;
  cfg->negatives = 0;
  cfg->device = 0;
  cfg->host_sigma = 0;
  cfg->deterministic = 0;
  cfg->batch_rounds = 0;
}

int gempe_engine_create(gempe_engine** out, std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                        const std::uint32_t* dst, std::uint32_t dim, const gempe_iteration_config* cfg,
                        std::uint64_t seed) {
  return gempe_engine_create_multi(out, n, m, src, dst, dim, cfg, seed, nullptr, 0);
}

int gempe_engine_create_multi(gempe_engine** out, std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                              const std::uint32_t* dst, std::uint32_t dim, const gempe_iteration_config* cfg,
                              std::uint64_t seed, const int* devices, int n_devices) {
  if (!out || !cfg || (n_devices > 0 && !devices)) return GEMPE_ERR_CONFIG;
  *out = nullptr;
  auto e = std::make_unique<gempe_engine>();
  e->cfg = *cfg;
  e->seed = seed;
  e->n = n;
  e->m = m;
  e->dim = dim;
  // config validation of the reference ctor (engine.cpp:152-154); hash_bits is validated by gempe_create
  const char* bad = dim < 1 ? "dimension must be >= 1"
                            : (cfg->lane_width < 1 ? "lane width must be >= 1"
                                                   : (cfg->max_iters < 1 ? "max_iters must be >= 1" : nullptr));
  gempe_options opt;
  gempe_default_options(&opt);
  opt.dim = dim;
  opt.hash_bits = cfg->hash_bits;
  opt.seed = seed;
  opt.neg_mode = cfg->neg_mode;
  opt.negatives = cfg->negatives;
  opt.math = cfg->fast_math ? GEMPE_MATH_TABLES : GEMPE_MATH_EXACT;
  opt.device = cfg->device;
  opt.deterministic = cfg->deterministic;
  int rc = GEMPE_ERR_CONFIG;
  if (!bad && n_devices > 1) {  // vertices sharded over the listed devices, one rank each (group.cpp)
    rc = gempe_group_create(&e->group, n, m, src, dst, &opt, devices, n_devices, 0);
    if (rc == GEMPE_OK) e->ctx = gempe_group_context(e->group, 0);
    else set_create_error(gempe_group_last_error(nullptr));
  } else if (!bad) {
    if (n_devices == 1) opt.device = devices[0];
    rc = gempe_create(&e->ctx, n, m, src, dst, &opt);
  }
  if (bad) set_create_error(bad);
  if (bad || rc != GEMPE_OK) return rc;  // message: gempe_last_error(NULL)
  *out = e.release();
  return GEMPE_OK;
}

void gempe_engine_destroy(gempe_engine* e) { delete e; }
const char* gempe_engine_last_error(const gempe_engine* e) { return e ? e->error.c_str() : ""; }
gempe_ctx* gempe_engine_context(gempe_engine* e) { return e->ctx; }
int gempe_engine_degenerate(const gempe_engine* e) { return e->ctx ? e->ctx->degenerate : 0; }
int gempe_engine_iteration(const gempe_engine* e) { return e->iter; }
double gempe_engine_sigma(const gempe_engine* e) { return e->sigma; }

int gempe_engine_run_single_iteration(gempe_engine* e, double* pe_estimate, double* sigma) {
  return guarded(e, [&] {
    if (!e->ctx) throw config_error("engine was not constructed: " + e->error);
    single_iteration(e, pe_estimate, sigma);
  });
}

int gempe_engine_run(gempe_engine* e, gempe_embed_result* r) {
  return guarded(e, [&] {
    if (!e->ctx) throw config_error("engine was not constructed: " + e->error);
    if (!r || !r->embedding) throw config_error("result needs an embedding buffer");
    gempe_ctx* c = e->ctx;
    r->converged = 0;
    r->degenerate = c->degenerate;
    r->pe_trace_len = 0;
    r->iterations = 0;
    r->final_sigma = e->sigma;
    r->last_nonedge_weight = 1.0;
    if (c->degenerate) {  // engine.cpp:341-347: initial layout, identity relabel
      map_back(e, c->x[c->cur].get(), c->to_work, r->embedding);
      if (r->relabel_forward) std::copy(c->to_work.begin(), c->to_work.end(), r->relabel_forward);
      return;
    }
    // device sigma search: the whole loop runs on the device, the host looks every few rounds
    PhaseTimer timer;
    bool queued = false;
    if (!e->cfg.host_sigma && e->cfg.batch_rounds >= 0 && !e->group) {
      const bool small = gempe_pair_terms(c) < 4000000ull;  // launch-bound rounds: replay them as one CUDA graph
      const int batch = e->cfg.batch_rounds > 0 ? e->cfg.batch_rounds : (small ? 16 : 4);
      queued = run_queued(e, batch, small && batch > 1);
    }
    timer.lap(queued ? "run (queued rounds)" : "run (setup)");
    if (queued) {
      r->converged = e->queued_converged ? 1 : 0;
      if (!r->converged && e->queued_best) {
        map_back(e, static_cast<const float*>(gempe_run_best_snapshot(c)), e->best_to_work, r->embedding);
      } else {
        map_back(e, c->x[c->cur].get(), c->to_work, r->embedding);
      }
    }
    // converged when the last `window` rounds brought no new PE minimum beating the earlier best by tol
    // (engine.cpp:353-367)
    const int window = e->cfg.convergence_window;
    while (!queued && e->iter < e->cfg.max_iters) {
      single_iteration(e, nullptr, nullptr);
      const int k = static_cast<int>(e->pe_trace.size());
      if (k > window) {
        const double best_before = *std::min_element(e->pe_trace.begin(), e->pe_trace.begin() + (k - window));
        const double best_recent = *std::min_element(e->pe_trace.begin() + (k - window), e->pe_trace.end());
        if (best_before - best_recent < e->cfg.convergence_tol * std::fabs(best_before)) {
          r->converged = 1;
          break;
        }
      }
    }
    if (queued) {
      // exported above
    } else if (!r->converged && e->best_x.size()) {
      map_back(e, e->best_x.get(), e->best_to_work, r->embedding);
    } else {
      map_back(e, c->x[c->cur].get(), c->to_work, r->embedding);
    }
    r->pe_trace_len = static_cast<std::int32_t>(e->pe_trace.size());
    if (r->pe_trace) {
      const int copy = std::min<int>(r->pe_trace_cap, r->pe_trace_len);
      std::copy(e->pe_trace.begin(), e->pe_trace.begin() + copy, r->pe_trace);
    }
    r->final_sigma = e->sigma;
    r->iterations = e->iter;
    if (r->relabel_forward) std::copy(c->to_work.begin(), c->to_work.end(), r->relabel_forward);
    if (e->have_hist) {
      if (r->last_hist_edge) std::copy(e->last_hist.edge.begin(), e->last_hist.edge.end(), r->last_hist_edge);
      if (r->last_hist_nonedge) std::copy(e->last_hist.nonedge.begin(), e->last_hist.nonedge.end(), r->last_hist_nonedge);
      r->last_nonedge_weight = e->last_hist.nonedge_weight;
    }
  });
}

}  // extern "C"
