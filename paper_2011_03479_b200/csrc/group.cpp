// Multi-GPU host of the GEMPE round inside ONE process (include/gempe.h "gempe_group"): one context per
// device, vertices sharded over them, every rank holding the full X_t, CSR and edge filter.  The round sequence is the
// one of INTEGRATION.md section 5, driven from the calling thread through the ranks' own streams and ordered with
// CUDA events only -- no kernel waits on another rank's kernel, no host synchronisation inside a round:
//
//   rank r:  sample own anchors + pack (partner, anchor) records by owner     [records land at their owners]
//            -- event barrier: every rank's pack of this round (and, behind it in stream order, its gather of the
//               previous round) has finished --
//            bucket the received records, gather + update own vertices         [updated rows land on every rank]
//
// With peer access between all devices (NVLink / NVSwitch, or several ranks on one device) the pack kernel stores its
// records straight into the owners' receive areas and the gather kernel stores every updated row into every rank's
// X_{t+1}: the transfers are the kernels' own stores, nothing else moves.  Without peer access the same data moves
// with copy engines (cudaMemcpyPeerAsync): the packed regions as an all-to-all, the owned row blocks as an all-gather.
// The 2 x 512 tallies are summed on the device (a kernel reading the ranks' tallies) for the sigma search that every
// rank runs redundantly, or on the host for gempe_group_iterate.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "context.hpp"

using namespace gempe;

struct gempe_group {
  std::vector<gempe_ctx*> ctx;
  std::vector<int> device;
  std::vector<cudaEvent_t> packed, bucketed, gathered, summed;  // one per rank, re-recorded every round
  std::vector<DeviceBuffer<unsigned long long>> total;           // job-wide tallies on every rank
  bool peer_stores = false;
  bool sigma_seeded = false;
  std::uint32_t n = 0, dim = 0;
  std::uint64_t m = 0;
  double mu = kDefaultMu;
  std::string error;

  ~gempe_group() {
    for (std::size_t r = 0; r < ctx.size(); ++r) {
      if (ctx[r]) cudaSetDevice(device[r]);
      for (auto* list : {&packed, &bucketed, &gathered, &summed}) {
        if (r < list->size() && (*list)[r]) cudaEventDestroy((*list)[r]);
      }
      if (r < total.size()) total[r].release();
      gempe_destroy(ctx[r]);
    }
  }
};

namespace {

thread_local std::string g_group_create_error;

struct group_failure : std::runtime_error {
  group_failure(int code, const std::string& msg) : std::runtime_error(msg), code(code) {}
  int code;
};

void must(gempe_ctx* c, int rc) {
  if (rc != GEMPE_OK) throw group_failure(rc, gempe_last_error(c));
}

template <typename Fn>
int guarded(gempe_group* g, Fn&& fn) {
  try {
    fn();
    return GEMPE_OK;
  } catch (const group_failure& e) {
    (g ? g->error : g_group_create_error) = e.what();
    return e.code;
  } catch (const config_error& e) {
    (g ? g->error : g_group_create_error) = e.what();
    return GEMPE_ERR_CONFIG;
  } catch (const cuda_error& e) {
    (g ? g->error : g_group_create_error) = e.what();
    return GEMPE_ERR_CUDA;
  } catch (const std::exception& e) {
    (g ? g->error : g_group_create_error) = e.what();
    return GEMPE_ERR_DATA;
  }
}

int world(const gempe_group* g) { return static_cast<int>(g->ctx.size()); }

void on(gempe_group* g, int r) { cuda_check(cudaSetDevice(g->device[r]), "cudaSetDevice"); }

// every pair of distinct devices can address each other's memory
bool enable_peer_access(const std::vector<int>& devices) {
  for (int a : devices) {
    for (int b : devices) {
      if (a == b) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) return false;
    }
  }
  for (int a : devices) {
    cuda_check(cudaSetDevice(a), "cudaSetDevice");
    for (int b : devices) {
      if (a == b) continue;
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else cuda_check(e, "cudaDeviceEnablePeerAccess");
    }
  }
  return true;
}

// (re)registers every rank's coordinate buffers and receive areas with every other rank (after creation and after a
// relabel, which reallocates the exchange buffers)
void connect(gempe_group* g) {
  const int w = world(g);
  for (int r = 0; r < w; ++r) must(g->ctx[r], gempe_clear_peers(g->ctx[r]));
  if (!g->peer_stores) return;
  for (int r = 0; r < w; ++r) {
    for (int q = 0; q < w; ++q) {
      if (q == r) continue;
      must(g->ctx[r], gempe_add_peer_pointers(g->ctx[r], gempe_device_coords_parity(g->ctx[q], 0),
                                              gempe_device_coords_parity(g->ctx[q], 1)));
      must(g->ctx[r], gempe_add_peer_exchange_pointer(g->ctx[r], q, gempe_exchange_recv_area(g->ctx[q])));
    }
  }
}

void wait_all(gempe_group* g, int r, const std::vector<cudaEvent_t>& events, bool include_self) {
  for (int q = 0; q < world(g); ++q) {
    if (q == r && !include_self) continue;
    cuda_check(cudaStreamWaitEvent(g->ctx[r]->stream, events[q], 0), "cudaStreamWaitEvent");
  }
}

// copy-engine all-to-all of the packed sample records (no peer access): region d / count d of rank r -> region r / count r
// of rank d
void exchange_records_by_copy(gempe_group* g) {
  const int w = world(g);
  struct Layout {
    void *send, *recv;
    std::uint32_t *send_count, *recv_count, capacity;
  };
  std::vector<Layout> lay(w);
  for (int r = 0; r < w; ++r) {
    must(g->ctx[r], gempe_exchange_layout(g->ctx[r], &lay[r].send, &lay[r].recv, &lay[r].send_count, &lay[r].recv_count,
                                          &lay[r].capacity));
  }
  for (int r = 0; r < w; ++r) {
    on(g, r);
    cudaStream_t s = g->ctx[r]->stream;
    // the destinations have bucketed what the previous round left in their receive areas
    wait_all(g, r, g->bucketed, false);
    const std::size_t bytes = static_cast<std::size_t>(lay[r].capacity) * sizeof(uint2);
    for (int d = 0; d < w; ++d) {
      cuda_check(cudaMemcpyPeerAsync(static_cast<char*>(lay[d].recv) + r * bytes, g->device[d],
                                     static_cast<char*>(lay[r].send) + d * bytes, g->device[r], bytes, s), "records");
      cuda_check(cudaMemcpyPeerAsync(lay[d].recv_count + r, g->device[d], lay[r].send_count + d, g->device[r],
                                     sizeof(std::uint32_t), s), "record counts");
    }
  }
}

// copy-engine all-gather of the rows every rank has just updated (no peer access); comm_chunks is 1: rank r owns rows
// [r * block_rows, (r + 1) * block_rows) of the padded coordinate matrix
void broadcast_rows_by_copy(gempe_group* g) {
  const int w = world(g);
  for (int r = 0; r < w; ++r) {
    on(g, r);
    gempe_ctx* c = g->ctx[r];
    const std::size_t block = static_cast<std::size_t>(c->block_rows) * c->ld;
    const float* mine = c->x[c->cur ^ 1].get() + r * block;
    for (int q = 0; q < w; ++q) {
      if (q == r) continue;
      float* theirs = g->ctx[q]->x[g->ctx[q]->cur ^ 1].get() + r * block;
      cuda_check(cudaMemcpyPeerAsync(theirs, g->device[q], mine, g->device[r], block * sizeof(float), c->stream), "rows");
    }
  }
}

// One sharded round on every rank's stream.  auto_sigma: the round reads sigma from each rank's device state.
void enqueue_round(gempe_group* g, bool auto_sigma, double mu, double sigma, std::uint64_t iter) {
  const int w = world(g);
  for (int r = 0; r < w; ++r) {
    on(g, r);
    if (auto_sigma) wait_all(g, r, g->summed, false);  // nobody still reads this rank's tallies of the previous round
    must(g->ctx[r], auto_sigma ? gempe_begin_round_auto(g->ctx[r], iter) : gempe_begin_round(g->ctx[r], mu, sigma, iter));
    if (g->peer_stores) cuda_check(cudaEventRecord(g->packed[r], g->ctx[r]->stream), "event");
  }
  if (!g->peer_stores) {
    exchange_records_by_copy(g);
    for (int r = 0; r < w; ++r) {
      on(g, r);
      cuda_check(cudaEventRecord(g->packed[r], g->ctx[r]->stream), "event");
    }
  }
  for (int r = 0; r < w; ++r) {
    on(g, r);
    // the barrier of the round: all records have arrived, and every rank has left the previous round's gather (it read
    // the buffer this round writes, and wrote the one this round reads)
    wait_all(g, r, g->packed, false);
    if (!g->peer_stores) wait_all(g, r, g->gathered, false);  // the row copies ride on the gathering rank's stream
    must(g->ctx[r], gempe_bucket_received(g->ctx[r]));
    cuda_check(cudaEventRecord(g->bucketed[r], g->ctx[r]->stream), "event");
    must(g->ctx[r], gempe_gather_chunk(g->ctx[r], 0));
  }
  if (!g->peer_stores) broadcast_rows_by_copy(g);
  for (int r = 0; r < w; ++r) {
    on(g, r);
    cuda_check(cudaEventRecord(g->gathered[r], g->ctx[r]->stream), "event");
    must(g->ctx[r], gempe_end_round(g->ctx[r]));
  }
}

// waits for every rank, raises a failed round's error on behalf of the whole group, returns the job-wide tallies
void finish_round(gempe_group* g, std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  const int w = world(g);
  std::vector<std::uint64_t> he(kBins), hn(kBins), sum_e(kBins, 0), sum_n(kBins, 0);
  int first_rc = GEMPE_OK;
  std::string first_msg;
  for (int r = 0; r < w; ++r) {  // every rank is drained before anything is thrown: no rank is left mid-round
    const int rc = gempe_sync(g->ctx[r], he.data(), hn.data());
    if (rc != GEMPE_OK && first_rc == GEMPE_OK) {
      first_rc = rc;
      first_msg = gempe_last_error(g->ctx[r]);
    }
    for (int b = 0; b < kBins; ++b) {
      sum_e[b] += he[b];
      sum_n[b] += hn[b];
    }
  }
  if (first_rc != GEMPE_OK) throw group_failure(first_rc, first_msg);
  if (hist_edge) std::copy(sum_e.begin(), sum_e.end(), hist_edge);
  if (hist_nonedge) std::copy(sum_n.begin(), sum_n.end(), hist_nonedge);
}

}  // namespace

extern "C" {

int gempe_group_create(gempe_group** out, std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                       const std::uint32_t* dst, const gempe_options* opt, const int* devices, int n_devices, int flags) {
  if (!out || !opt || !devices) {
    g_group_create_error = "null argument";
    return GEMPE_ERR_CONFIG;
  }
  *out = nullptr;
  std::unique_ptr<gempe_group> g;
  const int rc = guarded(nullptr, [&] {
    if (n_devices < 1 || n_devices > kMaxPeers + 1) throw config_error("a group has 1 .. 16 ranks");
    int present = 0;
    if (cudaGetDeviceCount(&present) != cudaSuccess || present == 0) {
      throw cuda_error("no CUDA device available: the GEMPE path has no CPU fallback");
    }
    for (int r = 0; r < n_devices; ++r) {
      if (devices[r] < 0 || devices[r] >= present) throw config_error("device ordinal out of range");
    }
    g = std::make_unique<gempe_group>();
    g->device.assign(devices, devices + n_devices);
    g->ctx.assign(n_devices, nullptr);
    g->n = n;
    g->m = m;
    g->dim = opt->dim;
    std::vector<int> distinct(g->device);
    std::sort(distinct.begin(), distinct.end());
    distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
    g->peer_stores = !(flags & GEMPE_GROUP_COPY_ENGINES) && enable_peer_access(distinct);
    // one context per rank, built concurrently (construction is host work + launches on the rank's own device)
    std::vector<int> codes(n_devices, GEMPE_OK);
    std::vector<std::string> messages(n_devices);
    std::vector<std::thread> builders;
    for (int r = 0; r < n_devices; ++r) {
      builders.emplace_back([&, r] {
        gempe_options o = *opt;
        o.device = devices[r];
        o.rank = r;
        o.world = n_devices;
        o.comm_chunks = 1;                   // nothing to pipeline: the rows travel while the kernel runs
        o.exchange = n_devices > 1 ? 1 : 0;  // sample only the own anchors, records go to the partners' owners
        codes[r] = gempe_create(&g->ctx[r], n, m, src, dst, &o);
        if (codes[r] != GEMPE_OK) messages[r] = gempe_last_error(nullptr);
      });
    }
    for (auto& t : builders) t.join();
    for (int r = 0; r < n_devices; ++r) {
      if (codes[r] != GEMPE_OK) throw group_failure(codes[r], messages[r]);
    }
    for (auto* list : {&g->packed, &g->bucketed, &g->gathered, &g->summed}) list->assign(n_devices, nullptr);
    g->total = std::vector<DeviceBuffer<unsigned long long>>(n_devices);
    for (int r = 0; r < n_devices; ++r) {
      on(g.get(), r);
      for (auto* list : {&g->packed, &g->bucketed, &g->gathered, &g->summed}) {
        cuda_check(cudaEventCreateWithFlags(&(*list)[r], cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord((*list)[r], g->ctx[r]->stream), "event");  // waitable from the first round on
      }
      g->total[r].allocate(2 * kBins, true);
    }
    if (!g->ctx[0]->degenerate && n_devices > 1) connect(g.get());
  });
  if (rc != GEMPE_OK) return rc;
  *out = g.release();
  return GEMPE_OK;
}

void gempe_group_destroy(gempe_group* g) { delete g; }
const char* gempe_group_last_error(const gempe_group* g) { return g ? g->error.c_str() : g_group_create_error.c_str(); }
int gempe_group_world(const gempe_group* g) { return world(g); }
gempe_ctx* gempe_group_context(gempe_group* g, int rank) {
  return rank >= 0 && rank < world(g) ? g->ctx[rank] : nullptr;
}
const char* gempe_group_exchange_path(const gempe_group* g) {
  if (world(g) == 1) return "single rank";
  return g->peer_stores ? "peer stores from the pack and gather kernels" : "copy engines (cudaMemcpyPeerAsync)";
}

int gempe_group_set_coords(gempe_group* g, const float* x_work) {
  return guarded(g, [&] {
    for (gempe_ctx* c : g->ctx) must(c, gempe_set_coords(c, x_work));
  });
}

int gempe_group_init_coords(gempe_group* g, int rule, std::uint64_t seed, double stddev) {
  return guarded(g, [&] {
    for (gempe_ctx* c : g->ctx) must(c, gempe_init_coords(c, rule, seed, stddev));
  });
}

int gempe_group_get_coords(gempe_group* g, float* x_work) {
  return guarded(g, [&] {
    for (gempe_ctx* c : g->ctx) cuda_check(cudaStreamSynchronize(c->stream), "group sync");  // peers' stores included
    must(g->ctx[0], gempe_get_coords(g->ctx[0], x_work));
  });
}

int gempe_group_iterate(gempe_group* g, double mu, double sigma, std::uint64_t iter_index, std::uint64_t* hist_edge,
                        std::uint64_t* hist_nonedge) {
  return guarded(g, [&] {
    if (world(g) == 1) {
      must(g->ctx[0], gempe_iterate(g->ctx[0], mu, sigma, iter_index, hist_edge, hist_nonedge));
      return;
    }
    enqueue_round(g, false, mu, sigma, iter_index);
    finish_round(g, hist_edge, hist_nonedge);
  });
}

int gempe_group_set_sigma(gempe_group* g, double mu, double sigma) {
  return guarded(g, [&] {
    for (gempe_ctx* c : g->ctx) must(c, gempe_set_sigma(c, mu, sigma));
    g->mu = mu;
    g->sigma_seeded = true;
  });
}

int gempe_group_iterate_auto(gempe_group* g, std::uint64_t iter_index, double* sigma, double* pe_estimate,
                             double* nonedge_weight, std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  return guarded(g, [&] {
    if (!g->sigma_seeded) throw config_error("gempe_group_set_sigma first");
    const int w = world(g);
    if (w == 1) {
      must(g->ctx[0], gempe_iterate_auto(g->ctx[0], iter_index, sigma, pe_estimate, nonedge_weight, hist_edge, hist_nonedge));
      return;
    }
    enqueue_round(g, true, 0.0, 0.0, iter_index);
    if (g->peer_stores) {
      // every rank sums all ranks' tallies on its own device and runs the same sigma search: no host round trip
      TallySources srcs{};
      srcs.count = w;
      for (int q = 0; q < w; ++q) srcs.hist[q] = g->ctx[q]->hist.get();
      const double pairs = static_cast<double>(static_cast<std::uint64_t>(g->n) * (g->n - 1) / 2);
      for (int r = 0; r < w; ++r) {
        on(g, r);
        gempe_ctx* c = g->ctx[r];
        wait_all(g, r, g->gathered, false);
        c->launches += launch_sum_tallies(srcs, g->total[r].get(), c->stream);
        cuda_check(cudaEventRecord(g->summed[r], c->stream), "event");
        c->launches += launch_sigma_update(g->total[r].get(), g->mu, pairs, static_cast<double>(g->m),
                                           c->opt.math == GEMPE_MATH_EXACT, c->sigma_state.get(), c->status.get(),
                                           c->sigma_single_block, nullptr, nullptr, nullptr, c->stream);
        cuda_check(cudaGetLastError(), "group sigma update");
      }
      finish_round(g, hist_edge, hist_nonedge);
    } else {
      // no peer access: the tallies meet on the host, every rank gets the sum back and searches on its device
      std::vector<std::uint64_t> he(kBins), hn(kBins);
      finish_round(g, he.data(), hn.data());
      const double pairs = static_cast<double>(static_cast<std::uint64_t>(g->n) * (g->n - 1) / 2);
      for (int r = 0; r < w; ++r) {
        on(g, r);
        gempe_ctx* c = g->ctx[r];
        cuda_check(cudaMemcpyAsync(g->total[r].get(), he.data(), kBins * sizeof(std::uint64_t), cudaMemcpyHostToDevice, c->stream), "tallies");
        cuda_check(cudaMemcpyAsync(g->total[r].get() + kBins, hn.data(), kBins * sizeof(std::uint64_t), cudaMemcpyHostToDevice, c->stream), "tallies");
        c->launches += launch_sigma_update(g->total[r].get(), g->mu, pairs, static_cast<double>(g->m),
                                           c->opt.math == GEMPE_MATH_EXACT, c->sigma_state.get(), c->status.get(),
                                           c->sigma_single_block, nullptr, nullptr, nullptr, c->stream);
        cuda_check(cudaEventRecord(g->summed[r], c->stream), "event");
        cuda_check(cudaStreamSynchronize(c->stream), "group sigma update");
      }
      if (hist_edge) std::copy(he.begin(), he.end(), hist_edge);
      if (hist_nonedge) std::copy(hn.begin(), hn.end(), hist_nonedge);
    }
    must(g->ctx[0], gempe_get_sigma_state(g->ctx[0], sigma, pe_estimate, nonedge_weight));
  });
}

int gempe_group_relabel(gempe_group* g, std::uint64_t relabel_seed) {
  return guarded(g, [&] {
    for (gempe_ctx* c : g->ctx) cuda_check(cudaStreamSynchronize(c->stream), "group sync");
    for (gempe_ctx* c : g->ctx) must(c, gempe_relabel(c, relabel_seed));
    if (world(g) > 1) connect(g);
  });
}

int gempe_group_replicas_agree(gempe_group* g) {
  // 1 when every rank holds bit-identical coordinates, 0 otherwise, negative on error (test / start-up check)
  std::vector<std::vector<float>> x(world(g));
  const int rc = guarded(g, [&] {
    for (gempe_ctx* c : g->ctx) cuda_check(cudaStreamSynchronize(c->stream), "group sync");
    for (int r = 0; r < world(g); ++r) {
      x[r].resize(static_cast<std::size_t>(g->n) * g->dim);
      must(g->ctx[r], gempe_get_coords(g->ctx[r], x[r].data()));
    }
  });
  if (rc != GEMPE_OK) return -rc;
  for (int r = 1; r < world(g); ++r) {
    if (std::memcmp(x[0].data(), x[r].data(), x[0].size() * sizeof(float)) != 0) return 0;
  }
  return 1;
}

}  // extern "C"
