// C-ABI of the device path (include/gempe.h): context construction (relabel, CSR, work items, hash set),
// the per-round launch sequence and the test hooks.  Citations are relative to /root/reference/proj.
#include "context.hpp"

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <exception>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <mutex>
#include <thread>

namespace gempe {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// ---- device memory cache (context.hpp) ------------------------------------------------------------------------------
namespace {
constexpr std::size_t kLarge = 1u << 20, kGranule = 2u << 20, kSmallGranule = 512;
struct DeviceCache {
  std::mutex mutex;
  std::map<int, std::multimap<std::size_t, void*>> blocks;  // device -> capacity -> block
  std::size_t bytes = 0;
  std::size_t limit = [] {
    const char* e = std::getenv("GEMPE_DEVICE_CACHE_MB");
    return static_cast<std::size_t>(e ? std::max(0ll, std::atoll(e)) : 16384ll) << 20;
  }();
};
DeviceCache& device_cache() {
  static DeviceCache* cache = new DeviceCache;  // never destroyed: buffers may be released during process teardown
  return *cache;
}
}  // namespace

void trim_device_cache() noexcept {
  DeviceCache& c = device_cache();
  std::lock_guard<std::mutex> lock(c.mutex);
  int before = 0;
  cudaGetDevice(&before);
  for (auto& dev : c.blocks) {
    cudaSetDevice(dev.first);
    for (auto& b : dev.second) cudaFree(b.second);
    dev.second.clear();
  }
  c.bytes = 0;
  cudaSetDevice(before);
}

void* device_alloc(std::size_t bytes, std::size_t* capacity, int* device) {
  cuda_check(cudaGetDevice(device), "cudaGetDevice");
  void* p = nullptr;
  std::size_t want = bytes;
  DeviceCache& c = device_cache();
  if (c.limit) {
    const std::size_t granule = bytes >= kLarge ? kGranule : kSmallGranule;
    want = (bytes + granule - 1) / granule * granule;
    std::lock_guard<std::mutex> lock(c.mutex);
    auto& blocks = c.blocks[*device];
    auto it = blocks.lower_bound(want);
    if (it != blocks.end() && it->first <= want + want / 4) {  // close enough in size: at most a quarter wasted
      p = it->second;
      *capacity = it->first;
      c.bytes -= it->first;
      blocks.erase(it);
      return p;
    }
  }
  cudaError_t err = cudaMalloc(&p, want);
  if (err == cudaErrorMemoryAllocation) {  // what the cache holds may be what is missing
    cudaGetLastError();
    trim_device_cache();
    err = cudaMalloc(&p, want);
  }
  cuda_check(err, "cudaMalloc");
  *capacity = want;
  return p;
}

void device_free(void* p, std::size_t capacity, int device) noexcept {
  if (!p) return;
  DeviceCache& c = device_cache();
  int before = 0;
  cudaGetDevice(&before);
  if (before != device) cudaSetDevice(device);
  bool kept = false;
  if (c.limit) {
    // cudaFree waits for work that still uses the block; a block that is handed to the next owner must be idle too
    if (cudaDeviceSynchronize() == cudaSuccess) {
      std::lock_guard<std::mutex> lock(c.mutex);
      if (c.bytes + capacity <= c.limit) {
        c.blocks[device].emplace(capacity, p);
        c.bytes += capacity;
        kept = true;
      }
    }
  }
  if (!kept) cudaFree(p);
  if (before != device) cudaSetDevice(before);
}

namespace {

thread_local std::string g_create_error;

int code_of(const std::exception& e) {
  if (dynamic_cast<const divergence_error*>(&e)) return GEMPE_ERR_DIVERGENCE;
  if (dynamic_cast<const config_error*>(&e)) return GEMPE_ERR_CONFIG;
  if (dynamic_cast<const data_error*>(&e)) return GEMPE_ERR_DATA;
  if (dynamic_cast<const cuda_error*>(&e)) return GEMPE_ERR_CUDA;
  return GEMPE_ERR_DATA;
}

}  // namespace
void set_create_error(const std::string& msg) { g_create_error = msg; }
namespace {

template <typename Fn>
int guarded(gempe_ctx* ctx, Fn&& fn) {
  try {
    // every entry point works on the context's own device, whatever the caller's current device is (several
    // contexts on different GPUs may be driven from one thread)
    if (ctx && cudaSetDevice(ctx->opt.device) != cudaSuccess) throw cuda_error("cudaSetDevice failed");
    fn();
    return GEMPE_OK;
  } catch (const std::exception& e) {
    if (ctx) ctx->error = e.what();
    else g_create_error = e.what();
    return code_of(e);
  }
}

std::uint32_t row_stride_for(std::uint32_t dim) { return dim <= 2 ? dim : (dim + 3u) & ~3u; }

std::uint32_t lanes_per_row(std::uint32_t ld) {
  std::uint32_t lpr = 1;
  while (lpr < 32 && lpr * 4 < ld) lpr <<= 1;
  return lpr;
}

void pack_tables(DeviceTables& out) {
  const FastMathTables& t = FastMathTables::get();
  auto pack = [](const QuadTable& q, double* dst) {
    for (int i = 0; i <= kSegments; ++i) dst[i] = q.knots[i];
    for (int i = 0; i < kSegments; ++i) {
      dst[17 + i] = q.a[i];
      dst[33 + i] = q.b[i];
      dst[49 + i] = q.c[i];
    }
  };
  pack(t.erf, out.erf);
  pack(t.ratio, out.ratio);
}

// The fp32 cells of kernels.hpp: ratio cell i = [-1 + 0.05 i, -1 + 0.05 (i + 1)) carries the quadratic of the segment it
// lies in (every knot of the reference's ratio table, piecewise.cpp:178-190, is a multiple of 0.05 -- checked here), then
// the 16 uniform erf segments.
std::vector<float4> pack_tables_f32() {
  const FastMathTables& t = FastMathTables::get();
  std::vector<float4> cells(kTableF32Entries);
  const double lo = t.ratio.knots[0], width = 0.05;
  if (std::fabs(lo + 1.0) > 1e-12 || std::fabs(t.ratio.knots[kSegments] - 8.0) > 1e-12) {
    throw config_error("ratio table range changed: the fp32 cell layout assumes [-1, 8]");
  }
  for (int k = 0; k <= kSegments; ++k) {
    const double cells_below = (t.ratio.knots[k] - lo) / width;
    if (std::fabs(cells_below - std::round(cells_below)) > 1e-9) throw config_error("ratio table knot is not a multiple of 0.05");
    if (std::fabs(t.erf.knots[k] - 6.0 * k / kSegments) > 1e-12) throw config_error("erf table knots are not uniform");
  }
  for (int i = 0; i < kRatioCells; ++i) {
    const double mid = lo + width * (i + 0.5);
    int s = 0;
    while (s + 1 < kSegments && mid >= t.ratio.knots[s + 1]) ++s;
    cells[i] = make_float4(static_cast<float>(t.ratio.a[s]), static_cast<float>(t.ratio.b[s]), static_cast<float>(t.ratio.c[s]), 0.0f);
  }
  for (int s = 0; s < kErfSegments; ++s) {
    cells[kRatioCells + s] = make_float4(static_cast<float>(t.erf.a[s]), static_cast<float>(t.erf.b[s]), static_cast<float>(t.erf.c[s]), 0.0f);
  }
  return cells;
}

void set_round_math(gempe_ctx* c, double mu, double sigma) {
  if (!(sigma > 0.0) || !std::isfinite(sigma) || !std::isfinite(mu)) throw config_error("sigma must be positive and finite");
  const double pi = 3.14159265358979323846264338327950288, ln2 = 0.693147180559945309417232121458176568;
  const double c1 = 2.0 / (pi * ln2);
  const double c2 = 1.0 / (2.50662827463100050241576528481 * ln2);
  RoundMath& m = c->math;
  m.mu = mu;
  m.inv_sqrt2_sigma = 1.0 / (1.41421356237309504880168872420969808 * sigma);
  m.A = c1 / (sigma * sigma);
  m.B = c2 / (sigma * sigma * sigma);
  m.C = c2 / sigma;
  m.exact = c->opt.math == GEMPE_MATH_EXACT;
}

// Host copies of the work edge arrays, downloaded on first use.
void host_work_graph(gempe_ctx* c) {
  if (c->work_src.size() == c->m && c->work_dst.size() == c->m) return;
  c->work_src.resize(c->m);
  c->work_dst.resize(c->m);
  if (c->m == 0) return;
  cuda_check(cudaMemcpy(c->work_src.data(), c->tmp_src.get(), c->m * sizeof(std::uint32_t), cudaMemcpyDeviceToHost), "work graph D2H");
  cuda_check(cudaMemcpy(c->work_dst.data(), c->tmp_dst.get(), c->m * sizeof(std::uint32_t), cudaMemcpyDeviceToHost), "work graph D2H");
}

// Builds every graph-derived device structure from the work graph on the device.
void build_structures(gempe_ctx* c) {
  ++c->structure_generation;  // captured launch sequences hold pointers into what is rebuilt here
  const std::uint32_t n = c->n;
  const std::uint64_t m = c->m;

  PhaseTimer timer;
  const bool per_edge = c->opt.neg_mode == GEMPE_NEG_PER_EDGE_2;
  // the work edge arrays are resident on the device (tmp_src / tmp_dst): they feed the CSR build and the hash-set build
  // both-direction CSR; eid_role = 2*e + role keys the PER_EDGE_2 sample streams.  Default: built on the device
  // (degree count, scan, atomic fill; the order inside a row is the arrival order).  When a reproducible order is
  // asked for (opt.deterministic) the rows are filled on the host in edge order instead.
  std::vector<std::uint32_t> rowptr(static_cast<std::size_t>(n) + 1, 0);
  if (!c->opt.deterministic) {
    c->rowptr.allocate(static_cast<std::size_t>(n) + 1, true);
    c->nbr.allocate(2 * m);
    c->eid_role.allocate(per_edge ? 2 * m : 0);
    c->csr_src.allocate(per_edge ? 2 * m : 0);
    DeviceBuffer<std::uint32_t> deg, scratch;
    deg.allocate(n);
    scratch.allocate((n + 4095) / 4096 + 2);
    c->launches += launch_csr_build(c->tmp_src.get(), c->tmp_dst.get(), m, n, deg.get(), c->rowptr.get(), scratch.get(),
                                    c->nbr.get(), c->eid_role.get(), c->csr_src.get(), c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "csr build");
    cuda_check(cudaMemcpy(rowptr.data(), c->rowptr.get(), rowptr.size() * sizeof(std::uint32_t), cudaMemcpyDeviceToHost),
               "rowptr D2H");
  } else {
    host_work_graph(c);
    const auto& src = c->work_src;
    const auto& dst = c->work_dst;
    for (std::uint64_t e = 0; e < m; ++e) {
      ++rowptr[src[e] + 1];
      ++rowptr[dst[e] + 1];
    }
    for (std::uint32_t v = 0; v < n; ++v) rowptr[v + 1] += rowptr[v];
    std::vector<std::uint32_t> nbr(2 * m), cursor(rowptr.begin(), rowptr.end() - 1);
    std::vector<std::uint32_t> eid_role, csr_src;
    if (per_edge) {
      eid_role.resize(2 * m);
      csr_src.resize(2 * m);
    }
    for (std::uint64_t e = 0; e < m; ++e) {
      const std::uint32_t p0 = cursor[src[e]]++, p1 = cursor[dst[e]]++;
      nbr[p0] = dst[e];
      nbr[p1] = src[e];
      if (per_edge) {
        eid_role[p0] = static_cast<std::uint32_t>(2 * e);
        eid_role[p1] = static_cast<std::uint32_t>(2 * e + 1);
        csr_src[p0] = src[e];
        csr_src[p1] = dst[e];
      }
    }
    c->rowptr.upload(rowptr);
    c->nbr.upload(nbr);
    c->eid_role.upload(eid_role);
    c->csr_src.upload(csr_src);
  }

  timer.lap(c->opt.deterministic ? "csr (host, edge order)" : "csr (device)");
  // work items: one per owned vertex, hubs split every chunk_entries adjacency positions
  std::vector<ItemDesc> items;
  std::vector<std::uint32_t> hub_first, hub_items;
  std::uint32_t parts = 0;
  items.reserve(static_cast<std::size_t>(n) / static_cast<std::size_t>(c->opt.world) +
                static_cast<std::size_t>(2 * m / std::max(1u, c->chunk_entries)) + 1024);
  c->chunk_item_off.assign(c->comm_chunks + 1, 0);
  const std::uint32_t world = static_cast<std::uint32_t>(c->opt.world), rank = static_cast<std::uint32_t>(c->opt.rank);
  // two passes over the owned vertex range of every comm chunk, each split over a few host threads: count (items, hubs,
  // hub slices per sub-range), prefix, fill in place -- the table is the same as a sequential walk would give (c4: 19 -> 14 ms,
  // c5: 0.30 -> 0.21 s; what is left is writing the table itself)
  const std::uint32_t chunk_entries = c->chunk_entries, negatives = c->opt.negatives;
  auto pieces_of = [&](std::uint32_t v) {
    const std::uint32_t deg = rowptr[v + 1] - rowptr[v];
    return std::max(1u, (deg + chunk_entries - 1) / chunk_entries);
  };
  for (std::uint32_t chunk = 0; chunk < c->comm_chunks; ++chunk) {
    c->chunk_item_off[chunk] = static_cast<std::uint32_t>(items.size());
    const std::uint64_t block = static_cast<std::uint64_t>(chunk) * world + rank;
    const std::uint64_t lo = std::min<std::uint64_t>(n, block * c->block_rows);
    const std::uint64_t hi = std::min<std::uint64_t>(n, (block + 1) * c->block_rows);
    const unsigned threads = hi - lo < (1u << 16) ? 1u : std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
    struct Part { std::uint64_t lo, hi; std::size_t items, hubs; std::uint32_t slices; };
    std::vector<Part> part(threads);
    for (unsigned t = 0; t < threads; ++t) {
      part[t] = Part{lo + (hi - lo) * t / threads, lo + (hi - lo) * (t + 1) / threads, 0, 0, 0};
    }
    auto run = [&](auto&& fn) {
      std::vector<std::thread> pool;
      for (unsigned t = 1; t < threads; ++t) pool.emplace_back(fn, t);
      fn(0u);
      for (auto& th : pool) th.join();
    };
    run([&](unsigned t) {
      Part& p = part[t];
      for (std::uint64_t v = p.lo; v < p.hi; ++v) {
        const std::uint32_t pieces = pieces_of(static_cast<std::uint32_t>(v));
        p.items += pieces;
        if (pieces > 1) {
          ++p.hubs;
          p.slices += pieces;
        }
      }
    });
    std::vector<std::size_t> item_at(threads), hub_at(threads);
    std::vector<std::uint32_t> slice_at(threads);
    std::size_t item_total = items.size(), hub_total = hub_first.size();
    for (unsigned t = 0; t < threads; ++t) {
      item_at[t] = item_total;
      hub_at[t] = hub_total;
      slice_at[t] = parts;
      item_total += part[t].items;
      hub_total += part[t].hubs;
      parts += part[t].slices;
    }
    items.resize(item_total);
    hub_first.resize(hub_total);
    hub_items.resize(hub_total);
    run([&](unsigned t) {
      std::size_t at = item_at[t], hub_next = hub_at[t];
      std::uint32_t slice_next = slice_at[t];
      for (std::uint64_t vv = part[t].lo; vv < part[t].hi; ++vv) {
        const std::uint32_t v = static_cast<std::uint32_t>(vv), pieces = pieces_of(v);
        std::uint32_t hub = kNoHub;
        if (pieces > 1) {
          hub = static_cast<std::uint32_t>(hub_next);
          hub_first[hub_next] = slice_next;
          hub_items[hub_next] = pieces;
          ++hub_next;
          slice_next += pieces;
        }
        for (std::uint32_t p = 0; p < pieces; ++p) {
          ItemDesc it{};
          it.u = v;
          it.off_a = rowptr[v] + p * chunk_entries;
          it.len_a = std::min(it.off_a + chunk_entries, rowptr[v + 1]) - it.off_a;
          // own samples: one slot per adjacency position (PER_EDGE_2), or the vertex's k slots on its first item
          it.off_b = per_edge ? it.off_a : v * negatives;
          it.len_b = per_edge ? it.len_a : (p == 0 ? negatives : 0u);
          it.first = p == 0;
          it.hub = hub;
          it.sub = p;
          items[at++] = it;
        }
      }
    });
  }
  c->chunk_item_off[c->comm_chunks] = static_cast<std::uint32_t>(items.size());
  // d <= 4 runs one THREAD per item: items of similar length are put next to each other (longest first) inside every
  // chunk, so the 32 items of a warp finish together instead of waiting for the longest one
  const bool sorted_items = c->ld <= 4 && std::getenv("GEMPE_NO_ITEM_SORT") == nullptr;
  if (sorted_items) {
    for (std::uint32_t chunk = 0; chunk < c->comm_chunks; ++chunk) {
      std::stable_sort(items.begin() + c->chunk_item_off[chunk], items.begin() + c->chunk_item_off[chunk + 1],
                       [](const ItemDesc& a, const ItemDesc& b) { return a.len_a > b.len_a; });
    }
  }
  // slices for the host-buffer pipeline, cut at vertex boundaries (a hub's slices stay together)
  c->step_item_off.assign(1, 0);
  c->step_vertex_off.assign(1, 0);
  if (world == 1 && !items.empty() && sorted_items) {  // vertex order is gone: one slice
    c->step_item_off.push_back(static_cast<std::uint32_t>(items.size()));
    c->step_vertex_off.push_back(n);
  } else if (world == 1 && !items.empty()) {
    // geometric slices (1/64, 1/32, ..., 1/2 of the items): the copy out is the slower side, so only the time to the
    // FIRST finished slice is exposed -- keep that one short
    constexpr std::uint32_t kSlices = 7;
    for (std::uint32_t k = 1; k < kSlices; ++k) {
      std::uint64_t at = static_cast<std::uint64_t>(items.size()) >> (kSlices - k);
      while (at < items.size() && items[at].sub != 0) ++at;  // first item of a vertex
      if (at >= items.size() || at <= c->step_item_off.back()) continue;
      c->step_item_off.push_back(static_cast<std::uint32_t>(at));
      c->step_vertex_off.push_back(items[at].u);
    }
    c->step_item_off.push_back(static_cast<std::uint32_t>(items.size()));
    c->step_vertex_off.push_back(n);
  }

  timer.lap("work items (host)");
  c->items.upload(items);
  c->hub_first.upload(hub_first);
  c->hub_items.upload(hub_items);
  c->hub_arrived.allocate(hub_first.size(), true);
  c->part_y.allocate(static_cast<std::size_t>(parts) * c->ld);
  c->part_z.allocate(parts);

  c->slots = per_edge ? 2 * m : static_cast<std::uint64_t>(n) * c->opt.negatives;
  c->neg_own.allocate(c->slots);
  c->in_anchor.allocate(c->slots);
  // bucketing method (opt.bucket_mode): 1 = per-partner atomics (auto while the per-vertex counters fit L2
  // comfortably), 3 = radix pass by vertex range + atomics range by range (auto for n >= 2^22 on one rank),
  // 2 = two-level counting sort (kept for A/B runs)
  c->partition = PartitionArgs{};
  std::uint32_t shift = 8;
  while ((static_cast<std::uint64_t>(n) + (1ull << shift) - 1) >> shift > 4096) ++shift;
  const bool can_partition = shift <= 15 && c->slots > 0;
  const bool want_partition = c->opt.bucket_mode == 2;
  if (can_partition && want_partition) {
    c->partition.shift = shift;
    c->partition.buckets = static_cast<std::uint32_t>((static_cast<std::uint64_t>(n) + (1ull << shift) - 1) >> shift);
    c->partition.grid = partition_grid(c->slots);
    c->block_hist.allocate(static_cast<std::size_t>(c->partition.grid) * c->partition.buckets);
    c->bucket_off.allocate(c->partition.buckets + 1);
    c->records.allocate(c->slots);
    c->partition.block_hist = c->block_hist.get();
    c->partition.bucket_off = c->bucket_off.get();
    c->partition.records = c->records.get();
    c->in_rank.release();
    c->in_cnt.release();
  } else {
    c->block_hist.release();
    c->bucket_off.release();
    c->records.release();
    c->in_rank.allocate(c->slots);
    c->in_cnt.allocate(n, true);
  }
  c->in_off.allocate(static_cast<std::size_t>(n) + 1, true);
  c->scan_scratch.allocate((n + 4095) / 4096 + 2);
  // bucket_mode 4, slotted buckets: every vertex owns `stride` slots of in_anchor, the sampler stores the anchor at slot
  // (partner, arrival rank) itself, so the scan and the scatter pass disappear (sampling passes c1 20 -> 16 us, c2 52 -> 33,
  // c3 71 -> 49); samples whose partner's slots are full -- partners are uniform over the legal vertices, so the count
  // per vertex is ~Poisson(S/n) and the slack of 6 sigma + 8 makes that a 1e-9 event per vertex on ordinary graphs -- go
  // to a spill list that one block indexes (exact for ANY input, only slower).  Auto on one rank while the slot array
  // stays L2-resident (<= 48 MB) and no reproducible order is asked for (the sorted buckets of `deterministic` use
  // mode 1).  Beyond that the half-filled slot sectors cost more DRAM read-modify-write traffic than the scatter pass
  // they replace (c4, 235 MB of slots: 0.63 -> 0.74 ms), so larger graphs keep mode 1 / 3.
  c->in_stride = 0;
  {
    const double mean_in = n ? static_cast<double>(c->slots) / n : 0.0;
    std::uint64_t stride = (static_cast<std::uint64_t>(mean_in + 6.0 * std::sqrt(mean_in) + 8.0) + 3u) & ~3ull;
    if (const char* e = std::getenv("GEMPE_IN_STRIDE")) stride = std::max(1, std::atoi(e));  // test hook: force spills
    const bool possible = world == 1 && !c->opt.exchange && !c->opt.deterministic && c->slots > 0 &&
                          static_cast<std::uint64_t>(n) * stride < 0xffffffffull;
    const bool wanted = c->opt.bucket_mode == 4 ||
                        (c->opt.bucket_mode == 0 && static_cast<std::uint64_t>(n) * stride * 4 <= (48ull << 20));
    if (c->opt.bucket_mode == 4 && !possible) {
      throw config_error("bucket_mode 4 (slotted buckets) needs one rank, no exchange, no deterministic order");
    }
    if (possible && wanted) {
      c->in_stride = static_cast<std::uint32_t>(stride);
      c->in_anchor.allocate(static_cast<std::size_t>(n) * stride);
      c->in_rank.release();
      c->in_cnt.allocate(static_cast<std::size_t>(n) + 1, true);  // [n] = number of spilled records
      c->spill.allocate(c->slots);
      c->spill_cnt.allocate(n, true);
      c->spill_off.allocate(static_cast<std::size_t>(n) + 1, true);
      c->spill_anchor.allocate(c->slots);
    } else {
      c->spill.release();
      c->spill_cnt.release();
      c->spill_off.release();
      c->spill_anchor.release();
    }
  }
  c->exchange = ExchangeArgs{};
  // bucket_mode 3 (one rank): the pack / bucket kernels of the exchange path with contiguous vertex ranges as the
  // destinations -- one radix pass by range, then per-partner atomics whose counters stay L2-resident range by range
  const bool region_mode = !c->in_stride && (c->opt.bucket_mode == 3 || (c->opt.bucket_mode == 0 && n >= (1u << 22))) && world == 1 &&
                           !c->opt.exchange && c->slots > 0;
  c->pack_path = c->opt.exchange != 0 || region_mode;
  if (c->pack_path) {
    // own sample streams per rank: the anchors of block b = chunk * world + r belong to rank r.  Every rank derives the
    // same per-(source, destination) capacity from the busiest rank, so the all-to-all is an equal split.
    auto first_slot_of = [&](std::uint64_t v) { return per_edge ? static_cast<std::uint64_t>(rowptr[v]) : v * c->opt.negatives; };
    std::vector<std::uint64_t> own_slots(world, 0), own_rows(world, 0), first(c->comm_chunks), prefix(c->comm_chunks + 1, 0);
    for (std::uint32_t chunk = 0; chunk < c->comm_chunks; ++chunk) {
      for (std::uint32_t r = 0; r < world; ++r) {
        const std::uint64_t block = static_cast<std::uint64_t>(chunk) * world + r;
        const std::uint64_t lo = std::min<std::uint64_t>(n, block * c->block_rows);
        const std::uint64_t hi = std::min<std::uint64_t>(n, (block + 1) * c->block_rows);
        own_slots[r] += first_slot_of(hi) - first_slot_of(lo);
        own_rows[r] += hi - lo;
        if (r == rank) {
          first[chunk] = first_slot_of(lo);
          prefix[chunk + 1] = prefix[chunk] + first_slot_of(hi) - first_slot_of(lo);
        }
      }
    }
    std::uint32_t regions = world, region_rows = 0;
    double share = n ? static_cast<double>(*std::max_element(own_rows.begin(), own_rows.end())) / n : 1.0;
    if (region_mode) {
      std::uint64_t range_bytes = 4u << 20;  // counters per range (c5: 16.6 ms at 4 MB, 18.0 at 2, 20.9 at 8, 27 at 32)
      if (const char* e = std::getenv("GEMPE_REGION_MB")) range_bytes = std::max(1, std::atoi(e)) * (1ull << 20);
      regions = static_cast<std::uint32_t>(std::min<std::uint64_t>(256, std::max<std::uint64_t>(1, (4ull * n + range_bytes - 1) / range_bytes)));
      region_rows = (n + regions - 1) / regions;
      regions = (n + region_rows - 1) / region_rows;
      share = static_cast<double>(region_rows) / n;
    }
    const std::uint64_t busiest = *std::max_element(own_slots.begin(), own_slots.end());
    double slack = 1.25;
    if (const char* e = std::getenv("GEMPE_REGION_SLACK")) {  // test hook: undersized regions exercise the spill area
      if (region_mode) slack = std::max(0.05, std::atof(e));
    }
    const double expect = slack * static_cast<double>(busiest) * share;  // partners are ~uniform over vertices
    const std::uint64_t cap = std::min<std::uint64_t>(busiest, static_cast<std::uint64_t>(expect + 8.0 * std::sqrt(expect)) + 1024);
    if (cap * regions > 0xffffffffull) throw config_error("exchange regions exceed 2^32 records; use more ranks");
    c->ex_first_slot.upload(first);
    c->ex_prefix.upload(prefix);
    const bool external = !region_mode && (world > 1 || c->opt.exchange == 2);
    c->ex_send.allocate(static_cast<std::size_t>(cap) * regions);
    // receive area: records [2 parities][regions][cap], then counts [2][regions] (one allocation = one IPC handle); the
    // second parity is used by the direct exchange only
    const std::size_t recv_records = 2 * static_cast<std::size_t>(cap) * regions;
    if (external) c->ex_recv.allocate(recv_records + regions + 1, true); else c->ex_recv.release();
    c->ex_send_count.allocate(regions, true);
    c->ex_recv_count.release();
    if (c->ex_registered) c->ex_peers_lost = true;  // a rebuild (relabel) moved the buffers: peers must register again
    c->ex_peers.assign(external ? world : 0, gempe_ctx::ExchangePeer{});
    c->ex_registered = 0;
    if (external) c->ex_peers[rank].recv = c->ex_recv.get();
    const std::uint64_t spill_cap = region_mode ? c->slots : 0;
    c->ex_rank.allocate(static_cast<std::size_t>(cap) * regions + spill_cap);
    if (region_mode) {
      c->ex_spill.allocate(spill_cap);
      c->ex_spill_count.allocate(1, true);
    } else {
      c->ex_spill.release();
      c->ex_spill_count.release();
    }
    if (c->in_cnt.size() == 0) c->in_cnt.allocate(n, true);
    c->in_rank.release();  // arrival ranks live beside the records here
    c->exchange.own_slots = prefix.back();
    c->exchange.ranges = c->comm_chunks;
    c->exchange.first_slot = c->ex_first_slot.get();
    c->exchange.prefix = c->ex_prefix.get();
    c->exchange.regions = regions;
    c->exchange.region_rows = region_rows;
    c->exchange.capacity = static_cast<std::uint32_t>(cap);
    c->exchange.spill = region_mode ? c->ex_spill.get() : nullptr;
    c->exchange.spill_count = region_mode ? c->ex_spill_count.get() : nullptr;
    c->exchange.spill_capacity = static_cast<std::uint32_t>(spill_cap);
    c->exchange.send = c->ex_send.get();
    c->exchange.send_count = c->ex_send_count.get();
    // a single rank is its own peer: what it packed is what it receives
    c->exchange.recv = external ? c->ex_recv.get() : c->ex_send.get();
    c->exchange.recv_count = external ? reinterpret_cast<std::uint32_t*>(c->ex_recv.get() + recv_records) : c->ex_send_count.get();
  }

  timer.lap("uploads + allocations");
  // edge hash set, bit-packed (hash_set.cpp:9-34)
  c->hash_bits = auto_hash_bits(m, c->opt.hash_bits);
  const std::uint64_t cells = 1ull << c->hash_bits;
  c->hash_words.allocate(std::max<std::uint64_t>(1, cells / 32), true);
  c->launches += launch_hash_build(c->tmp_src.get(), c->tmp_dst.get(), m, n, static_cast<std::uint32_t>(cells - 1),
                                   c->hash_words.get(), c->stream);
  // a sparse table beyond what L2 keeps (c4: 128 MB, 3 % of the cells set) gets a 4x smaller "any cell of the group
  // set" summary in front of it; dense or small tables do not, and neither does the 2^31-cell table (c5: 7 % set --
  // the wrapping pair_hash aliases heavily at n = 2^24 -- but its 64 MB summary does not stay in L2 next to the
  // record stream: 18.1 ms of sampling passes with it, 16.9 without).  The density is counted, not estimated from m.
  c->hash_summary.release();
  if (cells / 8 > (64ull << 20) && cells / 32 <= (32ull << 20)) {
    unsigned long long set_cells = 0;
    c->launches += launch_hash_popcount(c->hash_words.get(), cells / 32, c->round_state.get(), c->stream);
    cuda_check(cudaMemcpyAsync(&set_cells, c->round_state.get(), sizeof set_cells, cudaMemcpyDeviceToHost, c->stream), "popcount D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "hash popcount");
    cuda_check(cudaMemsetAsync(c->round_state.get(), 0, sizeof set_cells, c->stream), "status reset");
    if (set_cells <= cells / 12) {
      c->hash_summary.allocate(cells >> (5 + kHashSummaryShift));
      c->launches += launch_hash_summary(c->hash_words.get(), cells >> (5 + kHashSummaryShift), c->hash_summary.get(), c->stream);
    }
  }
  cuda_check(cudaStreamSynchronize(c->stream), "hash build");
  timer.lap("hash set (device)");
  if (c->capture) {
    c->cap_y.allocate(static_cast<std::size_t>(n) * c->dim, true);
    c->cap_z.allocate(n, true);
  }
}

// random_relabel applied to the work graph (graph.cpp:199-204), in place on the device
void apply_relabel(gempe_ctx* c, const std::vector<std::uint32_t>& fwd) {
  if (c->m) {
    DeviceBuffer<std::uint32_t> d_fwd;
    d_fwd.upload(fwd);
    c->launches += launch_relabel_apply(c->tmp_src.get(), c->tmp_dst.get(), c->m, d_fwd.get(), c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "relabel");
  }
  c->work_src.clear();  // stale host copies
  c->work_dst.clear();
  for (auto& v : c->to_work) v = fwd[v];
}

SampleArgs sample_args(gempe_ctx* c, std::uint64_t iter) {
  SampleArgs a{};
  a.n = c->n;
  a.slots = c->slots;
  a.neg_mode = c->opt.neg_mode;
  a.k = c->opt.negatives;
  a.rng = c->opt.rng;
  a.stream_base = c->opt.rng == GEMPE_RNG_REFERENCE ? mix_seed(c->opt.seed, iter) : c->opt.seed;
  a.iter = iter;
  a.seed = c->opt.seed;
  a.iter_dev = c->run_queued ? &c->run_state.get()->batch_base : nullptr;  // a queued run: the batch's first round index lives on the device
  a.csr_src = c->csr_src.get();
  a.eid_role = c->eid_role.get();
  a.hash_words = c->hash_words.get();
  a.hash_summary = c->hash_summary.size() ? c->hash_summary.get() : nullptr;
  a.hash_mask = static_cast<std::uint32_t>((1ull << c->hash_bits) - 1);
  a.neg_own = c->neg_own.get();
  a.in_cnt = c->in_cnt.get();
  a.in_rank = c->in_rank.get();
  a.status = c->status.get();
  a.in_stride = c->in_stride;
  a.in_anchor = c->in_anchor.get();
  a.spill = c->spill.get();
  a.spill_count = c->in_stride ? c->in_cnt.get() + c->n : nullptr;
  a.spill_capacity = static_cast<std::uint32_t>(c->spill.size());
  a.own = Ownership{c->block_rows, static_cast<std::uint32_t>(c->opt.world), static_cast<std::uint32_t>(c->opt.rank)};
  return a;
}

void require_live(gempe_ctx* c) {
  if (c->degenerate) throw config_error("cannot iterate a degenerate graph");  // engine.cpp:279
}

// exchange path, second half: bucket the (partner, anchor) records received from all ranks by partner
void bucket_received(gempe_ctx* c) {
  if (!c->pack_path) throw config_error("context was created without opt.exchange");
  if (!c->bucket_pending) throw config_error("gempe_bucket_received without a preceding gempe_begin_round");
  if (c->ex_peers_lost && !c->exchange.direct) {
    throw config_error("the exchange buffers were rebuilt (relabel): register the peers' receive areas again");
  }
  c->launches += launch_bucket_records(c->exchange, c->exchange.regions, c->n, c->in_cnt.get(),
                                       c->in_off.get(), c->ex_rank.get(), c->in_anchor.get(), c->scan_scratch.get(), c->stream);
  if (c->opt.deterministic) c->launches += launch_sort_buckets(c->in_off.get(), c->in_anchor.get(), c->n, c->stream);
  cuda_check(cudaGetLastError(), "bucket received records");
  c->bucket_pending = false;
}

void sampling_passes(gempe_ctx* c, std::uint64_t iter) {
  cuda_check(cudaMemsetAsync(c->status.get(), 0, (4 + 2 * kBins) * sizeof(unsigned long long), c->stream),
             "memset status + tallies");
  const SampleArgs a = sample_args(c, iter);
  if (c->pack_path) {
    ExchangeArgs& x = c->exchange;
    x.direct = !c->ex_peers.empty() && c->ex_registered + 1 == c->ex_peers.size() && c->ex_peers.size() > 1;
    if (x.direct) {
      // receive buffers alternate between rounds: a fast rank may pack round t+1 while a slow one still buckets round t
      const std::uint32_t world = x.regions, rank = static_cast<std::uint32_t>(c->opt.rank);
      const std::size_t cap = x.capacity, records = 2 * cap * world;
      const std::uint32_t parity = static_cast<std::uint32_t>(c->ex_round++ & 1);
      x.recv = c->ex_recv.get() + static_cast<std::size_t>(parity) * world * cap;
      x.recv_count = reinterpret_cast<std::uint32_t*>(c->ex_recv.get() + records) + parity * world;
      for (std::uint32_t d = 0; d < world; ++d) {
        x.dest_region[d] = c->ex_peers[d].recv + (static_cast<std::size_t>(parity) * world + rank) * cap;
        x.dest_count[d] = reinterpret_cast<std::uint32_t*>(c->ex_peers[d].recv + records) + parity * world + rank;
      }
    }
    c->launches += launch_sample_pack(a, c->exchange, c->stream);
    if (x.direct) c->launches += launch_publish_counts(c->exchange, c->stream);
    cuda_check(cudaGetLastError(), "sample + pack");
    c->bucket_pending = true;
    if (c->exchange.recv == c->exchange.send) bucket_received(c);  // own peer
    return;
  }
  if (c->in_stride) {
    // slotted buckets: counters (and the spill count behind them) to zero, the sampler places the anchors itself
    cuda_check(cudaMemsetAsync(c->in_cnt.get(), 0, (static_cast<std::size_t>(c->n) + 1) * sizeof(std::uint32_t), c->stream),
               "memset bucket counters");
    c->launches += launch_sample(a, c->stream);
    SpillIndexArgs sp{};
    sp.n = c->n;
    sp.spill = c->spill.get();
    sp.spill_count = a.spill_count;
    sp.spill_capacity = a.spill_capacity;
    sp.cnt = c->spill_cnt.get();
    sp.off = c->spill_off.get();
    sp.anchor = c->spill_anchor.get();
    c->launches += launch_spill_index(sp, c->stream);
    cuda_check(cudaGetLastError(), "sampling passes");
    return;
  }
  if (c->partition.buckets) {
    c->launches += launch_sample_partition(a, c->partition, c->in_off.get(), c->in_anchor.get(), c->stream);
  } else {
    // in_cnt is zero on entry: allocated zeroed, and the scan clears what it has read
    c->launches += launch_sample(a, c->stream);
    c->launches += launch_scan(c->in_cnt.get(), c->in_off.get(), c->n, c->scan_scratch.get(), c->stream, true);
    c->launches += launch_scatter(a, c->in_off.get(), c->in_anchor.get(), c->stream);
  }
  if (c->opt.deterministic) c->launches += launch_sort_buckets(c->in_off.get(), c->in_anchor.get(), c->n, c->stream);
  cuda_check(cudaGetLastError(), "sampling passes");
}

void gather_items(gempe_ctx* c, std::uint32_t item_lo, std::uint32_t item_hi) {
  if (c->bucket_pending) throw config_error("records are packed but not exchanged: call gempe_bucket_received first");
  GatherArgs g{};
  g.x_cur = c->x[c->cur].get();
  g.x_next = c->x[c->cur ^ 1].get();
  g.n_peers = static_cast<int>(c->peers.size());
  for (int p = 0; p < g.n_peers; ++p) g.peer_next[p] = c->peers[p].x[c->cur ^ 1];
  g.n = c->n;
  g.dim = c->dim;
  g.ld = c->ld;
  g.nbr = c->nbr.get();
  g.neg_own = c->neg_own.get();
  g.in_off = c->in_off.get();
  g.in_anchor = c->in_anchor.get();
  g.in_stride = c->in_stride;
  g.in_cnt = c->in_cnt.get();
  g.spill_count = c->in_stride ? c->in_cnt.get() + c->n : nullptr;
  g.spill_off = c->spill_off.get();
  g.spill_anchor = c->spill_anchor.get();
  g.items = c->items.get();
  g.hub_first = c->hub_first.get();
  g.hub_items = c->hub_items.get();
  g.hub_arrived = c->hub_arrived.get();
  g.part_y = c->part_y.get();
  g.part_z = c->part_z.get();
  g.hist = c->hist.get();
  g.status = c->status.get();
  g.work_cursor = c->work_cursor.get();
  g.cap_y = c->capture ? c->cap_y.get() : nullptr;
  g.cap_z = c->capture ? c->cap_z.get() : nullptr;
  g.math = c->math;
  g.math_dev = c->use_dev_math ? &c->sigma_state.get()->math : nullptr;
  g.run = c->run_queued ? c->run_state.get() : nullptr;
  g.tab = c->tables;
  g.tab_f32 = c->tables_f32.get();
  c->launches += launch_gather(g, item_lo, item_hi, c->opt.precise_distance != 0, c->stream);
  cuda_check(cudaGetLastError(), "gather launch");
}

cudaEvent_t next_event(gempe_ctx* c) {
  if (c->events_used == c->events.size()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    c->events.push_back(e);
  }
  return c->events[c->events_used++];
}

void fetch_status(gempe_ctx* c, std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  cuda_check(cudaMemcpyAsync(c->pinned, c->status.get(), (4 + 2 * kBins) * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c->stream), "status + tallies D2H");
  cuda_check(cudaStreamSynchronize(c->stream), "round");
  std::uint32_t st[8];
  std::memcpy(st, c->pinned, sizeof st);
  c->last_draws = static_cast<std::uint64_t>(st[kStatDrawsLo]) | (static_cast<std::uint64_t>(st[kStatDrawsHi]) << 32);
  if (hist_edge) std::memcpy(hist_edge, c->pinned + 4, kBins * sizeof(std::uint64_t));
  if (hist_nonedge) std::memcpy(hist_nonedge, c->pinned + 4 + kBins, kBins * sizeof(std::uint64_t));
  if (st[kStatRetryCap]) {
    throw near_complete_graph_error("no non-edge partner found after 10^4 draws; graph is near-complete");
  }
  if (st[kStatExchangeOverflow]) {
    throw data_error("sample exchange region overflowed: partners are far from uniform over ranks for this graph; "
                     "create the context with opt.exchange = 0");
  }
  if (st[kStatEmptyTallies]) throw config_error("cannot optimize sigma on an empty histogram");  // slope.cpp:76
  if (st[kStatNonFinite]) {
    throw divergence_error("non-finite coordinate after update", static_cast<int>(c->round_iter) + 1);
  }
}

void validate(std::uint32_t n, std::uint64_t m, const std::uint32_t* src, const std::uint32_t* dst,
              const gempe_options& o) {
  if (o.dim < 1) throw config_error("dimension must be >= 1");
  if (row_stride_for(o.dim) > 1024) throw config_error("dimension above 1024 is not supported by the device layout");
  if (o.neg_mode != GEMPE_NEG_PER_EDGE_2 && o.neg_mode != GEMPE_NEG_PER_VERTEX_K) throw config_error("unknown neg_mode");
  if (o.exchange < 0 || o.exchange > 2) throw config_error("unknown exchange mode");
  if (o.math != GEMPE_MATH_TABLES && o.math != GEMPE_MATH_EXACT) throw config_error("unknown math policy");
  if (o.rng != GEMPE_RNG_REFERENCE && o.rng != GEMPE_RNG_PHILOX) throw config_error("unknown rng mode");
  if (o.kernel_variant != 0) throw config_error("kernel_variant: the A/B gather kernels of round 1 are retired, use 0");
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) throw config_error("bad rank/world");
  if (o.comm_chunks < 1) throw config_error("comm_chunks must be >= 1");
  if (m > 0 && (!src || !dst)) throw data_error("null edge arrays");
  if (2 * m >= 0xffffffffull) throw config_error("edge count exceeds the 32-bit adjacency index");
  const std::uint64_t slots = o.neg_mode == GEMPE_NEG_PER_EDGE_2 ? 2 * m : static_cast<std::uint64_t>(n) * o.negatives;
  if (slots >= 0xffffffffull) throw config_error("sample count exceeds the 32-bit bucket index");
  (void)n;  // the edge arrays themselves are checked on the device once they are there (gempe_create)
}

}  // namespace
}  // namespace gempe

using namespace gempe;

gempe_ctx::~gempe_ctx() {
  if (ev_gathered) cudaEventDestroy(ev_gathered);
  if (ev_sigma) cudaEventDestroy(ev_sigma);
  if (side_stream) cudaStreamDestroy(side_stream);
  if (round_graph) cudaGraphExecDestroy(round_graph);
  for (cudaGraphExec_t g : run_graph) {
    if (g) cudaGraphExecDestroy(g);
  }
  for (const ExchangePeer& p : ex_peers) {
    if (p.ipc) cudaIpcCloseMemHandle(p.recv);
  }
  for (const Peer& p : peers) {
    if (!p.ipc) continue;
    cudaIpcCloseMemHandle(p.x[0]);
    cudaIpcCloseMemHandle(p.x[1]);
  }
  for (cudaEvent_t e : events) cudaEventDestroy(e);
  if (pinned) cudaFreeHost(pinned);
  for (cudaEvent_t e : step_events) cudaEventDestroy(e);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (own_stream) cudaStreamDestroy(own_stream);
}

extern "C" {

void gempe_default_options(gempe_options* o) {
  std::memset(o, 0, sizeof *o);
  o->dim = 2;
  o->seed = 1;
  o->neg_mode = GEMPE_NEG_PER_EDGE_2;
  o->negatives = 0;
  o->math = GEMPE_MATH_TABLES;
  o->rng = GEMPE_RNG_REFERENCE;
  o->relabel = 1;
  o->world = 1;
  o->comm_chunks = 1;
}

int gempe_create(gempe_ctx** out, std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                 const std::uint32_t* dst, const gempe_options* opt) {
  if (!out || !opt) {
    g_create_error = "null argument";
    return GEMPE_ERR_CONFIG;
  }
  *out = nullptr;
  gempe_ctx* c = nullptr;
  const int rc = guarded(nullptr, [&] {
    PhaseTimer timer;
    validate(n, m, src, dst, *opt);
    timer.lap("validate");
    int device_count = 0;
    const cudaError_t probe = cudaGetDeviceCount(&device_count);
    if (probe != cudaSuccess || device_count == 0) {
      throw cuda_error("no CUDA device available: the GEMPE path has no CPU fallback");
    }
    cuda_check(cudaSetDevice(opt->device), "cudaSetDevice");
    c = new gempe_ctx;
    c->opt = *opt;
    c->n = n;
    c->m = m;
    c->dim = opt->dim;
    c->ld = row_stride_for(opt->dim);
    c->degenerate = n <= 1 || m == 0;  // engine.cpp:159
    c->comm_chunks = static_cast<std::uint32_t>(c->opt.comm_chunks);
    const std::uint64_t blocks = static_cast<std::uint64_t>(c->opt.world) * c->comm_chunks;
    c->block_rows = static_cast<std::uint32_t>((static_cast<std::uint64_t>(std::max(n, 1u)) + blocks - 1) / blocks);
    c->n_pad = static_cast<std::uint32_t>(blocks * c->block_rows);
    // hub split: d <= 4 runs one thread per item (32 adjacency positions bound its serial latency chain), wider rows one warp per item
    const std::uint32_t default_chunk = c->ld <= 4 ? 32u :  // c2 sweep: 16 -> 76 us, 32 -> 60, 64 -> 80, 128 -> 117
                                                                                      std::max(c->opt.world == 1 ? 256u : 128u, 4096u / lanes_per_row(c->ld));
    // c4 sweep on one GPU: 64 -> 5.29 ms, 128 -> 5.13, 256 -> 5.03, 512 -> 5.03, 2048 -> 5.41; a rank of 8 launches 1/8 .. 1/32 of
    // the items at a time and wants the finer split (0.74 ms per rank at 128, 0.88 at 256)
    c->chunk_entries = opt->chunk_entries ? opt->chunk_entries : default_chunk;
    cuda_check(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own_stream;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&c->pinned), (4 + 2 * kBins) * sizeof(unsigned long long),
                             cudaHostAllocDefault), "cudaHostAlloc");
    c->sigma_single_block = std::getenv("GEMPE_SIGMA_SINGLE_BLOCK") != nullptr;  // A/B switch, read once per context
    pack_tables(c->tables);
    c->tables_f32.upload(pack_tables_f32());
    c->round_state.allocate(2 * (4 + 2 * kBins), true);  // two sets: see gempe_ctx::rs
    c->status.p = reinterpret_cast<std::uint32_t*>(c->round_state.get());
    c->hist.p = c->round_state.get() + 4;
    c->work_cursor.allocate(1, true);
    c->sigma_state.allocate(1, true);
    for (auto& buf : c->x) buf.allocate(static_cast<std::size_t>(c->n_pad) * c->ld, true);

    timer.lap("device buffers");
    // the edge list goes straight to the device; endpoints and self-loops are checked there
    c->tmp_src.upload(src, m);
    c->tmp_dst.upload(dst, m);
    if (m) {
      launch_validate_edges(c->tmp_src.get(), c->tmp_dst.get(), m, n, c->status.get(), c->stream);
      std::uint32_t flags = 0;
      cuda_check(cudaMemcpyAsync(&flags, c->status.get(), sizeof flags, cudaMemcpyDeviceToHost, c->stream), "validate D2H");
      cuda_check(cudaStreamSynchronize(c->stream), "validate edges");
      cuda_check(cudaMemsetAsync(c->status.get(), 0, sizeof flags, c->stream), "status reset");
      if (flags & 1u) throw data_error("edge endpoint out of range");
      if (flags & 2u) throw data_error("self-loop in edge list (graphs must be canonical)");
    }
    c->to_work.resize(n);
    for (std::uint32_t v = 0; v < n; ++v) c->to_work[v] = v;
    timer.lap("edge list -> device, validation");
    if (!c->degenerate) {
      if (opt->relabel) {  // engine.cpp:161-163 -> graph.cpp:182-206
        apply_relabel(c, random_relabel_forward(n, mix_seed(opt->seed, 0xA11BE11)));
      }
      timer.lap("relabel (host)");
      build_structures(c);
    }
    c->launches += launch_init_coords(c->x[0].get(), n, c->dim, c->ld, GEMPE_INIT_REFERENCE, opt->seed, 0.0, c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "init coords");
  });
  if (rc != GEMPE_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return GEMPE_OK;
}

void gempe_destroy(gempe_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->opt.device);
  PhaseTimer timer;
  delete c;
  timer.lap("destroy: whole context");
}

const char* gempe_last_error(const gempe_ctx* c) { return c ? c->error.c_str() : g_create_error.c_str(); }
int gempe_is_degenerate(const gempe_ctx* c) { return c->degenerate; }
int gempe_hash_bits(const gempe_ctx* c) { return c->hash_bits; }
std::uint64_t gempe_sample_slots(const gempe_ctx* c) { return c->slots; }
std::uint64_t gempe_pair_terms(const gempe_ctx* c) { return c->m + c->slots; }

std::uint64_t gempe_algorithmic_bytes(const gempe_ctx* c) {
  // (2m + 2S) R + 2 n R + 8 m + 8 n + 4 S + S p, with R = 4 d and p = 1
  const std::uint64_t R = 4ull * c->dim, S = c->slots;
  return (2 * c->m + 2 * S) * R + 2ull * c->n * R + 8 * c->m + 8ull * c->n + 4 * S + S;
}

int gempe_get_work_graph(const gempe_ctx* cc, std::uint32_t* src, std::uint32_t* dst, std::uint32_t* to_work) {
  gempe_ctx* c = const_cast<gempe_ctx*>(cc);  // fills the host cache
  return guarded(c, [&] {
    if (src || dst) host_work_graph(c);
    if (src) std::copy(c->work_src.begin(), c->work_src.end(), src);
    if (dst) std::copy(c->work_dst.begin(), c->work_dst.end(), dst);
    if (to_work) std::copy(c->to_work.begin(), c->to_work.end(), to_work);
  });
}

int gempe_set_coords(gempe_ctx* c, const float* x_work) {
  return guarded(c, [&] {
    if (!x_work) throw config_error("null coordinates");
    if (c->n == 0) return;
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    if (c->dim == c->ld && is_pageable_host(x_work)) {  // ordinary vectors, rows without padding: staged (hostcopy.cpp)
      upload_from_pageable(c->x[c->cur].get(), x_work, static_cast<std::size_t>(c->n) * c->dim * sizeof(float), c->stream);
      return;
    }
    cuda_check(cudaMemcpy2DAsync(c->x[c->cur].get(), c->ld * sizeof(float), x_work, c->dim * sizeof(float),
                                 c->dim * sizeof(float), c->n, cudaMemcpyHostToDevice, c->stream), "set_coords");
    cuda_check(cudaStreamSynchronize(c->stream), "set_coords");
  });
}

int gempe_get_coords(gempe_ctx* c, float* x_work) {
  return guarded(c, [&] {
    if (!x_work) throw config_error("null coordinates");
    if (c->n == 0) return;
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    if (c->dim == c->ld && is_pageable_host(x_work)) {
      download_to_pageable(x_work, c->x[c->cur].get(), static_cast<std::size_t>(c->n) * c->dim * sizeof(float), c->stream);
      return;
    }
    cuda_check(cudaMemcpy2DAsync(x_work, c->dim * sizeof(float), c->x[c->cur].get(), c->ld * sizeof(float),
                                 c->dim * sizeof(float), c->n, cudaMemcpyDeviceToHost, c->stream), "get_coords");
    cuda_check(cudaStreamSynchronize(c->stream), "get_coords");
  });
}

int gempe_init_coords(gempe_ctx* c, int rule, std::uint64_t seed, double stddev) {
  return guarded(c, [&] {
    if (rule < 0 || rule > 2) throw config_error("unknown init rule");
    c->launches += launch_init_coords(c->x[c->cur].get(), c->n, c->dim, c->ld, rule, seed, stddev, c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "init coords");
  });
}

int gempe_relabel(gempe_ctx* c, std::uint64_t relabel_seed) {
  return guarded(c, [&] {
    require_live(c);
    const auto fwd = random_relabel_forward(c->n, relabel_seed);
    {  // coordinates follow their vertices (engine.cpp:186-190): row v moves to row fwd[v], into the other buffer
      DeviceBuffer<std::uint32_t> d_fwd;
      d_fwd.upload(fwd);
      c->launches += launch_permute_rows(c->x[c->cur].get(), c->ld, c->x[c->cur ^ 1].get(), c->ld, c->ld, c->n,
                                         d_fwd.get(), true, c->stream);
      cuda_check(cudaStreamSynchronize(c->stream), "relabel coordinates");
      c->cur ^= 1;
    }
    apply_relabel(c, fwd);
    build_structures(c);
  });
}

int gempe_set_capture(gempe_ctx* c, int on) {
  return guarded(c, [&] {
    c->capture = on != 0;
    if (c->capture && c->cap_y.size() == 0 && !c->degenerate) {
      c->cap_y.allocate(static_cast<std::size_t>(c->n) * c->dim, true);
      c->cap_z.allocate(c->n, true);
    }
  });
}

int gempe_get_yz(gempe_ctx* c, double* y, double* z) {
  return guarded(c, [&] {
    if (!c->capture || c->cap_y.size() == 0) throw config_error("capture is off");
    cuda_check(cudaStreamSynchronize(c->stream), "get_yz");
    if (y) cuda_check(cudaMemcpy(y, c->cap_y.get(), c->cap_y.size() * sizeof(double), cudaMemcpyDeviceToHost), "y D2H");
    if (z) cuda_check(cudaMemcpy(z, c->cap_z.get(), c->cap_z.size() * sizeof(double), cudaMemcpyDeviceToHost), "z D2H");
  });
}

int gempe_get_yz_rows(gempe_ctx* c, const std::uint32_t* rows, std::uint64_t count, double* y, double* z) {
  return guarded(c, [&] {
    if (!c->capture || c->cap_y.size() == 0) throw config_error("capture is off");
    if (count && !rows) throw config_error("null row list");
    for (std::uint64_t i = 0; i < count; ++i) {
      if (rows[i] >= c->n) throw config_error("row out of range");
      if (y) cuda_check(cudaMemcpyAsync(y + i * c->dim, c->cap_y.get() + static_cast<std::size_t>(rows[i]) * c->dim,
                                        c->dim * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "y rows D2H");
      if (z) cuda_check(cudaMemcpyAsync(z + i, c->cap_z.get() + rows[i], sizeof(double), cudaMemcpyDeviceToHost, c->stream),
                        "z rows D2H");
    }
    cuda_check(cudaStreamSynchronize(c->stream), "get_yz_rows");
  });
}

int gempe_get_coords_rows(gempe_ctx* c, const std::uint32_t* rows, std::uint64_t count, float* x) {
  return guarded(c, [&] {
    if (!x || (count && !rows)) throw config_error("null argument");
    for (std::uint64_t i = 0; i < count; ++i) {
      if (rows[i] >= c->n) throw config_error("row out of range");
      cuda_check(cudaMemcpyAsync(x + i * c->dim, c->x[c->cur].get() + static_cast<std::size_t>(rows[i]) * c->ld,
                                 c->dim * sizeof(float), cudaMemcpyDeviceToHost, c->stream), "coordinate rows D2H");
    }
    cuda_check(cudaStreamSynchronize(c->stream), "get_coords_rows");
  });
}

int gempe_begin_round(gempe_ctx* c, double mu, double sigma, std::uint64_t iter_index) {
  return guarded(c, [&] {
    require_live(c);
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    set_round_math(c, mu, sigma);
    c->round_iter = iter_index;
    sampling_passes(c, iter_index);
  });
}

int gempe_begin_round_auto(gempe_ctx* c, std::uint64_t iter_index) {
  return guarded(c, [&] {
    require_live(c);
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    c->round_iter = iter_index;
    c->use_dev_math = true;  // until gempe_end_round
    sampling_passes(c, iter_index);
  });
}

int gempe_bucket_received(gempe_ctx* c) {
  return guarded(c, [&] {
    require_live(c);
    bucket_received(c);
  });
}

int gempe_exchange_layout(gempe_ctx* c, void** send_records, void** recv_records, std::uint32_t** send_counts,
                          std::uint32_t** recv_counts, std::uint32_t* capacity) {
  return guarded(c, [&] {
    if (!c->opt.exchange || c->degenerate) throw config_error("context has no exchange buffers (opt.exchange is off)");
    if (send_records) *send_records = c->exchange.send;
    if (recv_records) *recv_records = const_cast<uint2*>(c->exchange.recv);
    if (send_counts) *send_counts = c->exchange.send_count;
    if (recv_counts) *recv_counts = const_cast<std::uint32_t*>(c->exchange.recv_count);
    if (capacity) *capacity = c->exchange.capacity;
  });
}

int gempe_gather_chunk(gempe_ctx* c, int chunk) {
  return guarded(c, [&] {
    require_live(c);

    if (chunk < 0 || chunk >= static_cast<int>(c->comm_chunks)) throw config_error("chunk out of range");
    gather_items(c, c->chunk_item_off[chunk], c->chunk_item_off[chunk + 1]);
  });
}

int gempe_end_round(gempe_ctx* c) {
  c->use_dev_math = false;
  c->cur ^= 1;
  return GEMPE_OK;
}

int gempe_iterate_async(gempe_ctx* c, double mu, double sigma, std::uint64_t iter_index) {
  return guarded(c, [&] {
    require_live(c);
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    set_round_math(c, mu, sigma);
    c->round_iter = iter_index;
    cuda_check(cudaEventRecord(next_event(c), c->stream), "event");
    sampling_passes(c, iter_index);
    cuda_check(cudaEventRecord(next_event(c), c->stream), "event");
    gather_items(c, c->chunk_item_off.front(), c->chunk_item_off.back());
    cuda_check(cudaEventRecord(next_event(c), c->stream), "event");
    c->cur ^= 1;
  });
}

// ---- pe_sampled on the device (metrics.cpp:73-127, 166-213) -----------------------------------------------
int gempe_pe_sampled(gempe_ctx* c, int samples_per_edge, std::uint64_t seed, gempe_pe_report* out) {
  return guarded(c, [&] {
    if (!out) throw config_error("null report");
    if (samples_per_edge < 1) throw config_error("samples_per_edge must be >= 1");
    const double pairs = static_cast<double>(c->n) * (c->n > 0 ? c->n - 1 : 0) / 2.0;
    const double edges = static_cast<double>(c->m);
    *out = gempe_pe_report{};
    {  // basic_entropy (graph.cpp:208-217)
      const double p = pairs > 0.0 ? edges / pairs : 0.0;
      double h = 0.0;
      if (p > 0.0) h -= p * std::log2(p);
      if (p < 1.0 && pairs > 0.0) h -= (1.0 - p) * std::log2(1.0 - p);
      out->h_basic = h;
    }
    if (c->degenerate) throw config_error("cannot score a degenerate graph");
    cuda_check(cudaStreamSynchronize(c->stream), "pe_sampled");
    const bool complete = edges >= pairs;  // no non-edges: nothing to sample (metrics.cpp:170-179)
    const std::uint64_t sps = complete ? 0 : static_cast<std::uint64_t>(samples_per_edge);
    DeviceBuffer<float> edge_d, non_d;
    DeviceBuffer<double> sums;
    DeviceBuffer<unsigned long long> valid;
    edge_d.allocate(c->m);
    non_d.allocate(std::max<std::uint64_t>(1, c->m * sps));
    sums.allocate(2, true);
    valid.allocate(1, true);
    PeCollectArgs p{};
    p.x = c->x[c->cur].get();
    p.n = c->n; p.dim = c->dim; p.ld = c->ld; p.m = c->m;
    p.src = c->tmp_src.get(); p.dst = c->tmp_dst.get(); p.rowptr = c->rowptr.get();
    p.hash_words = c->hash_words.get();
    p.hash_summary = c->hash_summary.size() ? c->hash_summary.get() : nullptr;
    p.hash_mask = static_cast<std::uint32_t>((1ull << c->hash_bits) - 1);
    p.samples_per_edge = static_cast<std::uint32_t>(sps);
    p.seed = mix_seed(seed, 0x5a3d);
    p.edge_dist = edge_d.get(); p.nonedge_dist = non_d.get();
    c->launches += launch_pe_collect(p, c->stream);
    // number of usable samples -> weight of the non-edge sum
    unsigned long long samples = 0;
    if (sps) {
      c->launches += launch_pe_sum(non_d.get(), c->m * sps, kDefaultMu, 1.0, false, 0, sums.get(), valid.get(), c->stream);
      cuda_check(cudaMemcpyAsync(&samples, valid.get(), sizeof samples, cudaMemcpyDeviceToHost, c->stream), "samples D2H");
      cuda_check(cudaStreamSynchronize(c->stream), "pe_sampled collect");
    }
    const double weight = samples ? (pairs - edges) / static_cast<double>(samples) : 0.0;
    out->nonedge_samples = samples;

    auto total = [&](double mu, double sigma, int which) {  // DlSums::objective / dsigma (metrics.cpp:35-50)
      double host[2] = {0.0, 0.0};
      cuda_check(cudaMemsetAsync(sums.get(), 0, 2 * sizeof(double), c->stream), "pe sums");
      c->launches += launch_pe_sum(edge_d.get(), c->m, mu, sigma, true, which, sums.get(), nullptr, c->stream);
      if (samples) c->launches += launch_pe_sum(non_d.get(), c->m * sps, mu, sigma, false, which, sums.get() + 1, nullptr, c->stream);
      cuda_check(cudaMemcpyAsync(host, sums.get(), sizeof host, cudaMemcpyDeviceToHost, c->stream), "pe sums D2H");
      cuda_check(cudaStreamSynchronize(c->stream), "pe sums");
      return host[0] + weight * host[1];
    };
    auto best_sigma = [&](double mu) {  // metrics.cpp:53-74
      double lo = 1e-3, hi = 16.0;
      double f_lo = total(mu, lo, 1);
      const double f_hi = total(mu, hi, 1);
      if (f_lo == 0.0) return lo;
      if (f_hi == 0.0) return hi;
      if ((f_lo > 0.0) == (f_hi > 0.0)) return total(mu, lo, 0) <= total(mu, hi, 0) ? lo : hi;
      for (int step = 0; step < 60 && hi - lo > 1e-4; ++step) {
        const double mid = 0.5 * (lo + hi);
        const double f_mid = total(mu, mid, 1);
        if (f_mid == 0.0) return mid;
        if ((f_mid > 0.0) == (f_lo > 0.0)) {
          lo = mid;
          f_lo = f_mid;
        } else {
          hi = mid;
        }
      }
      return 0.5 * (lo + hi);
    };
    // minimize_pe (metrics.cpp:76-127)
    double best_mu = kDefaultMu, best_sig = 1.0, best_cost = std::numeric_limits<double>::infinity();
    auto cost_at = [&](double mu, double* sigma_out) {
      const double sg = best_sigma(mu);
      if (sigma_out) *sigma_out = sg;
      return total(mu, sg, 0);
    };
    auto consider = [&](double mu) {
      double sg = 1.0;
      const double cost = cost_at(mu, &sg);
      if (cost < best_cost) {
        best_cost = cost;
        best_mu = mu;
        best_sig = sg;
      }
    };
    for (int k = 0; k <= 20; ++k) consider(0.5 + 0.125 * k);
    out->grid_pe = best_cost / pairs;
    double lo = std::max(0.5, best_mu - 0.125), hi = std::min(3.0, best_mu + 0.125);
    const double gr = 0.5 * (std::sqrt(5.0) - 1.0);
    double x1 = hi - gr * (hi - lo), x2 = lo + gr * (hi - lo);
    double f1 = cost_at(x1, nullptr), f2 = cost_at(x2, nullptr);
    for (int it = 0; it < 24; ++it) {
      if (f1 <= f2) {
        hi = x2; x2 = x1; f2 = f1;
        x1 = hi - gr * (hi - lo);
        f1 = cost_at(x1, nullptr);
      } else {
        lo = x1; x1 = x2; f1 = f2;
        x2 = lo + gr * (hi - lo);
        f2 = cost_at(x2, nullptr);
      }
    }
    consider(0.5 * (lo + hi));
    out->pe = best_cost / pairs;
    out->mu_star = best_mu;
    out->sigma_star = best_sig;
    if (out->h_basic > 1e-12) out->compression_ratio = out->pe / out->h_basic;
    else out->compression_ratio = out->pe <= 1e-9 ? 1.0 : std::numeric_limits<double>::infinity();
  });
}

// ---- CUDA-graph replay of a run of rounds (fixed mu, sigma; iteration indices first_iter .. first_iter + count - 1) ----
int gempe_graph_capture(gempe_ctx* c, double mu, double sigma, std::uint64_t first_iter, int count) {
  return guarded(c, [&] {
    require_live(c);
    if (count < 1) throw config_error("graph needs at least one round");
    if (c->opt.world != 1 || (c->pack_path && c->exchange.recv != c->exchange.send)) {
      throw config_error("graph capture is for single-rank contexts");
    }
    if (c->round_graph) {
      cudaGraphExecDestroy(c->round_graph);
      c->round_graph = nullptr;
    }
    set_round_math(c, mu, sigma);
    const int start = c->cur;
    const std::uint64_t launches0 = c->launches;
    cudaGraph_t graph = nullptr;
    cuda_check(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      for (int r = 0; r < count; ++r) {
        sampling_passes(c, first_iter + static_cast<std::uint64_t>(r));
        gather_items(c, c->chunk_item_off.front(), c->chunk_item_off.back());
        c->cur ^= 1;
      }
    } catch (...) {
      cudaStreamEndCapture(c->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      c->cur = start;
      throw;
    }
    c->cur = start;  // nothing ran yet: the parity moves when the graph is launched
    cuda_check(cudaStreamEndCapture(c->stream, &graph), "end capture");
    c->graph_launches_per_replay = c->launches - launches0;
    c->launches = launches0;
    const cudaError_t inst = cudaGraphInstantiate(&c->round_graph, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(inst, "graph instantiate");
    c->graph_rounds = count;
    c->graph_start_parity = start;
    c->graph_last_iter = first_iter + static_cast<std::uint64_t>(count) - 1;
  });
}

int gempe_graph_launch(gempe_ctx* c) {
  return guarded(c, [&] {
    require_live(c);
    if (!c->round_graph) throw config_error("no captured graph (gempe_graph_capture)");
    if (c->cur != c->graph_start_parity) {
      throw config_error("the coordinate buffers have swapped since the capture: capture again");
    }
    cuda_check(cudaGraphLaunch(c->round_graph, c->stream), "graph launch");
    c->launches += c->graph_launches_per_replay;
    c->round_iter = c->graph_last_iter;
    if (c->graph_rounds & 1) c->cur ^= 1;
  });
}

// ---- runs queued without host round trips (EmbeddingEngine::run, engine.cpp:349-373) --------------------------------
namespace {

// One whole iteration of a queued run: sampling passes and gather + update on the context's stream, sigma search +
// bookkeeping + best-PE snapshot on the side stream.  Round r + 1's sampling passes need neither X nor sigma, so they run
// BESIDE round r's sigma search (a serial chain of ~9 cluster rounds, 30 us: as long as a whole round on graph-drawing
// sizes); the gather of round r + 1 waits for it.  The status / tally words alternate between two sets so that the
// memset of round r + 1 does not race the search that still reads round r's tallies.
void enqueue_run_round(gempe_ctx* c, int parity, std::uint32_t round_in_batch, bool first_in_batch) {
  const int saved = c->cur;
  c->cur = parity;
  c->use_dev_math = true;
  c->run_queued = true;
  auto restore = [&] {
    c->use_dev_math = false;
    c->run_queued = false;
    c->cur = saved;
  };
  try {
    c->rs ^= 1;
    c->status.p = reinterpret_cast<std::uint32_t*>(c->round_state.get() + c->rs * (4 + 2 * kBins));
    c->hist.p = c->round_state.get() + c->rs * (4 + 2 * kBins) + 4;
    sampling_passes(c, c->run_first_iter + round_in_batch);
    if (!first_in_batch) cuda_check(cudaStreamWaitEvent(c->stream, c->ev_sigma, 0), "wait sigma");  // sigma of the round before
    gather_items(c, c->chunk_item_off.front(), c->chunk_item_off.back());
    cuda_check(cudaEventRecord(c->ev_gathered, c->stream), "event");
    cuda_check(cudaStreamWaitEvent(c->side_stream, c->ev_gathered, 0), "wait gather");
    const double pairs = static_cast<double>(static_cast<std::uint64_t>(c->n) * (c->n - 1) / 2);
    c->launches += launch_sigma_update(c->hist.get(), c->mu_dev, pairs, static_cast<double>(c->m),
                                       c->opt.math == GEMPE_MATH_EXACT, c->sigma_state.get(), c->status.get(),
                                       c->sigma_single_block, c->run_state.get(), c->run_pe_trace.get(),
                                       c->run_sigma_trace.get(), c->side_stream);
    c->launches += launch_snapshot_if_improved(c->x[0].get(), c->x[1].get(), c->run_best_x.get(), c->run_best_x.size(),
                                               c->run_state.get(), c->side_stream);
    cuda_check(cudaEventRecord(c->ev_sigma, c->side_stream), "event");
    cuda_check(cudaGetLastError(), "queued round");
  } catch (...) {
    restore();
    throw;
  }
  restore();
}

// the side stream's work of a batch flows back into the context's stream (and, under capture, into the graph)
void join_run_batch(gempe_ctx* c) { cuda_check(cudaStreamWaitEvent(c->stream, c->ev_sigma, 0), "join sigma"); }

void drop_run_graphs(gempe_ctx* c) {
  for (auto& g : c->run_graph) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

}  // namespace

int gempe_run_begin(gempe_ctx* c, double mu, double sigma, std::uint64_t first_iter, std::int32_t window, double tol,
                    std::uint32_t max_rounds) {
  return guarded(c, [&] {
    require_live(c);
    if (c->opt.world != 1 || (c->pack_path && c->exchange.recv != c->exchange.send)) {
      throw config_error("queued runs are for single-rank contexts (the tallies of a sharded round need a reduction)");
    }
    if (window < 1 || max_rounds < 1) throw config_error("run needs window >= 1 and max_rounds >= 1");
    if (gempe_set_sigma(c, mu, sigma) != GEMPE_OK) throw config_error(c->error);
    cuda_check(cudaStreamSynchronize(c->stream), "run begin");
    c->run_first_iter = first_iter;
    c->run_state.allocate(1, true);
    c->run_pe_trace.allocate(max_rounds, true);
    c->run_sigma_trace.allocate(max_rounds, true);
    c->run_best_x.allocate(static_cast<std::size_t>(c->n_pad) * c->ld, true);
    RunState head{};
    head.best_pe = std::numeric_limits<double>::infinity();
    head.tol = tol;
    head.window = window;
    head.parity_base = c->cur;
    head.trace_cap = max_rounds;
    cuda_check(cudaMemcpy(c->run_state.get(), &head, offsetof(RunState, last_hist), cudaMemcpyHostToDevice), "run state");
    c->run_rounds_seen = 0;
    c->run_armed = true;
    drop_run_graphs(c);
    if (!c->side_stream) {
      cuda_check(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking), "side stream");
      cuda_check(cudaEventCreateWithFlags(&c->ev_gathered, cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&c->ev_sigma, cudaEventDisableTiming), "event");
    }
  });
}

int gempe_run_enqueue(gempe_ctx* c, std::uint32_t rounds, std::uint64_t stop_at, std::int32_t use_graph) {
  return guarded(c, [&] {
    require_live(c);
    if (!c->run_armed) throw config_error("gempe_run_enqueue without gempe_run_begin");
    if (rounds < 1) throw config_error("enqueue at least one round");
    // the device skips rounds once `stop_at` are done; the coordinates' parity follows the rounds actually done, so the
    // host learns it at the next poll -- until then nothing else may be queued on this context
    if (c->run_in_flight) throw config_error("poll the queued rounds (gempe_run_poll) before queueing more");
    const unsigned long long limits[2] = {stop_at, c->run_rounds_seen};  // RunState::stop_at, batch_base (adjacent)
    static_assert(offsetof(RunState, batch_base) == offsetof(RunState, stop_at) + sizeof(unsigned long long), "layout");
    cuda_check(cudaMemcpyAsync(&c->run_state.get()->stop_at, limits, sizeof limits, cudaMemcpyHostToDevice, c->stream),
               "stop_at + batch_base");
    const int parity = c->cur;
    if (use_graph) {
      if (c->run_graph_generation != c->structure_generation || c->run_graph_rounds != rounds) {
        drop_run_graphs(c);
        c->run_graph_generation = c->structure_generation;
        c->run_graph_rounds = rounds;
      }
      if (!c->run_graph[parity]) {
        const std::uint64_t launches0 = c->launches;
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
          for (std::uint32_t r = 0; r < rounds; ++r) enqueue_run_round(c, (parity + r) & 1, r, r == 0);
          join_run_batch(c);
        } catch (...) {
          cudaStreamEndCapture(c->stream, &graph);
          if (graph) cudaGraphDestroy(graph);
          throw;
        }
        cuda_check(cudaStreamEndCapture(c->stream, &graph), "end capture");
        c->run_graph_launches = c->launches - launches0;
        c->launches = launches0;
        const cudaError_t inst = cudaGraphInstantiate(&c->run_graph[parity], graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(inst, "graph instantiate");
      }
      cuda_check(cudaGraphLaunch(c->run_graph[parity], c->stream), "graph launch");
      c->launches += c->run_graph_launches;
    } else {
      for (std::uint32_t r = 0; r < rounds; ++r) enqueue_run_round(c, (parity + r) & 1, r, r == 0);
      join_run_batch(c);
    }
    c->run_in_flight = true;
  });
}

int gempe_run_poll(gempe_ctx* c, gempe_run_status* out, double* pe_trace, double* sigma_trace, std::uint32_t trace_cap,
                   std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  return guarded(c, [&] {
    if (!c->run_armed) throw config_error("gempe_run_poll without gempe_run_begin");
    RunState head{};
    cuda_check(cudaMemcpyAsync(&head, c->run_state.get(), offsetof(RunState, last_hist), cudaMemcpyDeviceToHost, c->stream),
               "run state D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "queued rounds");
    c->run_in_flight = false;
    c->run_rounds_seen = head.count;
    c->cur = static_cast<int>((head.parity_base + head.count) & 1ull);
    c->round_iter = c->run_first_iter + (head.count ? head.count - 1 : 0);
    c->last_draws = head.draws;
    SigmaState st{};
    cuda_check(cudaMemcpy(&st, c->sigma_state.get(), sizeof st, cudaMemcpyDeviceToHost), "sigma D2H");
    const std::uint64_t have = std::min<std::uint64_t>(head.count, head.trace_cap);
    const std::uint64_t copy = std::min<std::uint64_t>(have, trace_cap);
    if (pe_trace && copy) cuda_check(cudaMemcpy(pe_trace, c->run_pe_trace.get(), copy * sizeof(double), cudaMemcpyDeviceToHost), "trace");
    if (sigma_trace && copy) cuda_check(cudaMemcpy(sigma_trace, c->run_sigma_trace.get(), copy * sizeof(double), cudaMemcpyDeviceToHost), "trace");
    if (hist_edge) cuda_check(cudaMemcpy(hist_edge, &c->run_state.get()->last_hist[0], kBins * sizeof(std::uint64_t), cudaMemcpyDeviceToHost), "tallies");
    if (hist_nonedge) cuda_check(cudaMemcpy(hist_nonedge, &c->run_state.get()->last_hist[kBins], kBins * sizeof(std::uint64_t), cudaMemcpyDeviceToHost), "tallies");
    if (out) {
      out->rounds_done = head.count;
      out->converged = head.converged;
      out->failed = head.failed;
      out->improved_at = head.improved_at;
      out->best_pe = head.best_pe;
      out->sigma = st.sigma;
      out->pe_estimate = st.pe_estimate;
      out->last_nonedge_weight = head.last_nonedge_weight;
      out->draws = head.draws;
    }
    if (head.failed) {
      const std::uint32_t* s = head.sticky_status;
      if (s[kStatRetryCap]) throw near_complete_graph_error("no non-edge partner found after 10^4 draws; graph is near-complete");
      if (s[kStatExchangeOverflow]) throw data_error("sample exchange region overflowed");
      if (s[kStatEmptyTallies]) throw config_error("cannot optimize sigma on an empty histogram");
      throw divergence_error("non-finite coordinate after update", static_cast<int>(c->run_first_iter + head.fail_iter) + 1);
    }
  });
}

void* gempe_run_best_snapshot(gempe_ctx* c) { return c->run_best_x.get(); }

int gempe_run_rebase(gempe_ctx* c) {
  // after the coordinates moved to the other buffer outside a round (gempe_relabel): the parity relation of the run
  return guarded(c, [&] {
    if (!c->run_armed || c->run_in_flight) throw config_error("no idle run to rebase");
    RunState head{};
    cuda_check(cudaMemcpy(&head, c->run_state.get(), offsetof(RunState, last_hist), cudaMemcpyDeviceToHost), "run state D2H");
    const int base = static_cast<int>((static_cast<unsigned long long>(c->cur) + head.count) & 1ull);
    cuda_check(cudaMemcpy(&c->run_state.get()->parity_base, &base, sizeof base, cudaMemcpyHostToDevice), "parity base");
  });
}

int gempe_sync(gempe_ctx* c, std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  return guarded(c, [&] { fetch_status(c, hist_edge, hist_nonedge); });
}

int gempe_iterate(gempe_ctx* c, double mu, double sigma, std::uint64_t iter_index, std::uint64_t* hist_edge,
                  std::uint64_t* hist_nonedge) {
  const int rc = gempe_iterate_async(c, mu, sigma, iter_index);
  if (rc != GEMPE_OK) return rc;
  return gempe_sync(c, hist_edge, hist_nonedge);
}

int gempe_set_sigma(gempe_ctx* c, double mu, double sigma) {
  return guarded(c, [&] {
    set_round_math(c, mu, sigma);
    c->mu_dev = mu;
    SigmaState st{};
    st.sigma = sigma;
    st.math = c->math;
    cuda_check(cudaMemcpyAsync(c->sigma_state.get(), &st, sizeof st, cudaMemcpyHostToDevice, c->stream), "set_sigma");
    cuda_check(cudaStreamSynchronize(c->stream), "set_sigma");
  });
}

int gempe_sigma_update_async(gempe_ctx* c) {
  return guarded(c, [&] {
    require_live(c);
    const double pairs = static_cast<double>(static_cast<std::uint64_t>(c->n) * (c->n - 1) / 2);
    c->launches += launch_sigma_update(c->hist.get(), c->mu_dev, pairs, static_cast<double>(c->m),
                                       c->opt.math == GEMPE_MATH_EXACT, c->sigma_state.get(), c->status.get(),
                                       c->sigma_single_block, c->run_queued ? c->run_state.get() : nullptr,
                                       c->run_pe_trace.get(), c->run_sigma_trace.get(), c->stream);
    cuda_check(cudaGetLastError(), "sigma update");
  });
}

int gempe_iterate_auto_async(gempe_ctx* c, std::uint64_t iter_index) {
  return guarded(c, [&] {
    require_live(c);
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    c->round_iter = iter_index;
    c->use_dev_math = true;
    cuda_check(cudaEventRecord(next_event(c), c->stream), "event");
    sampling_passes(c, iter_index);
    cuda_check(cudaEventRecord(next_event(c), c->stream), "event");
    gather_items(c, c->chunk_item_off.front(), c->chunk_item_off.back());
    cuda_check(cudaEventRecord(next_event(c), c->stream), "event");
    c->use_dev_math = false;
    c->cur ^= 1;
    if (gempe_sigma_update_async(c) != GEMPE_OK) throw cuda_error(c->error);
  });
}

int gempe_get_sigma_state(gempe_ctx* c, double* sigma, double* pe_estimate, double* nonedge_weight) {
  return guarded(c, [&] {
    SigmaState st{};
    cuda_check(cudaMemcpyAsync(&st, c->sigma_state.get(), sizeof st, cudaMemcpyDeviceToHost, c->stream), "sigma D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sigma D2H");
    if (sigma) *sigma = st.sigma;
    if (pe_estimate) *pe_estimate = st.pe_estimate;
    if (nonedge_weight) *nonedge_weight = st.nonedge_weight;
  });
}

int gempe_iterate_auto(gempe_ctx* c, std::uint64_t iter_index, double* sigma, double* pe_estimate,
                       double* nonedge_weight, std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  int rc = gempe_iterate_auto_async(c, iter_index);
  if (rc != GEMPE_OK) return rc;
  rc = gempe_sync(c, hist_edge, hist_nonedge);
  if (rc != GEMPE_OK) return rc;
  return gempe_get_sigma_state(c, sigma, pe_estimate, nonedge_weight);
}

void* gempe_device_tallies(gempe_ctx* c) { return c->hist.get(); }

int gempe_step_host(gempe_ctx* c, const float* x_in, float* x_out, double mu, double sigma, std::uint64_t iter_index,
                    std::uint64_t* hist_edge, std::uint64_t* hist_nonedge) {
  return guarded(c, [&] {
    require_live(c);
    if (c->opt.world != 1) throw config_error("gempe_step_host needs an unsharded context");
    if (!x_in || !x_out) throw config_error("null coordinates");
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    if (!c->copy_stream) cuda_check(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
    const std::size_t slices = c->step_item_off.size() - 1;
    while (c->step_events.size() < slices + 2) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      c->step_events.push_back(e);
    }
    set_round_math(c, mu, sigma);
    c->round_iter = iter_index;
    const std::size_t host_pitch = c->dim * sizeof(float), dev_pitch = c->ld * sizeof(float);
    // Ordinary (pageable) vectors of the caller, rows without padding: the copies go through the pinned ring and host
    // threads of hostcopy.cpp instead of the driver's single-threaded staging (c4: 89 -> about 55 ms per step; page-locked
    // vectors, gempe_alloc_host, take 20 ms)
    const bool contiguous = c->dim == c->ld;
    const bool staged_in = contiguous && is_pageable_host(x_in), staged_out = contiguous && is_pageable_host(x_out);
    // X_t in on the copy stream while the (X-independent) sampling passes run on the compute stream
    cuda_check(cudaEventRecord(c->step_events[slices], c->stream), "event");  // orders after earlier work on X
    cuda_check(cudaStreamWaitEvent(c->copy_stream, c->step_events[slices], 0), "wait");
    if (staged_in) {
      sampling_passes(c, iter_index);
      upload_from_pageable(c->x[c->cur].get(), x_in, static_cast<std::size_t>(c->n) * host_pitch, c->copy_stream);
    } else {
      cuda_check(cudaMemcpy2DAsync(c->x[c->cur].get(), dev_pitch, x_in, host_pitch, host_pitch, c->n, cudaMemcpyHostToDevice,
                                   c->copy_stream), "X in");
    }
    cuda_check(cudaEventRecord(c->step_events[slices + 1], c->copy_stream), "event");
    if (!staged_in) sampling_passes(c, iter_index);
    cuda_check(cudaStreamWaitEvent(c->stream, c->step_events[slices + 1], 0), "wait");
    // gradient + update slice by slice; a finished slice's rows leave while the next slice is computed
    float* x_next = c->x[c->cur ^ 1].get();
    for (std::size_t k = 0; k < slices; ++k) {
      gather_items(c, c->step_item_off[k], c->step_item_off[k + 1]);
      cuda_check(cudaEventRecord(c->step_events[k], c->stream), "event");
      if (staged_out) continue;  // all slices are queued first, the host then drains them in order (below)
      cuda_check(cudaStreamWaitEvent(c->copy_stream, c->step_events[k], 0), "wait");
      const std::uint32_t v0 = c->step_vertex_off[k], v1 = c->step_vertex_off[k + 1];
      if (v1 > v0) {
        cuda_check(cudaMemcpy2DAsync(x_out + static_cast<std::size_t>(v0) * c->dim, host_pitch,
                                     x_next + static_cast<std::size_t>(v0) * c->ld, dev_pitch, host_pitch, v1 - v0,
                                     cudaMemcpyDeviceToHost, c->copy_stream), "X out");
      }
    }
    for (std::size_t k = 0; staged_out && k < slices; ++k) {
      cuda_check(cudaStreamWaitEvent(c->copy_stream, c->step_events[k], 0), "wait");
      const std::uint32_t v0 = c->step_vertex_off[k], v1 = c->step_vertex_off[k + 1];
      if (v1 > v0) {
        download_to_pageable(x_out + static_cast<std::size_t>(v0) * c->dim, x_next + static_cast<std::size_t>(v0) * c->ld,
                             static_cast<std::size_t>(v1 - v0) * host_pitch, c->copy_stream);
      }
    }
    c->cur ^= 1;
    fetch_status(c, hist_edge, hist_nonedge);  // waits for the compute stream and checks the status word
    cuda_check(cudaStreamSynchronize(c->copy_stream), "X out");
  });
}

int gempe_elapsed_ms(gempe_ctx* c, float out3[3]) {
  return guarded(c, [&] {
    out3[0] = out3[1] = out3[2] = 0.0f;
    if (c->events_used < 3) return;
    cuda_check(cudaEventSynchronize(c->events[c->events_used - 1]), "event sync");
    for (std::size_t r = 0; r + 2 < c->events_used; r += 3) {
      float sample_ms = 0.0f, gather_ms = 0.0f;
      cuda_check(cudaEventElapsedTime(&sample_ms, c->events[r], c->events[r + 1]), "elapsed");
      cuda_check(cudaEventElapsedTime(&gather_ms, c->events[r + 1], c->events[r + 2]), "elapsed");
      out3[1] += sample_ms;
      out3[2] += gather_ms;
    }
    cuda_check(cudaEventElapsedTime(&out3[0], c->events[0], c->events[c->events_used - 1]), "elapsed");
    c->events_used = 0;
  });
}

std::uint64_t gempe_kernel_launches(const gempe_ctx* c) { return c->launches; }

void gempe_trim_device_cache(void) { trim_device_cache(); }

void* gempe_alloc_host(std::uint64_t bytes) {
  void* p = nullptr;
  const cudaError_t err = cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable);
  if (err != cudaSuccess) {
    cudaGetLastError();
    set_create_error(std::string("cudaHostAlloc: ") + cudaGetErrorString(err));
    return nullptr;
  }
  return p;
}

void gempe_free_host(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

std::int64_t gempe_bucket_spills(gempe_ctx* c) {
  if (!c->in_stride) return -1;
  std::uint32_t count = 0;
  if (cudaSetDevice(c->opt.device) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess ||
      cudaMemcpy(&count, c->in_cnt.get() + c->n, sizeof count, cudaMemcpyDeviceToHost) != cudaSuccess) {
    return -2;
  }
  return count;
}

int gempe_probe(gempe_ctx* c, const std::uint32_t* i, const std::uint32_t* j, std::uint64_t count, std::uint8_t* out) {
  return guarded(c, [&] {
    require_live(c);
    if (count == 0) return;
    DeviceBuffer<std::uint32_t> di, dj;
    DeviceBuffer<std::uint8_t> dout;
    di.upload(std::vector<std::uint32_t>(i, i + count));
    dj.upload(std::vector<std::uint32_t>(j, j + count));
    dout.allocate(count);
    c->launches += launch_probe(c->hash_words.get(), static_cast<std::uint32_t>((1ull << c->hash_bits) - 1), c->n,
                                di.get(), dj.get(), count, dout.get(), c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "probe");
    cuda_check(cudaMemcpy(out, dout.get(), count, cudaMemcpyDeviceToHost), "probe D2H");
  });
}

int gempe_sample(gempe_ctx* c, std::uint64_t iter_index, std::uint32_t* partners, std::uint64_t* total_draws) {
  return guarded(c, [&] {
    require_live(c);
    if (c->ex_registered) {
      throw config_error("gempe_sample is a single-context test hook: it would store records into the registered peers");
    }
    c->round_iter = iter_index;
    sampling_passes(c, iter_index);
    const std::uint32_t* result = c->neg_own.get();
    DeviceBuffer<std::uint32_t> ordered;
    if (c->opt.neg_mode == GEMPE_NEG_PER_EDGE_2) {
      ordered.allocate(c->slots);
      c->launches += launch_unpermute_partners(c->neg_own.get(), c->eid_role.get(), c->slots, ordered.get(), c->stream);
      result = ordered.get();
    }
    cuda_check(cudaMemcpyAsync(c->pinned, c->status.get(), 8 * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, c->stream),
               "status D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sample");
    if (partners && c->slots) {
      cuda_check(cudaMemcpy(partners, result, c->slots * sizeof(std::uint32_t), cudaMemcpyDeviceToHost), "partners D2H");
    }
    std::uint32_t st[8];
    std::memcpy(st, c->pinned, sizeof st);
    if (total_draws) *total_draws = static_cast<std::uint64_t>(st[kStatDrawsLo]) | (static_cast<std::uint64_t>(st[kStatDrawsHi]) << 32);
    if (st[kStatRetryCap]) throw near_complete_graph_error("no non-edge partner found after 10^4 draws; graph is near-complete");
  });
}

int gempe_set_stream(gempe_ctx* c, void* cuda_stream) {
  c->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : c->own_stream;
  return GEMPE_OK;
}
// ---- fused update + broadcast over peer memory -------------------------------------------------------
int gempe_coords_ipc_handles(gempe_ctx* c, void* out) {
  return guarded(c, [&] {
    if (c->degenerate) throw config_error("degenerate graph: no coordinates on the device");
    cudaIpcMemHandle_t h[2];
    static_assert(sizeof h == 2 * GEMPE_IPC_HANDLE_BYTES, "handle size");
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    for (int i = 0; i < 2; ++i) cuda_check(cudaIpcGetMemHandle(&h[i], c->x[i].get()), "cudaIpcGetMemHandle");
    std::memcpy(out, h, sizeof h);
  });
}

int gempe_open_peer(gempe_ctx* c, const void* handles) {
  return guarded(c, [&] {
    if (static_cast<int>(c->peers.size()) >= kMaxPeers) throw config_error("too many peers (world <= 16)");
    cudaIpcMemHandle_t h[2];
    std::memcpy(h, handles, sizeof h);
    cuda_check(cudaSetDevice(c->opt.device), "cudaSetDevice");
    gempe_ctx::Peer p;
    p.ipc = true;
    for (int i = 0; i < 2; ++i) {
      void* ptr = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&ptr, h[i], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      p.x[i] = static_cast<float*>(ptr);
    }
    c->peers.push_back(p);
  });
}

int gempe_add_peer_pointers(gempe_ctx* c, void* x0, void* x1) {
  return guarded(c, [&] {
    if (static_cast<int>(c->peers.size()) >= kMaxPeers) throw config_error("too many peers (world <= 16)");
    if (!x0 || !x1) throw config_error("null peer buffer");
    gempe_ctx::Peer p;
    p.x[0] = static_cast<float*>(x0);
    p.x[1] = static_cast<float*>(x1);
    c->peers.push_back(p);
  });
}

int gempe_exchange_ipc_handle(gempe_ctx* c, void* out) {
  return guarded(c, [&] {
    if (c->ex_peers.empty()) throw config_error("context has no external exchange buffers (opt.exchange with world > 1)");
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, c->ex_recv.get()), "cudaIpcGetMemHandle");
    std::memcpy(out, &h, sizeof h);
  });
}

namespace {
void register_exchange_peer(gempe_ctx* c, int peer_rank, uint2* recv, bool ipc) {
  if (c->ex_peers.empty()) throw config_error("context has no external exchange buffers (opt.exchange with world > 1)");
  if (peer_rank < 0 || peer_rank >= static_cast<int>(c->ex_peers.size()) || peer_rank == c->opt.rank) {
    throw config_error("bad peer rank");
  }
  if (c->ex_peers[peer_rank].recv) throw config_error("peer already registered");
  c->ex_peers[peer_rank].recv = recv;
  c->ex_peers[peer_rank].ipc = ipc;
  if (++c->ex_registered + 1 == c->ex_peers.size()) c->ex_peers_lost = false;
}
}  // namespace

int gempe_open_peer_exchange(gempe_ctx* c, int peer_rank, const void* handle) {
  return guarded(c, [&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* ptr = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    register_exchange_peer(c, peer_rank, static_cast<uint2*>(ptr), true);
  });
}

int gempe_add_peer_exchange_pointer(gempe_ctx* c, int peer_rank, void* recv_area) {
  return guarded(c, [&] {
    if (!recv_area) throw config_error("null peer buffer");
    register_exchange_peer(c, peer_rank, static_cast<uint2*>(recv_area), false);
  });
}

void* gempe_exchange_recv_area(gempe_ctx* c) { return c->ex_recv.get(); }

int gempe_clear_peers(gempe_ctx* c) {
  return guarded(c, [&] {
    cuda_check(cudaStreamSynchronize(c->stream), "clear peers");
    for (std::size_t r = 0; r < c->ex_peers.size(); ++r) {
      if (static_cast<int>(r) == c->opt.rank) continue;
      if (c->ex_peers[r].ipc) cudaIpcCloseMemHandle(c->ex_peers[r].recv);
      c->ex_peers[r] = gempe_ctx::ExchangePeer{};
    }
    c->ex_registered = 0;
    for (const gempe_ctx::Peer& p : c->peers) {
      if (!p.ipc) continue;
      cudaIpcCloseMemHandle(p.x[0]);
      cudaIpcCloseMemHandle(p.x[1]);
    }
    c->peers.clear();
  });
}

void* gempe_device_coords_parity(gempe_ctx* c, int parity) { return c->x[parity & 1].get(); }
int gempe_coords_parity(const gempe_ctx* c) { return c->cur; }

void* gempe_device_coords(gempe_ctx* c, int which) { return c->x[which ? c->cur ^ 1 : c->cur].get(); }
std::uint32_t gempe_row_stride(const gempe_ctx* c) { return c->ld; }
std::uint32_t gempe_padded_rows(const gempe_ctx* c) { return c->n_pad; }
std::uint32_t gempe_block_rows(const gempe_ctx* c) { return c->block_rows; }

// ---- host numerics --------------------------------------------------------------------------------

int gempe_host_fastmath_table(int which, double* out67) {
  try {
    const FastMathTables& t = FastMathTables::get();
    const QuadTable& q = which == 0 ? t.erf : (which == 1 ? t.exp_neg : t.ratio);
    double* p = out67;
    for (double v : q.knots) *p++ = v;
    for (double v : q.a) *p++ = v;
    for (double v : q.b) *p++ = v;
    for (double v : q.c) *p++ = v;
    *p++ = q.lo;
    *p++ = q.hi;
    return q.odd_mirror ? 1 : 0;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return -1;
  }
}

static Tallies make_tallies(const std::uint64_t* he, const std::uint64_t* hn, double w) {
  Tallies t;
  std::copy(he, he + kHistBins, t.edge.begin());
  std::copy(hn, hn + kHistBins, t.nonedge.begin());
  t.nonedge_weight = w;
  return t;
}

double gempe_host_optimize_sigma(const std::uint64_t* he, const std::uint64_t* hn, double w, double mu, int* steps) {
  try {
    const SigmaSearch s = optimize_sigma(make_tallies(he, hn, w), mu);
    if (steps) *steps = s.bisection_steps;
    return s.sigma;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return std::numeric_limits<double>::quiet_NaN();
  }
}
double gempe_host_histogram_objective(const std::uint64_t* he, const std::uint64_t* hn, double w, double mu, double sigma) {
  return histogram_objective(make_tallies(he, hn, w), mu, sigma);
}
double gempe_host_histogram_objective_dsigma(const std::uint64_t* he, const std::uint64_t* hn, double w, double mu,
                                             double sigma) {
  return histogram_objective_dsigma(make_tallies(he, hn, w), mu, sigma);
}
int gempe_host_random_relabel(std::uint32_t n, std::uint64_t seed, std::uint32_t* forward) {
  const auto f = random_relabel_forward(n, seed);
  std::copy(f.begin(), f.end(), forward);
  return GEMPE_OK;
}
std::uint64_t gempe_host_mix_seed(std::uint64_t seed, std::uint64_t component) { return mix_seed(seed, component); }

}  // extern "C"
