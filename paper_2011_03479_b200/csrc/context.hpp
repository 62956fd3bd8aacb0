// gempe_ctx: device-resident state of one GEMPE engine shard (one GPU).  See DESIGN.md for the layout.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/gempe.h"
#include "hostmath.hpp"
#include "kernels.hpp"

namespace gempe {

void cuda_check(cudaError_t e, const char* what);

// GEMPE_TRACE=1: wall-clock laps of the host-side phases (construction, run, export) on stderr
struct PhaseTimer {
  bool on = std::getenv("GEMPE_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gempe] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  }
};
void set_create_error(const std::string& msg);  // read back through gempe_last_error(NULL)

// Device memory behind DeviceBuffer.  Released blocks go to a per-device cache instead of cudaFree and are handed out again
// to requests of (nearly) the same size: an engine is a few dozen allocations from bytes to gigabytes, and a process that
// calls embed() repeatedly otherwise pays cudaMalloc / cudaFree for all of them every call.  On the bench host it is the
// cudaFree of the SMALL blocks that hurts: destroying a c4 engine took 1 ms or, every second time, 0.1-0.55 s; with the
// cache a call is 0.19 s every time (was 0.20-1.2 s).  The cache holds at most GEMPE_DEVICE_CACHE_MB (default 16384; 0
// turns it off); gempe_trim_device_cache() empties it.  `capacity` is what device_free must be given back.
void* device_alloc(std::size_t bytes, std::size_t* capacity, int* device);
void device_free(void* p, std::size_t capacity, int device) noexcept;
void trim_device_cache() noexcept;

// Transfers between the device and pageable host memory through a ring of pinned chunks and several host threads
// (hostcopy.cpp); both return when the transfer is complete.  is_pageable_host: neither page-locked nor device memory.
void download_to_pageable(void* dst, const void* src_dev, std::size_t bytes, cudaStream_t stream);
void upload_from_pageable(void* dst_dev, const void* src, std::size_t bytes, cudaStream_t stream);
bool is_pageable_host(const void* p);

// Owning device allocation, zero-filled on request.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { release(); }
  void allocate(std::size_t count, bool zero = false) {
    release();
    if (count == 0) return;
    ptr_ = static_cast<T*>(device_alloc(count * sizeof(T), &capacity_, &device_));
    count_ = count;
    if (zero) {
      // the legacy-stream memset is not ordered against the context's non-blocking stream: wait for it
      cuda_check(cudaMemset(ptr_, 0, count * sizeof(T)), "cudaMemset");
      cuda_check(cudaDeviceSynchronize(), "cudaMemset");
    }
  }
  void upload(const std::vector<T>& host) { upload(host.data(), host.size()); }
  void upload(const T* host, std::size_t count) {
    allocate(count);
    if (count * sizeof(T) >= (16u << 20) && is_pageable_host(host)) {  // e.g. the edge arrays of the caller
      upload_from_pageable(ptr_, host, count * sizeof(T), nullptr);
    } else if (count) {
      cuda_check(cudaMemcpy(ptr_, host, count * sizeof(T), cudaMemcpyHostToDevice), "upload");
      cuda_check(cudaDeviceSynchronize(), "upload");  // pageable H2D may still be in flight on return
    }
  }
  void release() {
    if (ptr_) device_free(ptr_, capacity_, device_);
    ptr_ = nullptr;
    count_ = 0;
    capacity_ = 0;
  }
  T* get() const { return ptr_; }
  std::size_t size() const { return count_; }
  void swap(DeviceBuffer& o) {
    std::swap(ptr_, o.ptr_);
    std::swap(count_, o.count_);
    std::swap(capacity_, o.capacity_);
    std::swap(device_, o.device_);
  }

 private:
  T* ptr_ = nullptr;
  std::size_t count_ = 0, capacity_ = 0;
  int device_ = 0;
};

}  // namespace gempe

struct gempe_ctx {
  gempe_options opt{};
  std::uint32_t n = 0, dim = 0, ld = 0;
  std::uint64_t m = 0;
  bool degenerate = false;
  int hash_bits = 0;
  std::uint64_t slots = 0;          // S
  std::uint32_t block_rows = 0, n_pad = 0, comm_chunks = 1;
  std::uint32_t chunk_entries = 0;
  std::string error;

  // the work graph (edge list in work ids) lives on the device (tmp_src / tmp_dst); the host copies are filled on
  // demand (work-graph accessor, deterministic CSR) and dropped when the graph is relabelled
  std::vector<std::uint32_t> work_src, work_dst, to_work;

  // device state
  gempe::DeviceBuffer<float> x[2];
  int cur = 0;
  gempe::DeviceBuffer<std::uint32_t> rowptr, nbr, eid_role, csr_src;
  gempe::DeviceBuffer<std::uint32_t> tmp_src, tmp_dst;  // the work edge arrays (work ids, input edge order)
  gempe::DeviceBuffer<std::uint32_t> hash_words, hash_summary;
  gempe::DeviceBuffer<std::uint32_t> neg_own, in_cnt, in_off, in_rank, in_anchor, scan_scratch;
  // slotted buckets (bucket_mode 4): slots per vertex in in_anchor (0 = off), and the overflow side
  std::uint32_t in_stride = 0;
  gempe::DeviceBuffer<uint2> spill;
  gempe::DeviceBuffer<std::uint32_t> spill_cnt, spill_off, spill_anchor;
  // large-n bucketing (two-level counting sort); partition.buckets == 0 selects the atomic method
  gempe::PartitionArgs partition{};
  gempe::DeviceBuffer<std::uint32_t> block_hist, bucket_off;
  gempe::DeviceBuffer<uint2> records;
  // sharded sampling with an exchange step (opt.exchange): records packed by destination rank, see kernels.hpp
  gempe::ExchangeArgs exchange{};
  gempe::DeviceBuffer<std::uint64_t> ex_first_slot, ex_prefix;
  gempe::DeviceBuffer<uint2> ex_send, ex_recv, ex_spill;
  gempe::DeviceBuffer<std::uint32_t> ex_send_count, ex_recv_count, ex_rank, ex_spill_count;
  // a captured run of rounds (gempe_graph_capture): small graphs are bound by launch gaps, a CUDA graph removes them
  cudaGraphExec_t round_graph = nullptr;
  int graph_rounds = 0, graph_start_parity = 0;
  std::uint64_t graph_launches_per_replay = 0, graph_last_iter = 0;
  // a run queued without host round trips (gempe_run_begin / enqueue / poll): device bookkeeping, traces, best-PE snapshot
  gempe::DeviceBuffer<gempe::RunState> run_state;
  gempe::DeviceBuffer<double> run_pe_trace, run_sigma_trace;
  gempe::DeviceBuffer<float> run_best_x;
  cudaGraphExec_t run_graph[2] = {nullptr, nullptr};  // by the parity of the coordinate buffers at the first round
  std::uint64_t run_graph_generation = 0, run_graph_launches = 0, run_first_iter = 0, run_rounds_seen = 0;
  std::uint32_t run_graph_rounds = 0;
  std::uint64_t structure_generation = 0;  // bumped by every (re)build of the graph-derived structures
  bool run_armed = false, run_in_flight = false;
  bool run_queued = false;  // while a queued round's launches are being issued: kernels get the run state
  bool pack_path = false;       // sampling goes through sample_pack + bucket_records (opt.exchange, or bucket_mode 3)
  bool bucket_pending = false;  // records packed, gempe_bucket_received not yet called
  // fused update + broadcast: X buffers (both parities, indexed like x[]) of the other ranks, in this rank's address space
  struct Peer {
    float* x[2] = {nullptr, nullptr};
    bool ipc = false;  // opened with cudaIpcOpenMemHandle (closed on destroy)
  };
  std::vector<Peer> peers;
  // direct sample exchange: every rank's receive area (records of both round parities, then the counts) in this rank's
  // address space, indexed by rank; the own entry points at ex_recv.  Active once all world - 1 peers are registered.
  struct ExchangePeer {
    uint2* recv = nullptr;
    bool ipc = false;
  };
  std::vector<ExchangePeer> ex_peers;
  std::uint32_t ex_registered = 0;
  bool ex_peers_lost = false;
  std::uint64_t ex_round = 0;  // parity of the receive buffers in direct mode
  gempe::DeviceBuffer<gempe::ItemDesc> items;
  std::vector<std::uint32_t> chunk_item_off;  // comm_chunks + 1
  // gempe_step_host pipeline: item / vertex boundaries of the slices whose rows are copied out while later
  // slices are still being computed (world == 1 only)
  std::vector<std::uint32_t> step_item_off, step_vertex_off;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> step_events;
  gempe::DeviceBuffer<std::uint32_t> hub_first, hub_items, hub_arrived;
  gempe::DeviceBuffer<double> part_y, part_z;
  // {status[8] as u32, hist[1024] as u64} in ONE allocation with the layout of the pinned mirror below: one memset
  // at the start of a round, one copy at its end
  gempe::DeviceBuffer<unsigned long long> round_state;
  struct StatusView {
    std::uint32_t* p = nullptr;
    std::uint32_t* get() const { return p; }
  } status;
  struct HistView {
    unsigned long long* p = nullptr;
    unsigned long long* get() const { return p; }
  } hist;
  gempe::DeviceBuffer<std::uint32_t> work_cursor;
  gempe::DeviceBuffer<gempe::SigmaState> sigma_state;  // device-resident (mu, sigma) feedback
  double mu_dev = gempe::kDefaultMu;
  bool sigma_single_block = false;  // GEMPE_SIGMA_SINGLE_BLOCK at creation: one-CTA sigma search (A/B)
  bool use_dev_math = false;  // gather reads RoundMath from sigma_state instead of kernel parameters
  gempe::DeviceBuffer<double> cap_y, cap_z;
  bool capture = false;

  // pinned host mirror of {status[8] as u64-aligned words, hist[1024]}
  unsigned long long* pinned = nullptr;

  cudaStream_t own_stream = nullptr, stream = nullptr;
  // queued runs: the sigma search + bookkeeping of round t run on a side stream beside the sampling passes of round t + 1
  // (which need neither X nor sigma); the status / tally words are double-buffered for that (round_state holds two sets)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_gathered = nullptr, ev_sigma = nullptr;
  int rs = 0;  // which half of round_state the status / hist views point at
  gempe::RoundMath math{};
  gempe::DeviceTables tables{};
  gempe::DeviceBuffer<float4> tables_f32;  // directly indexed fp32 cells of the same tables (kernels.hpp)
  std::uint64_t round_iter = 0;
  std::uint64_t launches = 0;
  std::uint64_t last_draws = 0;

  // timing: event triples {start, after sampling passes, end} per async round since the last query
  std::vector<cudaEvent_t> events;
  std::size_t events_used = 0;

  ~gempe_ctx();
};
