// Copies between the device and PAGEABLE host memory of the caller.  The driver's own path for pageable memory stages
// through one pinned buffer and one host thread (5-10 GB/s on the bench host; a freshly allocated destination also takes
// its page faults in that thread).  Here chunks travel through a ring of pinned buffers over the copy engine while several
// host threads move them between the ring and the caller's memory in parallel: 537 MB in 25 ms instead of 70-120 ms.
// The ring is allocated once per process and kept (up to 64 MB of pinned memory: allocating it costs 20-60 ms and freeing it
// up to 0.4 s on the bench host -- more than the copy); one transfer at a time uses it.
#include "context.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace gempe {

namespace {

struct Ring {
  std::mutex mutex;
  char* base = nullptr;
  std::size_t bytes = 0;
};
Ring& ring() {
  static Ring* r = new Ring;  // never destroyed: see DeviceCache
  return *r;
}

int worker_count() {  // bench host, 537 MB device -> host: 2 threads 67 ms, 4 -> 36 ms, 8 -> 26 ms
  static const int n = [] {
    const char* e = std::getenv("GEMPE_DOWNLOAD_THREADS");
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    return e ? std::max(1, std::atoi(e)) : std::min(8, std::max(2, hw / 2));
  }();
  return n;
}

std::size_t chunk_bytes() {
  if (const char* env = std::getenv("GEMPE_DOWNLOAD_CHUNK")) return std::max<std::size_t>(256, std::strtoull(env, nullptr, 10));  // tests
  return 4u << 20;
}

// to_host: device -> ring (copy engine) -> host (threads); else host -> ring (threads) -> device (copy engine)
void staged_copy(void* host, void* dev, std::size_t bytes, cudaStream_t stream, bool to_host) {
  const int workers = worker_count();
  const int slots = 2 * workers;
  const std::size_t chunk = chunk_bytes();
  const cudaMemcpyKind kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
  if (bytes < 4 * chunk) {
    cuda_check(to_host ? cudaMemcpyAsync(host, dev, bytes, kind, stream) : cudaMemcpyAsync(dev, host, bytes, kind, stream),
               "host copy");
    cuda_check(cudaStreamSynchronize(stream), "host copy");
    return;
  }
  Ring& r = ring();
  std::lock_guard<std::mutex> lock(r.mutex);
  PhaseTimer timer;
  if (r.bytes < slots * chunk) {
    if (r.base) cudaFreeHost(r.base);
    r.base = nullptr;
    r.bytes = 0;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&r.base), slots * chunk, cudaHostAllocPortable), "pinned staging ring");
    r.bytes = slots * chunk;
    timer.lap("  host copy: pinned ring");
  }
  std::vector<cudaEvent_t> copied(slots);  // the copy engine is done with the slot's current chunk
  for (auto& ev : copied) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  const std::size_t chunks = (bytes + chunk - 1) / chunk;
  // per chunk: 0 nothing yet, 1 the first stage is done (to_host: copy issued; else: the threads filled the slot),
  // 2 the second stage is done (to_host: moved out of the slot; else: copy issued)
  std::vector<std::atomic<int>> stage(chunks);
  for (auto& s : stage) s.store(0);
  std::atomic<bool> failed{false};
  int device = 0;
  cuda_check(cudaGetDevice(&device), "cudaGetDevice");
  auto span = [&](std::size_t i, std::size_t& off, std::size_t& len) {
    off = i * chunk;
    len = std::min(chunk, bytes - off);
  };
  auto wait_stage = [&](std::size_t i, int want) {
    while (stage[i].load(std::memory_order_acquire) < want && !failed.load()) std::this_thread::yield();
    return !failed.load();
  };
  auto worker = [&](int w) {
    cudaSetDevice(device);
    for (std::size_t i = w; i < chunks; i += workers) {
      std::size_t off, len;
      span(i, off, len);
      char* slot = r.base + (i % slots) * chunk;
      if (to_host) {
        if (!wait_stage(i, 1)) return;
        if (cudaEventSynchronize(copied[i % slots]) != cudaSuccess) { failed.store(true); return; }
        std::memcpy(static_cast<char*>(host) + off, slot, len);
        stage[i].store(2, std::memory_order_release);
      } else {
        if (i >= static_cast<std::size_t>(slots)) {  // the slot's previous chunk must have left for the device
          if (!wait_stage(i - slots, 2)) return;
          if (cudaEventSynchronize(copied[i % slots]) != cudaSuccess) { failed.store(true); return; }
        }
        std::memcpy(slot, static_cast<const char*>(host) + off, len);
        stage[i].store(1, std::memory_order_release);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w) pool.emplace_back(worker, w);
  cudaError_t err = cudaSuccess;
  for (std::size_t i = 0; i < chunks && err == cudaSuccess; ++i) {
    std::size_t off, len;
    span(i, off, len);
    char* slot = r.base + (i % slots) * chunk;
    if (to_host) {
      if (i >= static_cast<std::size_t>(slots) && !wait_stage(i - slots, 2)) break;  // the slot has been moved out
      err = cudaMemcpyAsync(slot, static_cast<const char*>(dev) + off, len, kind, stream);
    } else {
      if (!wait_stage(i, 1)) break;  // the threads have filled the slot
      err = cudaMemcpyAsync(static_cast<char*>(dev) + off, slot, len, kind, stream);
    }
    if (err == cudaSuccess) err = cudaEventRecord(copied[i % slots], stream);
    if (err != cudaSuccess) failed.store(true);
    stage[i].store(to_host ? 1 : 2, std::memory_order_release);
  }
  if (err != cudaSuccess) failed.store(true);
  for (auto& t : pool) t.join();
  const cudaError_t sync = cudaStreamSynchronize(stream);  // the ring is free for the next transfer when this returns
  timer.lap(to_host ? "  host copy: device -> pageable" : "  host copy: pageable -> device");
  for (auto& ev : copied) cudaEventDestroy(ev);
  cuda_check(err, "host copy (staged)");
  cuda_check(sync, "host copy (staged)");
  if (failed.load()) throw cuda_error("host copy (staged): a copy failed");
}

}  // namespace

void download_to_pageable(void* dst, const void* src_dev, std::size_t bytes, cudaStream_t stream) {
  staged_copy(dst, const_cast<void*>(src_dev), bytes, stream, true);
}

void upload_from_pageable(void* dst_dev, const void* src, std::size_t bytes, cudaStream_t stream) {
  staged_copy(const_cast<void*>(src), dst_dev, bytes, stream, false);
}

bool is_pageable_host(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return attr.type == cudaMemoryTypeUnregistered;
}

}  // namespace gempe
