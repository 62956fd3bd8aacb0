// sm_100a kernels of the GEMPE round.  No tensor cores: the round is an HBM-bound sparse row gather plus
// a per-vertex reduction.  Citations are relative to /root/reference/proj.
//
//   hash_build / probe        bit-packed direct-mapped edge filter  (hash_set.cpp:9-34, hash_set.hpp:28-30)
//   sample                    one thread per sample stream          (sampler.cpp:7-31, engine.cpp:227-237)
//   scan / scatter / sort     bucket the accepted samples by PARTNER so the partner-side term of
//                             add_pair (engine.cpp:68-72) becomes a gather instead of an atomic scatter
//   gather                    per work item (vertex or hub slice): pair_distance + parabola_impl + add_pair
//                             for every row it touches, warp-shuffle reduction, fused x = y/z update
//                             (engine.cpp:45-73, 253-276, sigmoid.hpp:88-101, histogram.hpp:24-29)
#include "kernels.hpp"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "device_fns.cuh"

namespace gempe {

namespace {

constexpr int kThreads = 256;
constexpr int kPartThreads = 512;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool is_local(const Ownership& o, std::uint32_t v) {
  return o.world == 1 || (v / o.block_rows) % o.world == o.rank;
}

__device__ __forceinline__ bool hash_test(const std::uint32_t* __restrict__ words, std::uint32_t mask,
                                          std::uint32_t n, std::uint32_t i, std::uint32_t j) {
  const std::uint32_t h = pair_hash(i, j, n, mask);
  return (__ldg(words + (h >> 5)) >> (h & 31u)) & 1u;
}

// Same answer through the summary bitmap (bit g = "some cell of group g is set", kSummaryGroup cells per group): a
// sparse table that does not fit L2 is consulted only for the minority of probes whose group is occupied.
constexpr int kSummaryShift = kHashSummaryShift;
__device__ __forceinline__ bool hash_test(const std::uint32_t* __restrict__ words,
                                          const std::uint32_t* __restrict__ summary, std::uint32_t mask,
                                          std::uint32_t n, std::uint32_t i, std::uint32_t j) {
  const std::uint32_t h = pair_hash(i, j, n, mask);
  if (summary) {
    const std::uint32_t g = h >> kSummaryShift;
    if (!((__ldg(summary + (g >> 5)) >> (g & 31u)) & 1u)) return false;
  }
  return (__ldg(words + (h >> 5)) >> (h & 31u)) & 1u;
}

// ---------------------------------------------------------------------------------- hash set

__global__ void hash_build_kernel(const std::uint32_t* __restrict__ src, const std::uint32_t* __restrict__ dst,
                                  std::uint64_t m, std::uint32_t n, std::uint32_t mask,
                                  std::uint32_t* __restrict__ words) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t e = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += stride) {
    const std::uint32_t i = src[e], j = dst[e];
    const std::uint32_t h0 = pair_hash(i, j, n, mask), h1 = pair_hash(j, i, n, mask);
    atomicOr(words + (h0 >> 5), 1u << (h0 & 31u));
    atomicOr(words + (h1 >> 5), 1u << (h1 & 31u));
  }
}

// number of set cells (decides whether a summary pays: wrapping pair_hash aliases heavily for large n, so the table
// can be far emptier than 2m cells)
__global__ void hash_popcount_kernel(const std::uint32_t* __restrict__ words, std::uint64_t nwords,
                                     unsigned long long* __restrict__ total) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  unsigned long long mine = 0;
  for (std::uint64_t w = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < nwords; w += stride) {
    mine += __popc(words[w]);
  }
  for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(kFull, mine, off);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, mine);
}

// summary word s covers table words 4s .. 4s+3: bit 8q + k = any of bits 4k .. 4k+3 of word 4s + q
__global__ void hash_summary_kernel(const std::uint32_t* __restrict__ words, std::uint64_t nsummary,
                                    std::uint32_t* __restrict__ summary) {
  static_assert(kSummaryShift == 2, "layout below assumes 4 cells per summary bit");
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t sidx = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; sidx < nsummary; sidx += stride) {
    const uint4 w = *reinterpret_cast<const uint4*>(words + 4 * sidx);
    const std::uint32_t in[4] = {w.x, w.y, w.z, w.w};
    std::uint32_t out = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int k = 0; k < 8; ++k) out |= ((in[q] >> (4 * k)) & 0xfu ? 1u : 0u) << (8 * q + k);
    }
    summary[sidx] = out;
  }
}

__global__ void validate_edges_kernel(const std::uint32_t* __restrict__ src, const std::uint32_t* __restrict__ dst,
                                      std::uint64_t m, std::uint32_t n, std::uint32_t* __restrict__ flags) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  std::uint32_t bad = 0;
  for (std::uint64_t e = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += stride) {
    const std::uint32_t i = src[e], j = dst[e];
    if (i >= n || j >= n) bad |= 1u;
    else if (i == j) bad |= 2u;
  }
  if (bad) atomicOr(flags, bad);
}

__global__ void probe_kernel(const std::uint32_t* __restrict__ words, std::uint32_t mask, std::uint32_t n,
                             const std::uint32_t* __restrict__ i, const std::uint32_t* __restrict__ j,
                             std::uint64_t count, std::uint8_t* __restrict__ out) {
  const std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < count) out[t] = hash_test(words, mask, n, i[t], j[t]) ? 1 : 0;
}

// ---------------------------------------------------------------------------------- construction on the device

// random_relabel applied to the edge arrays (graph.cpp:199-204): ids -> forward[ids], in place
__global__ void relabel_apply_kernel(std::uint32_t* __restrict__ src, std::uint32_t* __restrict__ dst, std::uint64_t m,
                                     const std::uint32_t* __restrict__ forward) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t e = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += stride) {
    src[e] = __ldg(forward + src[e]);
    dst[e] = __ldg(forward + dst[e]);
  }
}

__global__ void degree_count_kernel(const std::uint32_t* __restrict__ src, const std::uint32_t* __restrict__ dst,
                                    std::uint64_t m, std::uint32_t* __restrict__ deg) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t e = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += stride) {
    atomicAdd(deg + src[e], 1u);
    atomicAdd(deg + dst[e], 1u);
  }
}

// both-direction CSR fill; the order inside a row is whatever the atomics give (the host build is used when a
// reproducible order is asked for)
__global__ void csr_fill_kernel(const std::uint32_t* __restrict__ src, const std::uint32_t* __restrict__ dst, std::uint64_t m,
                                const std::uint32_t* __restrict__ rowptr, std::uint32_t* __restrict__ cursor,
                                std::uint32_t* __restrict__ nbr, std::uint32_t* __restrict__ eid_role,
                                std::uint32_t* __restrict__ csr_src) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t e = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m; e += stride) {
    const std::uint32_t a = src[e], b = dst[e];
    const std::uint32_t p0 = rowptr[a] + atomicAdd(cursor + a, 1u);
    const std::uint32_t p1 = rowptr[b] + atomicAdd(cursor + b, 1u);
    nbr[p0] = b;
    nbr[p1] = a;
    if (eid_role) {
      eid_role[p0] = static_cast<std::uint32_t>(2 * e);
      eid_role[p1] = static_cast<std::uint32_t>(2 * e + 1);
      csr_src[p0] = a;
      csr_src[p1] = b;
    }
  }
}

// ---------------------------------------------------------------------------------- sampler

// PER_VERTEX_K: slot t belongs to anchor t / k.  The slot count fits 32 bits (checked when the context is created), so
// this is one 32-bit division instead of the 64-bit software routine
__device__ __forceinline__ std::uint32_t slot_anchor(std::uint64_t t, std::uint32_t k) {
  return static_cast<std::uint32_t>(t) / k;
}

// One sample stream: replays expand_seed32(seed, iter, unit, draw) followed by the LCG "advance, then use" loop
// of sample_non_edges (reference mode), or a Philox4x32-10 stream.  Returns the accepted partner.
__device__ __forceinline__ std::uint32_t sample_slot(const SampleArgs& a, std::uint64_t t, std::uint32_t& anchor,
                                                     std::uint32_t& draws) {
  std::uint64_t unit, draw;
  if (a.neg_mode == 0) {
    anchor = __ldg(a.csr_src + t);
    const std::uint32_t er = __ldg(a.eid_role + t);
    unit = er >> 1;
    draw = er & 1u;
  } else {
    anchor = slot_anchor(t, a.k);
    unit = anchor;
    draw = t - static_cast<std::uint64_t>(anchor) * a.k;
  }
  // the round's index may live on the device (a queued run): the stream base follows it
  const std::uint64_t iter = a.iter + (a.iter_dev ? static_cast<std::uint64_t>(*a.iter_dev) : 0ull);
  const std::uint64_t stream_base = a.iter_dev ? (a.rng == 0 ? mix(a.seed, iter) : a.seed) : a.stream_base;
  if (a.rng == 0) {
    std::uint32_t s = static_cast<std::uint32_t>(mix(mix(stream_base, unit), draw) >> 16);
    for (int tries = 0; tries < kMaxRetries; ++tries) {
      s = s * kLcgMul + 1u;
      ++draws;
      const std::uint32_t g = uniform_index(s, a.n);
      if (g == anchor) continue;
      if (hash_test(a.hash_words, a.hash_summary, a.hash_mask, a.n, anchor, g)) continue;
      return g;
    }
  } else {
    const std::uint64_t slot = a.neg_mode == 0 ? ((unit << 1) | draw) : t;
    for (int tries = 0; tries < kMaxRetries; tries += 4) {
      std::uint32_t ctr[4] = {static_cast<std::uint32_t>(slot), static_cast<std::uint32_t>(slot >> 32),
                              static_cast<std::uint32_t>(tries >> 2), static_cast<std::uint32_t>(iter)};
      philox4x32(ctr, static_cast<std::uint32_t>(stream_base), static_cast<std::uint32_t>(stream_base >> 32));
      for (int q = 0; q < 4; ++q) {
        ++draws;
        const std::uint32_t g = static_cast<std::uint32_t>((static_cast<std::uint64_t>(ctr[q]) * a.n) >> 32);
        if (g == anchor) continue;
        if (hash_test(a.hash_words, a.hash_summary, a.hash_mask, a.n, anchor, g)) continue;
        return g;
      }
    }
  }
  // near_complete_graph_error (sampler.cpp:18-21); keep memory-safe output
  atomicOr(a.status + kStatRetryCap, 1u);
  return anchor + 1 < a.n ? anchor + 1 : 0;
}

// Q independent streams per thread (reference LCG mode only): the draw of every open stream is made, then the probes
// of all of them are issued before any answer is consumed -- the chain seed -> draw -> summary word -> table word is
// latency, and one chain per thread leaves the memory system idle (the sampling kernel ran at 40 % issue activity).
// Same streams, same draws, same partners as sample_slot; `draws` is the sum over the Q streams.
template <int Q>
__device__ __forceinline__ void sample_slots_lcg(const SampleArgs& a, const std::uint64_t (&t)[Q], const bool (&on)[Q],
                                                 std::uint32_t (&anchor)[Q], std::uint32_t (&partner)[Q],
                                                 std::uint32_t& draws) {
  const std::uint64_t iter = a.iter + (a.iter_dev ? static_cast<std::uint64_t>(*a.iter_dev) : 0ull);
  const std::uint64_t stream_base = a.iter_dev ? mix(a.seed, iter) : a.stream_base;
  std::uint32_t s[Q];
  bool open[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    open[q] = on[q];
    anchor[q] = 0;
    partner[q] = 0;
    s[q] = 0;
    if (!on[q]) continue;
    std::uint64_t unit, draw;
    if (a.neg_mode == 0) {
      anchor[q] = __ldg(a.csr_src + t[q]);
      const std::uint32_t er = __ldg(a.eid_role + t[q]);
      unit = er >> 1;
      draw = er & 1u;
    } else {
      anchor[q] = slot_anchor(t[q], a.k);
      unit = anchor[q];
      draw = t[q] - static_cast<std::uint64_t>(anchor[q]) * a.k;
    }
    s[q] = static_cast<std::uint32_t>(mix(mix(stream_base, unit), draw) >> 16);
  }
  for (int tries = 0; tries < kMaxRetries; ++tries) {
    std::uint32_t g[Q], h[Q];
    bool probe[Q], hit[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      probe[q] = false;
      g[q] = h[q] = 0;
      if (open[q]) {
        s[q] = s[q] * kLcgMul + 1u;
        ++draws;
        g[q] = uniform_index(s[q], a.n);
        probe[q] = g[q] != anchor[q];
        h[q] = pair_hash(anchor[q], g[q], a.n, a.hash_mask);
      }
    }
    if (a.hash_summary) {  // first the small "any cell of the group set" bitmap, all streams at once
      std::uint32_t sw[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) sw[q] = probe[q] ? __ldg(a.hash_summary + (h[q] >> (kSummaryShift + 5))) : 0u;
#pragma unroll
      for (int q = 0; q < Q; ++q) hit[q] = probe[q] && ((sw[q] >> ((h[q] >> kSummaryShift) & 31u)) & 1u);
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) hit[q] = probe[q];
    }
    {
      std::uint32_t tw[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) tw[q] = hit[q] ? __ldg(a.hash_words + (h[q] >> 5)) : 0u;
#pragma unroll
      for (int q = 0; q < Q; ++q) hit[q] = hit[q] && ((tw[q] >> (h[q] & 31u)) & 1u);
    }
    bool any = false;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (open[q] && probe[q] && !hit[q]) {
        partner[q] = g[q];
        open[q] = false;
      }
      any |= open[q];
    }
    if (!any) return;
  }
  // near_complete_graph_error (sampler.cpp:18-21); keep memory-safe output
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (open[q]) {
      atomicOr(a.status + kStatRetryCap, 1u);
      partner[q] = anchor[q] + 1 < a.n ? anchor[q] + 1 : 0;
    }
  }
}

// Total draw count (test hook / p-bar of the roofline formula).  Called by every thread of the block: one global
// atomic per block -- per-warp atomics on this single address serialise in L2 and dominated the sampling kernel.
__device__ __forceinline__ void add_draws(const SampleArgs& a, std::uint32_t draws) {
  __shared__ std::uint32_t block_draws;
  if (threadIdx.x == 0) block_draws = 0;
  __syncthreads();
  for (int off = 16; off > 0; off >>= 1) draws += __shfl_xor_sync(kFull, draws, off);
  if ((threadIdx.x & 31) == 0 && draws) atomicAdd(&block_draws, draws);
  __syncthreads();
  if (threadIdx.x == 0 && block_draws) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.status + kStatDrawsLo), static_cast<unsigned long long>(block_draws));
  }
}

// ---- bucketing by partner, method A (small n): one returning atomic per sample on the partner's counter, then
// scan + scatter.  Every array it touches at random (in_cnt, in_off) fits L2 for n up to a few million.
constexpr int kSampleIlp = 2;  // sample streams per thread (sample_slots_lcg)
__global__ void __launch_bounds__(kThreads, 6) sample_kernel(const SampleArgs a) {
  const std::uint64_t t0 = static_cast<std::uint64_t>(blockIdx.x) * (kThreads * kSampleIlp) + threadIdx.x;
  std::uint32_t draws = 0;
  std::uint64_t t[kSampleIlp];
  bool on[kSampleIlp];
  std::uint32_t anchor[kSampleIlp], partner[kSampleIlp];
#pragma unroll
  for (int q = 0; q < kSampleIlp; ++q) {
    t[q] = t0 + q * kThreads;
    on[q] = t[q] < a.slots;
  }
  if (a.rng == 0) {
    sample_slots_lcg<kSampleIlp>(a, t, on, anchor, partner, draws);
  } else {
#pragma unroll
    for (int q = 0; q < kSampleIlp; ++q)
      if (on[q]) partner[q] = sample_slot(a, t[q], anchor[q], draws);
  }
  // the returning atomics of all streams before any of their answers is stored
  std::uint32_t rank[kSampleIlp];
#pragma unroll
  for (int q = 0; q < kSampleIlp; ++q) {
    rank[q] = kNotLocal;
    if (on[q] && is_local(a.own, partner[q])) rank[q] = atomicAdd(a.in_cnt + partner[q], 1u);
  }
#pragma unroll
  for (int q = 0; q < kSampleIlp; ++q) {
    if (!on[q]) continue;
    if (a.in_stride) {  // slotted buckets: the arrival rank is the slot
      a.neg_own[t[q]] = partner[q];
      if (rank[q] == kNotLocal) continue;
      if (rank[q] < a.in_stride) {
        a.in_anchor[static_cast<std::size_t>(partner[q]) * a.in_stride + rank[q]] = anchor[q];
      } else {
        const std::uint32_t at = atomicAdd(a.spill_count, 1u);
        if (at < a.spill_capacity) a.spill[at] = make_uint2(partner[q], anchor[q]);
        else atomicOr(a.status + kStatExchangeOverflow, 1u);
      }
    } else {  // large graphs: both arrays are read once by later kernels and must not displace the counters / summary
      __stcs(a.neg_own + t[q], partner[q]);
      __stcs(a.in_rank + t[q], rank[q]);
    }
  }
  add_draws(a, draws);
}

// Slotted buckets, overflow side (rare: a partner drew more samples than its slots hold).  ONE block: leaves at once when
// nothing spilled; otherwise counts the spilled records per partner, scans the n counters with a running carry and
// groups the anchors by partner -- O(n + spill) work for one SM, the price of a round that overflowed.
__global__ void __launch_bounds__(1024) spill_index_kernel(const SpillIndexArgs a) {
  const std::uint32_t count = min(*a.spill_count, a.spill_capacity);
  if (count == 0) return;
  __shared__ std::uint32_t warp_tot[32];
  __shared__ std::uint32_t carry;
  for (std::uint32_t i = threadIdx.x; i < count; i += 1024) atomicAdd(a.cnt + a.spill[i].x, 1u);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (std::uint32_t base = 0; base < a.n; base += 1024) {
    const std::uint32_t i = base + threadIdx.x;
    const std::uint32_t v = i < a.n ? a.cnt[i] : 0u;
    std::uint32_t inc = v;
    for (int off = 1; off < 32; off <<= 1) {
      const std::uint32_t o = __shfl_up_sync(kFull, inc, off);
      if (lane >= off) inc += o;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const std::uint32_t w = warp_tot[lane];
      std::uint32_t winc = w;
      for (int off = 1; off < 32; off <<= 1) {
        const std::uint32_t o = __shfl_up_sync(kFull, winc, off);
        if (lane >= off) winc += o;
      }
      warp_tot[lane] = winc - w;
    }
    __syncthreads();
    const std::uint32_t excl = carry + warp_tot[warp] + inc - v;
    if (i < a.n) {
      a.off[i] = excl;
      a.cnt[i] = 0;  // becomes the placement cursor below, and is zero again afterwards
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.off[a.n] = carry;
  __syncthreads();
  for (std::uint32_t i = threadIdx.x; i < count; i += 1024) {
    const uint2 rec = a.spill[i];
    a.anchor[a.off[rec.x] + atomicAdd(a.cnt + rec.x, 1u)] = rec.y;
  }
  __syncthreads();
  for (std::uint32_t i = threadIdx.x; i < count; i += 1024) a.cnt[a.spill[i].x] = 0;
}

constexpr int kScatterIlp = 4;  // samples per thread: rank / partner -> offset -> store is a chain of dependent accesses
// blockIdx.y = part: the samples are walked gridDim.y times, each walk placing only the partners of one contiguous vertex
// range, so the window of in_anchor that receives random 4-byte stores (S * 4 bytes in all) stays in L2 while the index
// streams pass through (launch_scatter sizes the parts).  A window beyond L2 is written back half-filled and fetched
// again: 277 MB of DRAM writes for 84 MB of anchors on c4.
__global__ void __launch_bounds__(kThreads) scatter_kernel(const SampleArgs a, const std::uint32_t* __restrict__ in_off,
                                                           std::uint32_t* __restrict__ in_anchor, std::uint32_t part_rows) {
  const std::uint64_t t0 = static_cast<std::uint64_t>(blockIdx.x) * (kThreads * kScatterIlp) + threadIdx.x;
  const std::uint32_t lo = blockIdx.y * part_rows, hi = lo + part_rows;  // part_rows * gridDim.y >= n
  std::uint32_t rank[kScatterIlp], partner[kScatterIlp], off[kScatterIlp];
  bool mine[kScatterIlp];
#pragma unroll
  for (int q = 0; q < kScatterIlp; ++q) {
    const std::uint64_t t = t0 + q * kThreads;
    partner[q] = 0xffffffffu;
    if (t < a.slots) partner[q] = __ldcs(a.neg_own + t);  // read once per walk: must not push the window out of L2
  }
#pragma unroll
  for (int q = 0; q < kScatterIlp; ++q) {
    mine[q] = partner[q] >= lo && partner[q] < hi;  // 0xffffffff (no slot) is in no part: hi <= n + part_rows < 2^32
    rank[q] = mine[q] ? __ldcs(a.in_rank + t0 + q * kThreads) : kNotLocal;
    off[q] = mine[q] ? in_off[partner[q]] : 0u;
  }
#pragma unroll
  for (int q = 0; q < kScatterIlp; ++q) {
    if (mine[q] && rank[q] != kNotLocal) {
      const std::uint64_t t = t0 + q * kThreads;
      in_anchor[off[q] + rank[q]] = a.neg_mode == 0 ? __ldg(a.csr_src + t) : slot_anchor(t, a.k);
    }
  }
}

// ---- sharded sampling with an exchange step (world > 1): every rank samples ONLY the streams of the anchors it owns,
// packs (partner, anchor) records by the partner's owner rank, the ranks exchange the packed regions (one equal-split
// all-to-all over NVLink), and each rank buckets what it received.  Sampling work therefore scales with 1/world.
__global__ void __launch_bounds__(kThreads, 8) sample_pack_kernel(const SampleArgs a, const ExchangeArgs x) {
  const std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  std::uint32_t draws = 0;
  bool have = false;
  std::uint32_t partner = 0, anchor = 0, dest = 0;
  if (i < x.own_slots) {
    // own slot i -> global slot: ranges[c] = first global slot of the c-th owned block, prefix[c] = own slots before it
    std::uint32_t c = 0, hi = x.ranges;  // largest c with prefix[c] <= i
    while (hi - c > 1) {
      const std::uint32_t mid = (c + hi) >> 1;
      if (__ldg(x.prefix + mid) <= i) c = mid; else hi = mid;
    }
    const std::uint64_t t = x.first_slot[c] + (i - x.prefix[c]);
    partner = sample_slot(a, t, anchor, draws);
    __stcs(a.neg_own + t, partner);  // streamed: read again by the gather only
    dest = x.region_rows ? partner / x.region_rows : (partner / a.own.block_rows) % a.own.world;
    have = true;
  }
  add_draws(a, draws);
  // one global atomic per destination rank and BLOCK: ranks within the block come from shared counters
  extern __shared__ std::uint32_t sh_pack[];  // [regions] counts, then [regions] bases
  std::uint32_t* sh_cnt = sh_pack;
  std::uint32_t* sh_base = sh_pack + x.regions;
  for (std::uint32_t d = threadIdx.x; d < x.regions; d += blockDim.x) sh_cnt[d] = 0;
  __syncthreads();
  std::uint32_t local = 0;
  if (have) local = atomicAdd(sh_cnt + dest, 1u);
  __syncthreads();
  for (std::uint32_t d = threadIdx.x; d < x.regions; d += blockDim.x) {
    sh_base[d] = sh_cnt[d] ? atomicAdd(x.send_count + d, sh_cnt[d]) : 0u;
  }
  __syncthreads();
  if (have) {
    const std::uint32_t pos = sh_base[dest] + local;
    if (pos < x.capacity) {
      uint2* region = x.direct ? x.dest_region[dest] : x.send + static_cast<std::size_t>(dest) * x.capacity;
      if (x.direct) region[pos] = make_uint2(partner, anchor);
      else __stcs(region + pos, make_uint2(partner, anchor));
    } else {
      const std::uint32_t at = x.spill ? atomicAdd(x.spill_count, 1u) : 0xffffffffu;
      if (at < x.spill_capacity) x.spill[at] = make_uint2(partner, anchor);
      else atomicOr(a.status + kStatExchangeOverflow, 1u);
    }
  }
  if (x.direct) __threadfence_system();  // peer stores are performed before the grid retires
}

// direct exchange: tell every destination how many records this rank left in its region there
__global__ void publish_counts_kernel(const ExchangeArgs x) {
  const std::uint32_t d = threadIdx.x;
  if (d < x.regions) *x.dest_count[d] = x.send_count[d];
  __threadfence_system();
}

// received records -> per-partner counts and arrival ranks.  blockIdx.y = source region: the regions are walked one
// after another, so with contiguous vertex ranges the counters touched at any time are one range's (L2-resident).
// kRecIlp records per thread: both kernels are chains of dependent memory operations (record -> counter / offset ->
// store) at a few per cent issue utilisation, so independent chains per thread are what fills the memory system
constexpr int kRecIlp = 4;
__global__ void __launch_bounds__(kThreads) count_records_kernel(const ExchangeArgs x, std::uint32_t* __restrict__ in_cnt,
                                                                 std::uint32_t* __restrict__ rec_rank) {
  const std::uint32_t from = blockIdx.y, count = min(x.recv_count[from], x.capacity);
  const std::uint32_t j0 = blockIdx.x * (kThreads * kRecIlp) + threadIdx.x;
  const std::size_t base = static_cast<std::size_t>(from) * x.capacity;
  std::uint32_t partner[kRecIlp], rank[kRecIlp];
#pragma unroll
  for (int q = 0; q < kRecIlp; ++q) {
    const std::uint32_t j = j0 + q * kThreads;
    partner[q] = j < count ? __ldcs(reinterpret_cast<const std::uint32_t*>(x.recv + base + j)) : 0xffffffffu;
  }
#pragma unroll
  for (int q = 0; q < kRecIlp; ++q) rank[q] = partner[q] != 0xffffffffu ? atomicAdd(in_cnt + partner[q], 1u) : 0u;
#pragma unroll
  for (int q = 0; q < kRecIlp; ++q) {
    const std::uint32_t j = j0 + q * kThreads;
    if (j < count) __stcs(rec_rank + base + j, rank[q]);
  }
}

__global__ void __launch_bounds__(kThreads) scatter_records_kernel(const ExchangeArgs x,
                                                                   const std::uint32_t* __restrict__ rec_rank,
                                                                   const std::uint32_t* __restrict__ in_off,
                                                                   std::uint32_t* __restrict__ in_anchor) {
  const std::uint32_t from = blockIdx.y, count = min(x.recv_count[from], x.capacity);
  const std::uint32_t j0 = blockIdx.x * (kThreads * kRecIlp) + threadIdx.x;
  const std::size_t base = static_cast<std::size_t>(from) * x.capacity;
  uint2 rec[kRecIlp];
  std::uint32_t rank[kRecIlp], off[kRecIlp];
#pragma unroll
  for (int q = 0; q < kRecIlp; ++q) {
    const std::uint32_t j = j0 + q * kThreads;
    rec[q] = make_uint2(0xffffffffu, 0u);
    rank[q] = 0;
    if (j < count) {
      rec[q] = __ldcs(x.recv + base + j);  // streams: the window of in_anchor they scatter into is what L2 should keep
      rank[q] = __ldcs(rec_rank + base + j);
    }
  }
#pragma unroll
  for (int q = 0; q < kRecIlp; ++q) off[q] = rec[q].x != 0xffffffffu ? in_off[rec[q].x] : 0u;
#pragma unroll
  for (int q = 0; q < kRecIlp; ++q) {
    if (rec[q].x != 0xffffffffu) in_anchor[off[q] + rank[q]] = rec[q].y;
  }
}

// the spill area (see ExchangeArgs): same two steps, grid-stride, normally zero records
__global__ void __launch_bounds__(kThreads) count_spill_kernel(const ExchangeArgs x, std::uint32_t* __restrict__ in_cnt,
                                                               std::uint32_t* __restrict__ spill_rank) {
  const std::uint32_t count = min(*x.spill_count, x.spill_capacity);
  for (std::uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
    spill_rank[j] = atomicAdd(in_cnt + x.spill[j].x, 1u);
  }
}
__global__ void __launch_bounds__(kThreads) scatter_spill_kernel(const ExchangeArgs x,
                                                                 const std::uint32_t* __restrict__ spill_rank,
                                                                 const std::uint32_t* __restrict__ in_off,
                                                                 std::uint32_t* __restrict__ in_anchor) {
  const std::uint32_t count = min(*x.spill_count, x.spill_capacity);
  for (std::uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
    const uint2 rec = x.spill[j];
    in_anchor[in_off[rec.x] + spill_rank[j]] = rec.y;
  }
}

// ---- bucketing by partner, method B (large n): two-level counting sort with streaming traffic only.
//   1. sample_count_kernel: persistent blocks sample their slots (grid-stride tiles) and histogram the partners'
//      COARSE buckets (partner >> shift, <= 8192 buckets) in shared memory; one histogram row per block.
//   2. bucket_scan kernels: column scan over the blocks (base of every (block, bucket) run) + bucket offsets.
//   3. partition_kernel: same tiles; (partner, anchor) records go to their run of the coarse bucket, positions from
//      shared-memory cursors -- no global atomics, writes land in a few hundred open runs.
//   4. bucket_finalize_kernel: one block per coarse bucket counts its vertices in shared memory, scans, writes
//      in_off for its vertex range and places the anchors; random writes stay inside the bucket's window (L2).
__global__ void __launch_bounds__(kPartThreads) sample_count_kernel(const SampleArgs a, const PartitionArgs p) {
  extern __shared__ std::uint32_t sh_cnt[];
  for (std::uint32_t b = threadIdx.x; b < p.buckets; b += kPartThreads) sh_cnt[b] = 0;
  __syncthreads();
  std::uint32_t draws = 0;
  for (std::uint64_t base = static_cast<std::uint64_t>(blockIdx.x) * kPartThreads; base < a.slots;
       base += static_cast<std::uint64_t>(gridDim.x) * kPartThreads) {
    const std::uint64_t t = base + threadIdx.x;
    if (t < a.slots) {
      std::uint32_t anchor;
      const std::uint32_t partner = sample_slot(a, t, anchor, draws);
      a.neg_own[t] = partner;
      if (is_local(a.own, partner)) atomicAdd(&sh_cnt[partner >> p.shift], 1u);
    }
  }
  add_draws(a, draws);
  __syncthreads();
  for (std::uint32_t b = threadIdx.x; b < p.buckets; b += kPartThreads) {
    p.block_hist[static_cast<std::size_t>(blockIdx.x) * p.buckets + b] = sh_cnt[b];
  }
}

__global__ void bucket_column_scan_kernel(const PartitionArgs p, std::uint32_t blocks) {
  const std::uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= p.buckets) return;
  std::uint32_t run = 0;
  for (std::uint32_t k = 0; k < blocks; ++k) {
    const std::size_t at = static_cast<std::size_t>(k) * p.buckets + b;
    const std::uint32_t c = p.block_hist[at];
    p.block_hist[at] = run;
    run += c;
  }
  p.bucket_off[b] = run;  // bucket total, turned into an offset by bucket_offsets_kernel
}

__global__ void bucket_offsets_kernel(const PartitionArgs p, std::uint32_t* __restrict__ in_off, std::uint32_t n) {
  // single block of 1024 threads: in-place exclusive scan of bucket_off[0..buckets) with a running carry
  __shared__ std::uint32_t warp_tot[32];
  __shared__ std::uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (std::uint32_t base = 0; base < p.buckets; base += 1024) {
    const std::uint32_t i = base + threadIdx.x;
    const std::uint32_t v = i < p.buckets ? p.bucket_off[i] : 0;
    std::uint32_t inc = v;
    for (int off = 1; off < 32; off <<= 1) {
      const std::uint32_t o = __shfl_up_sync(kFull, inc, off);
      if (lane >= off) inc += o;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const std::uint32_t w = warp_tot[lane];
      std::uint32_t winc = w;
      for (int off = 1; off < 32; off <<= 1) {
        const std::uint32_t o = __shfl_up_sync(kFull, winc, off);
        if (lane >= off) winc += o;
      }
      warp_tot[lane] = winc - w;
    }
    __syncthreads();
    const std::uint32_t excl = carry + warp_tot[warp] + inc - v;
    if (i < p.buckets) p.bucket_off[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.bucket_off[p.buckets] = carry;
    in_off[n] = carry;
  }
}

// One partition block replays the tile sets of several counting blocks one after another (rows row, row + gridDim,
// ...), so that only gridDim.x * buckets runs are open at any time: with one block per SM their partially written
// sectors (a few tens of MB) stay in L2 until they are complete.
__global__ void __launch_bounds__(1024) partition_kernel(const SampleArgs a, const PartitionArgs p) {
  extern __shared__ std::uint32_t sh_cur[];
  for (std::uint32_t row = blockIdx.x; row < p.grid; row += gridDim.x) {
    __syncthreads();
    for (std::uint32_t b = threadIdx.x; b < p.buckets; b += blockDim.x) {
      sh_cur[b] = p.bucket_off[b] + p.block_hist[static_cast<std::size_t>(row) * p.buckets + b];
    }
    __syncthreads();
    // the counting block used kPartThreads-wide tiles at row*kPartThreads + j*grid*kPartThreads: the two halves of
    // this 1024-thread block take alternate tiles of the row
    constexpr int kIlp = 4;  // independent tiles in flight per thread
    const std::uint64_t stride = blockDim.x / kPartThreads;
    for (std::uint64_t tile = threadIdx.x / kPartThreads;; tile += stride * kIlp) {
      if ((static_cast<std::uint64_t>(row) + tile * p.grid) * kPartThreads >= a.slots) break;
      std::uint64_t t[kIlp];
      std::uint32_t partner[kIlp];
#pragma unroll
      for (int q = 0; q < kIlp; ++q) {
        t[q] = (static_cast<std::uint64_t>(row) + (tile + q * stride) * p.grid) * kPartThreads + threadIdx.x % kPartThreads;
        partner[q] = t[q] < a.slots ? a.neg_own[t[q]] : 0xffffffffu;
      }
#pragma unroll
      for (int q = 0; q < kIlp; ++q) {
        if (t[q] < a.slots && is_local(a.own, partner[q])) {
          const std::uint32_t anchor = a.neg_mode == 0 ? __ldg(a.csr_src + t[q]) : slot_anchor(t[q], a.k);
          const std::uint32_t pos = atomicAdd(&sh_cur[partner[q] >> p.shift], 1u);
          p.records[pos] = make_uint2(partner[q], anchor);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kPartThreads) bucket_finalize_kernel(const PartitionArgs p, std::uint32_t n,
                                                                       std::uint32_t* __restrict__ in_off,
                                                                       std::uint32_t* __restrict__ in_anchor) {
  extern __shared__ std::uint32_t sh_v[];  // per-vertex counts, then cursors; [vb]
  __shared__ std::uint32_t warp_tot[kPartThreads / 32];
  const std::uint32_t b = blockIdx.x, vb = 1u << p.shift, vmask = vb - 1;
  const std::uint32_t lo = p.bucket_off[b], hi = p.bucket_off[b + 1];
  for (std::uint32_t v = threadIdx.x; v < vb; v += kPartThreads) sh_v[v] = 0;
  __syncthreads();
  for (std::uint32_t i = lo + threadIdx.x; i < hi; i += kPartThreads) atomicAdd(&sh_v[p.records[i].x & vmask], 1u);
  __syncthreads();
  // block-wide exclusive scan of sh_v[0..vb): each thread owns a contiguous chunk
  const std::uint32_t chunk = (vb + kPartThreads - 1) / kPartThreads;
  const std::uint32_t first = threadIdx.x * chunk;
  std::uint32_t local = 0;
  for (std::uint32_t q = 0; q < chunk; ++q) local += first + q < vb ? sh_v[first + q] : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t inc = local;
  for (int off = 1; off < 32; off <<= 1) {
    const std::uint32_t o = __shfl_up_sync(kFull, inc, off);
    if (lane >= off) inc += o;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  std::uint32_t run = inc - local;
  for (int w = 0; w < warp; ++w) run += warp_tot[w];
  for (std::uint32_t q = 0; q < chunk; ++q) {
    if (first + q < vb) {
      const std::uint32_t c = sh_v[first + q];
      sh_v[first + q] = run;  // cursor of this vertex inside the bucket
      const std::uint64_t v = static_cast<std::uint64_t>(b) * vb + first + q;
      if (v < n) in_off[v] = lo + run;
      run += c;
    }
  }
  __syncthreads();
  for (std::uint32_t i = lo + threadIdx.x; i < hi; i += kPartThreads) {
    const uint2 rec = p.records[i];
    in_anchor[lo + atomicAdd(&sh_v[rec.x & vmask], 1u)] = rec.y;
  }
}

__global__ void unpermute_kernel(const std::uint32_t* __restrict__ neg_own, const std::uint32_t* __restrict__ eid_role,
                                 std::uint64_t slots, std::uint32_t* __restrict__ out) {
  const std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < slots) out[eid_role[t]] = neg_own[t];
}

// One warp per vertex: rank-sort of the (small, Poisson-sized) incoming bucket, in place via registers for
// buckets up to 32*kSortRegs entries; larger buckets fall back to an O(len^2) global pass.
#ifndef GEMPE_GRAB
#define GEMPE_GRAB 4
#endif
constexpr int kGrab = GEMPE_GRAB;  // work items claimed per atomic by a persistent warp
constexpr int kSortRegs = 8;
__global__ void __launch_bounds__(kThreads) sort_buckets_kernel(const std::uint32_t* __restrict__ in_off,
                                                                std::uint32_t* __restrict__ in_anchor, std::uint32_t n) {
  const std::uint32_t v = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= n) return;
  const std::uint32_t lo = in_off[v], len = in_off[v + 1] - lo;
  if (len < 2) return;
  std::uint32_t* b = in_anchor + lo;
  if (len <= 32u * kSortRegs) {
    std::uint32_t val[kSortRegs], pos[kSortRegs];
#pragma unroll
    for (int q = 0; q < kSortRegs; ++q) {
      const std::uint32_t i = lane + 32u * q;
      val[q] = i < len ? b[i] : 0xffffffffu;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kSortRegs; ++q) {
      const std::uint32_t i = lane + 32u * q;
      std::uint32_t p = 0;
      if (i < len) {
        for (std::uint32_t j = 0; j < len; ++j) {
          const std::uint32_t o = b[j];
          p += (o < val[q]) || (o == val[q] && j < i);
        }
      }
      pos[q] = p;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kSortRegs; ++q) {
      if (lane + 32u * q < len) b[pos[q]] = val[q];
    }
  } else {
    // odd-even transposition sort by the warp, in place (rare: only heavy-tailed buckets)
    for (std::uint32_t pass = 0; pass < len; ++pass) {
      for (std::uint32_t i = (pass & 1u) + 2u * lane; i + 1 < len; i += 64u) {
        const std::uint32_t x = b[i], y = b[i + 1];
        if (x > y) {
          b[i] = y;
          b[i + 1] = x;
        }
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------------- exclusive scan

constexpr int kScanTile = 4096;  // 256 threads x 16

__global__ void __launch_bounds__(kThreads) scan_tile_sums_kernel(const std::uint32_t* __restrict__ in, std::uint32_t n,
                                                                  std::uint32_t* __restrict__ tile_sum) {
  __shared__ std::uint32_t warp_sum[kThreads / 32];
  const std::uint32_t base = blockIdx.x * kScanTile;
  std::uint32_t s = 0;
  for (int q = 0; q < 16; ++q) {
    const std::uint32_t i = base + q * kThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    std::uint32_t t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += warp_sum[w];
    tile_sum[blockIdx.x] = t;
  }
}

__global__ void scan_tile_offsets_kernel(std::uint32_t* __restrict__ tile_sum, std::uint32_t tiles) {
  // single block of 1024 threads, in-place exclusive scan with a running carry
  __shared__ std::uint32_t warp_tot[32];
  __shared__ std::uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (std::uint32_t base = 0; base < tiles; base += 1024) {
    const std::uint32_t i = base + threadIdx.x;
    const std::uint32_t v = i < tiles ? tile_sum[i] : 0;
    std::uint32_t inc = v;
    for (int off = 1; off < 32; off <<= 1) {
      const std::uint32_t o = __shfl_up_sync(kFull, inc, off);
      if (lane >= off) inc += o;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      std::uint32_t w = warp_tot[lane], winc = w;
      for (int off = 1; off < 32; off <<= 1) {
        const std::uint32_t o = __shfl_up_sync(kFull, winc, off);
        if (lane >= off) winc += o;
      }
      warp_tot[lane] = winc - w;  // exclusive warp offsets
    }
    __syncthreads();
    const std::uint32_t excl = carry + warp_tot[warp] + inc - v;
    if (i < tiles) tile_sum[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_sum[tiles] = carry;
}

__global__ void __launch_bounds__(kThreads) scan_apply_kernel(std::uint32_t* __restrict__ in, std::uint32_t n,
                                                              const std::uint32_t* __restrict__ tile_off,
                                                              std::uint32_t* __restrict__ out, bool clear_input) {
  __shared__ std::uint32_t warp_tot[kThreads / 32];
  const std::uint32_t base = blockIdx.x * kScanTile + threadIdx.x * 16;
  std::uint32_t v[16], s = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    v[q] = base + q < n ? in[base + q] : 0;
    s += v[q];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t inc = s;
  for (int off = 1; off < 32; off <<= 1) {
    const std::uint32_t o = __shfl_up_sync(kFull, inc, off);
    if (lane >= off) inc += o;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  std::uint32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += warp_tot[w];
  std::uint32_t run = tile_off[blockIdx.x] + woff + inc - s;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (base + q < n) {
      out[base + q] = run;
      if (clear_input) in[base + q] = 0;  // the counters are ready for the next round
    }
    run += v[q];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_off[gridDim.x];
}

// ---------------------------------------------------------------------------------- initial coordinates

__global__ void init_coords_kernel(float* __restrict__ x, std::uint32_t n, std::uint32_t dim, std::uint32_t ld,
                                   int rule, std::uint64_t state0, double stddev) {
  const std::uint64_t total = static_cast<std::uint64_t>(n) * ld;
  const std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const std::uint32_t v = static_cast<std::uint32_t>(t / ld), c = static_cast<std::uint32_t>(t % ld);
  float out = 0.0f;
  if (c < dim) {
    const std::uint64_t i = static_cast<std::uint64_t>(v) * dim + c;
    if (rule == 0) {
      // SplitMix::next_double of the i-th draw (rng.hpp:48-56): the stream is a counter, state0 + (i+1) golden
      const std::uint64_t z = sm64(state0 + i * kGolden64);
      out = __double2float_rn(__ull2double_rn(z >> 11) * 0x1.0p-53);
    } else if (rule == 1) {
      const std::uint64_t z = sm64(state0 + i * kGolden64);
      out = __double2float_rn(2.0 * (__ull2double_rn(z >> 11) * 0x1.0p-53) - 1.0);
    } else {
      const std::uint64_t z0 = sm64(state0 + (2 * i) * kGolden64), z1 = sm64(state0 + (2 * i + 1) * kGolden64);
      const double u0 = (__ull2double_rn(z0 >> 11) + 1.0) * 0x1.0p-53, u1 = __ull2double_rn(z1 >> 11) * 0x1.0p-53;
      out = __double2float_rn(stddev * sqrt(-2.0 * log(u0)) * cospi(2.0 * u1));
    }
  }
  x[t] = out;
}

// ---------------------------------------------------------------------------------- gather + update

struct SmemTables {
  double erf[65];
  double ratio[65];
};

// largest s in [0,15] with knots[s] <= x (piecewise.hpp:36-47) for x >= knots[0]
__device__ __forceinline__ int segment_of(const double* __restrict__ knots, double x) {
  int s = x >= knots[8] ? 8 : 0;
  s += x >= knots[s + 4] ? 4 : 0;
  s += x >= knots[s + 2] ? 2 : 0;
  s += x >= knots[s + 1] ? 1 : 0;
  return s;
}

__device__ __forceinline__ double quad_eval(const double* __restrict__ t, double x) {
  const int s = segment_of(t, x);
  return (t[17 + s] * x + t[33 + s]) * x + t[49 + s];
}

__device__ __forceinline__ double tail_series(double x) {  // sigmoid.hpp:41-44
  const double r = 1.0 / (x * x);
  const double series = 1.0 + r * (-0.5 + r * (0.75 + r * (-1.875 + 6.5625 * r)));
  return x * 1.77245385090551602729816748334 / series;
}

// G(x) = e^{-x^2} / erfc(x): FastMath::gauss_erfc_ratio (piecewise.hpp:72-79) or ExactMath (sigmoid.hpp:61-65)
__device__ __forceinline__ double gauss_erfc_ratio(double x, int exact, const SmemTables& tab) {
  if (exact) return x <= 6.0 ? exp(-x * x) / erfc(x) : tail_series(x);
  if (x >= -1.0) return x > 8.0 ? tail_series(x) : quad_eval(tab.ratio, x);
  if (x < -6.0) return 0.0;
  // 1 - erf_table(x) with the odd-mirrored table: erf_table(x) = -q(-x) for x < 0
  return exp(-x * x) / (1.0 + quad_eval(tab.erf, -x));
}

// parabola_impl + the scalar part of add_pair (sigmoid.hpp:88-101, engine.cpp:56-61):
//   wf = float(w),  sf = delta > 0 ? float(max(d_target, 0) / delta) : 0,  both 0 when !(w > 0).
__device__ __forceinline__ void pair_terms(double delta, bool is_edge, const RoundMath& m, const SmemTables& tab,
                                           float& wf, float& sf) {
  const double dm = delta - m.mu;
  const double u = dm * m.inv_sqrt2_sigma;
  const double g = gauss_erfc_ratio(is_edge ? u : -u, m.exact, tab);
  const double sg = is_edge ? -g : g;
  const double w = m.A * g * g + m.B * dm * sg;
  if (!(w > 0.0)) {
    wf = 0.0f;
    sf = 0.0f;
    return;
  }
  wf = static_cast<float>(w);
  // d_target = delta + sign C g / w  =>  max(d_target,0)/delta = max(delta w + sign C g, 0) / (delta w)
  const double dw = delta * w;
  const double num = dw + m.C * sg;
  sf = (delta > 0.0 && num > 0.0) ? static_cast<float>(num / dw) : 0.0f;
}

// ---- fp32 evaluation of the same formulas (default, non-PRECISE kernels) -------------------------------------
// delta is only known to ~3e-7 in this mode, so the scalar chain is carried in fp32 as well (relative error
// ~1e-6 on wf and sf, two orders below the 1e-4 parity bar); tallies stay exact through the double recheck.
struct SmemTablesF {
  float4 cell[kTableF32Entries];  // ratio cells, then erf segments: {a, b, c, 0} (kernels.hpp)
};
struct RoundMathF {
  float mu, inv_sqrt2_sigma, A, B, C;
};

// MUFU approximations without the denormal guards the intrinsics carry (arguments and results here are far from the
// denormal range; a flushed 1e-39 changes nothing at the 1e-4 bar)
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float exp_approx(float x) {  // e^x
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * 1.4426950408889634f));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {  // relative error 2^-23; the tallies are rechecked in double
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// the ratio table's quadratic at x in [-1, 8]: the cell index IS the segment search (a value within rounding of a knot
// may land in the neighbouring segment; the fit is continuous across knots)
__device__ __forceinline__ float ratio_table_f(const SmemTablesF& tab, float x) {
  const int i = min(max(__float2int_rd(fmaf(x, 20.0f, 20.0f)), 0), kRatioCells - 1);
  const float4 q = tab.cell[i];
  return fmaf(fmaf(q.x, x, q.y), x, q.z);
}
// the erf table's quadratic at x in [0, 6]
__device__ __forceinline__ float erf_table_f(const SmemTablesF& tab, float x) {
  const int s = min(__float2int_rd(x * (16.0f / 6.0f)), kErfSegments - 1);
  const float4 q = tab.cell[kRatioCells + s];
  return fmaf(fmaf(q.x, x, q.y), x, q.z);
}
__device__ __forceinline__ float tail_series_f(float x) {
  const float r = rcp_approx(x * x);
  const float series = fmaf(r, fmaf(r, fmaf(r, fmaf(6.5625f, r, -1.875f), 0.75f), -0.5f), 1.0f);
  return x * 1.7724538509055160273f * rcp_approx(series);
}
__device__ __forceinline__ float gauss_erfc_ratio_f(float x, int exact, const SmemTablesF& tab) {
  if (exact) return x <= 6.0f ? __fdividef(__expf(-x * x), erfcf(x)) : tail_series_f(x);
  if (x >= -1.0f) return x > 8.0f ? tail_series_f(x) : ratio_table_f(tab, x);
  if (x < -6.0f) return 0.0f;
  return exp_approx(-x * x) * rcp_approx(1.0f + erf_table_f(tab, -x));
}
__device__ __forceinline__ void pair_terms_f(float delta, bool is_edge, const RoundMathF& m, int exact,
                                             const SmemTablesF& tab, float& wf, float& sf) {
  const float dm = delta - m.mu;
  const float g = gauss_erfc_ratio_f(is_edge ? dm * m.inv_sqrt2_sigma : -dm * m.inv_sqrt2_sigma, exact, tab);
  const float sg = is_edge ? -g : g;
  const float w = fmaf(m.A * g, g, m.B * dm * sg);
  wf = 0.0f;
  sf = 0.0f;
  if (w > 0.0f) {
    wf = w;
    const float dw = delta * w;
    const float num = fmaf(m.C, sg, dw);
    if (delta > 0.0f && num > 0.0f) sf = num * rcp_approx(dw);
  }
}

// per-block copy of the round's tables into shared memory: the double knot/coefficient arrays (PRECISE) or the
// directly indexed fp32 cells
template <int THREADS>
__device__ __forceinline__ void load_tables(SmemTables& sh, const GatherArgs& a) {
  for (int i = threadIdx.x; i < 65; i += THREADS) {
    sh.erf[i] = a.tab.erf[i];
    sh.ratio[i] = a.tab.ratio[i];
  }
}
template <int THREADS>
__device__ __forceinline__ void load_tables(SmemTablesF& sh, const GatherArgs& a) {
  for (int i = threadIdx.x; i < kTableF32Entries; i += THREADS) sh.cell[i] = __ldg(a.tab_f32 + i);
}

template <int VEC>
__device__ __forceinline__ void load_row(const float* __restrict__ p, float (&v)[VEC]) {
  if constexpr (VEC == 4) {
#ifdef GEMPE_ROW_LOADS_CG
    const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
#else
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
#endif
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (VEC == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = __ldg(p);
  }
}

template <int VEC>
__device__ __forceinline__ void store_row(float* __restrict__ p, const float (&v)[VEC]) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

// the updated row goes to this rank's X_{t+1} and to every peer's (GatherArgs::peer_next)
template <int VEC>
__device__ __forceinline__ void store_row_everywhere(const GatherArgs& a, std::size_t offset, const float (&v)[VEC]) {
  store_row<VEC>(a.x_next + offset, v);
  for (int p = 0; p < a.n_peers; ++p) store_row<VEC>(a.peer_next[p] + offset, v);
}

__device__ __forceinline__ double shfl_xor_f64(double v, int off) {
  return __shfl_xor_sync(kFull, v, off);
}

// ---------------------------------------------------------------------------------- gather, batched
//
// Same work decomposition as gather_kernel, but the per-pair scalar math (sqrt, parabola_impl) is no longer
// evaluated redundantly by all LPR lanes of a row.  A persistent warp claims work items from a global cursor
// and walks each item's lists in batches of E = (32/LPR) * TB entries: every lane group keeps TB rows in
// registers -- as DIFFERENCES x_u - x_v, the only form both the distance and the update need -- the TB per-row
// partial squared distances are reduced with a transposed (recursive-halving) shuffle pattern that leaves
// entry t of the group in lanes t*REP .. t*REP + REP - 1 (REP = LPR/TB lanes hold the same total), each lane evaluates
// the parabola of ITS entry, and one coefficient per row is shuffled back for the accumulation
//     y_u = sum_t wf_t (x_v + sf_t (x_u - x_v)) = (sum_t wf_t) x_u + sum_t wf_t (sf_t - 1) (x_u - x_v),
// i.e. one packed FFMA2 per two floats and row (add_pair, engine.cpp:66-72, regrouped; exact same real value).
// The three lists of an item (adjacency / own samples / incoming samples) are walked as one virtual list whose
// ids are fetched two batches ahead; the rows of the next batch are pulled into L2 with
// prefetch.global.L2 while the current batch is being computed.
//
// Lane (grp, r) fetches the id of entry grp*TB + r/REP of a batch, which is also the entry it owns after the reduction;
// ids and coefficients travel by sub-group shuffles (width LPR) with immediate source lanes.  Slot t of every lane of a
// group holds the SAME row (entry grp*TB + t), so one load instruction reads whole 128-byte lines of G rows.  (A
// lane-dependent slot order makes the reduction select-free, but then one load instruction touches TB different rows
// with 32 bytes each: measured 10.5 ms instead of 4.6 ms on c4.)  FEW lanes per row minimise shuffles and selects: LPR = 8 at
// d = 128 (a lane holds four 16-byte vectors of a row, 128 bytes apart), four rows per group -- 4 id shuffles, 4 coefficient
// shuffles and a 4 -> 1 transposed reduction per batch of 16 rows, instead of 16 / 16 / 16 -> 1 with one warp per row: 1.75 G
// instead of 2.19 G warp instructions on c4.  But the own row and the accumulator then take 32 registers, the kernel
// needs 128 and runs 16 instead of 20 warps per SM, which costs more than the instructions save (launch_gather).
//
// PRECISE = true : pair_distance exactly as the reference (double differences, double accumulation), double
//                  parabola chain.
// PRECISE = false: differences, per-lane partial sums, the cross-lane sum and the parabola chain in fp32 (relative
//                  error <= ~3e-7 on delta, ~1e-6 on the weights); a tallied pair whose histogram position lands
//                  within 4e-6 (relative) of a bin edge is recomputed in double, so the 2x512 tallies stay exact.
// FULL            : ld == LPR*NV*VEC, no column predicates.

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
#ifndef GEMPE_PREFETCH_LEVEL
#define GEMPE_PREFETCH_LEVEL 2
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) {
#if GEMPE_PREFETCH_LEVEL == 1
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}


template <int LPR, int NV, int VEC, int TB, int U, bool PRECISE, bool FULL, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) gather_batched_kernel(const GatherArgs a, std::uint32_t item_lo,
                                                                       std::uint32_t item_hi) {
  constexpr int G = 32 / LPR;
  constexpr int E = G * TB;
  constexpr int REP = LPR / TB;
  static_assert(TB <= LPR && (TB & (TB - 1)) == 0, "TB must be a power of two <= LPR");
  constexpr int ROW_BYTES_MAX = LPR * NV * VEC * 4;
  constexpr int LINES = ROW_BYTES_MAX >= 128 ? ROW_BYTES_MAX / 128 : 1;  // 128-byte lines per row
  constexpr bool kPrefetch = ROW_BYTES_MAX >= 128 && U == 1;
  using red_t = typename std::conditional<PRECISE, double, float>::type;
  if (a.run && run_stopped(a.run)) return;  // a queued round after the run has stopped
  __shared__ unsigned int sh_hist[2 * kBins];
  using tab_t = typename std::conditional<PRECISE, SmemTables, SmemTablesF>::type;
  __shared__ tab_t sh_tab;
  for (int i = threadIdx.x; i < 2 * kBins; i += THREADS) sh_hist[i] = 0;
  load_tables<THREADS>(sh_tab, a);
  const RoundMath rm = a.math_dev ? *a.math_dev : a.math;  // sigma may live on the device (sigma_update_kernel)
  const RoundMathF mf{static_cast<float>(rm.mu), static_cast<float>(rm.inv_sqrt2_sigma),
                      static_cast<float>(rm.A), static_cast<float>(rm.B), static_cast<float>(rm.C)};
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int grp = lane / LPR, r = lane % LPR;
  const int mine = grp * TB + r / REP;  // the batch entry this lane fetches and, after the reduction, owns
  const std::uint32_t ld = a.ld;
  bool act[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) act[j] = FULL || static_cast<std::uint32_t>((r + LPR * j) * VEC) < ld;
  // this lane's column block of every row, and the row pitch in bytes (a compile-time constant when FULL, so the row
  // address is one shift-add; otherwise one 32x32->64 multiply-add)
  const char* x_lane = reinterpret_cast<const char*>(a.x_cur + r * VEC);
  const std::uint32_t row_bytes = FULL ? static_cast<std::uint32_t>(ROW_BYTES_MAX) : ld * 4u;
  auto row_ptr = [&](std::uint32_t row, int j) {
    return reinterpret_cast<const float*>(x_lane + static_cast<std::uint64_t>(row) * row_bytes + LPR * j * VEC * 4);
  };
  // the REP lanes that share an entry split its row's lines between them for the L2 prefetch
  constexpr int kPfLines = LINES >= REP ? LINES / REP : 1;
  const char* pf_lane = reinterpret_cast<const char*>(a.x_cur) + (r % REP) * 128;
  const bool pf_lane_on = LINES >= REP || (r % REP) < LINES;

  // persistent warps: every warp claims kGrab consecutive work items at a time from a global cursor, so no warp
  // idles behind a heavy neighbour and the per-block setup above is paid once per resident block
  for (;;) {
    std::uint32_t claim = 0;
    if (lane == 0) claim = atomicAdd(a.work_cursor, static_cast<std::uint32_t>(kGrab));
    claim = __shfl_sync(kFull, claim, 0);
    if (claim >= item_hi - item_lo) break;
    const std::uint32_t claim_end = min(claim + kGrab, item_hi - item_lo);
    for (std::uint32_t item = item_lo + claim; item < item_lo + claim_end; ++item) {
      // the item's descriptor: two 16-byte loads (the claim's descriptors share one 128-byte line)
      const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(a.items + item));
      const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(a.items + item) + 1);
      const std::uint32_t u = d0.x, lenA = d0.z, lenB = d1.x, hub = d1.z;

      // virtual list = [adjacency slice | own samples | incoming samples], as offsets into nbr / neg_own / in_anchor
      std::uint32_t offC = 0, lenC = 0, offD = 0, lenD = 0;
      if (d1.y) {  // first item of the vertex: it takes the incoming samples as well
        if (a.in_stride) {  // slotted buckets: the vertex's own slots, then what spilled (normally nothing)
          offC = u * a.in_stride;
          lenC = min(a.in_cnt[u], a.in_stride);
          if (*a.spill_count) {
            offD = a.spill_off[u];
            lenD = a.spill_off[u + 1] - offD;
          }
        } else {
          offC = __ldg(a.in_off + u);
          lenC = __ldg(a.in_off + u + 1) - offC;
        }
      }
      const std::uint32_t endB = lenA + lenB, endC = endB + lenC, total = endC + lenD;

      // one list entry (vertex id) per lane and sub-batch: lane (grp, r) holds entry grp*TB + r/REP of the sub-batch.
      // Validity and kind (0 edge, 1 sample tallied here, 2 incoming sample) follow from the entry's position alone, so
      // nothing has to wait on these loads until the ids are needed as addresses two batches later.
      // entry e of the virtual list lives at index e + d of its array (wrapping 32-bit arithmetic)
      const std::uint32_t dA = d0.y, dB = d0.w - lenA, dC = offC - endB, dD = offD - endC;
      auto fetch = [&](std::uint32_t base, std::uint32_t (&ent)[U]) {
#pragma unroll
        for (int s = 0; s < U; ++s) {
          const std::uint32_t e = base + s * E + mine;
          const bool in_a = e < lenA, in_b = e < endB, in_c = e < endC;
          const std::uint32_t idx = e + (in_a ? dA : (in_b ? dB : (in_c ? dC : dD)));
          const std::uint32_t* arr = in_a ? a.nbr : (in_b ? a.neg_own : (in_c ? a.in_anchor : a.spill_anchor));
          ent[s] = u;  // own row past the list end: zero difference, zero weight
          if (e < total) ent[s] = __ldg(arr + idx);
        }
      };

      float xu[NV][VEC];
      float y[NV][VEC];  // sum_t wf_t (sf_t - 1) (x_u - x_v)
#pragma unroll
      for (int j = 0; j < NV; ++j) {
#pragma unroll
        for (int c = 0; c < VEC; ++c) xu[j][c] = 0.0f, y[j][c] = 0.0f;
        if (act[j]) load_row<VEC>(row_ptr(u, j), xu[j]);
      }
      float zacc = 0.0f;

      std::uint32_t cur[U], nxt[U];
      fetch(0, cur);
      fetch(E * U, nxt);

      for (std::uint32_t base = 0; base < total; base += E * U) {
        // TB rows per lane group and sub-batch, all loads issued before any use; slot t = entry grp*TB + t
        float xv[U][TB][NV][VEC];
#pragma unroll
        for (int s = 0; s < U; ++s) {
#pragma unroll
          for (int t = 0; t < TB; ++t) {
            const std::uint32_t src_row = __shfl_sync(kFull, cur[s], t * REP, LPR);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              if constexpr (!FULL) {
#pragma unroll
                for (int c = 0; c < VEC; ++c) xv[s][t][j][c] = 0.0f;
              }
              if (act[j]) load_row<VEC>(row_ptr(src_row, j), xv[s][t][j]);
            }
          }
        }
        // rows of the next batch -> L2 (their entries arrived during the previous batch), entries of the batch
        // after that -> registers
        if constexpr (kPrefetch) {
          if (pf_lane_on && base + E + mine < total) {  // the lane's own entry of the next batch: no shuffles
            const char* row = pf_lane + static_cast<std::uint64_t>(nxt[0]) * row_bytes;
#pragma unroll
            for (int i = 0; i < kPfLines; ++i) prefetch_l2(row + i * REP * 128);
          }
        }
        std::uint32_t nn[U];
        fetch(base + 2 * E * U, nn);

#pragma unroll
        for (int s = 0; s < U; ++s) {
          // rows become differences x_u - x_v; per-row partial squared distance; transposed reduction
          red_t p[TB];
#pragma unroll
          for (int t = 0; t < TB; ++t) {
            if constexpr (PRECISE) {
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < NV; ++j)
#pragma unroll
                for (int c = 0; c < VEC; ++c) {
                  const double diff = static_cast<double>(xu[j][c]) - static_cast<double>(xv[s][t][j][c]);
                  acc = fma(diff, diff, acc);
                  xv[s][t][j][c] = xu[j][c] - xv[s][t][j][c];
                }
              p[t] = acc;
            } else if constexpr (VEC % 2 == 0) {
              float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int j = 0; j < NV; ++j)
#pragma unroll
                for (int c = 0; c < VEC; c += 2) {
                  const float2 diff = ffma2(make_float2(xv[s][t][j][c], xv[s][t][j][c + 1]), make_float2(-1.0f, -1.0f),
                                            make_float2(xu[j][c], xu[j][c + 1]));
                  acc = ffma2(diff, diff, acc);
                  xv[s][t][j][c] = diff.x;
                  xv[s][t][j][c + 1] = diff.y;
                }
              p[t] = acc.x + acc.y;
            } else {
              float acc = 0.0f;
#pragma unroll
              for (int j = 0; j < NV; ++j) {
                const float diff = xu[j][0] - xv[s][t][j][0];
                acc = fmaf(diff, diff, acc);
                xv[s][t][j][0] = diff;
              }
              p[t] = acc;
            }
          }
          {
            // transposed (recursive-halving) reduction: at lane distance `off` the lower lane keeps the first half of the
            // rows and takes the partner's partial sums of them, the upper lane the second half
            int width = TB;
#pragma unroll
            for (int off = LPR / 2; off >= 1; off >>= 1) {
              if (width > 1) {
                const int half = width / 2;
                const bool upper = (r & off) != 0;
#pragma unroll
                for (int i = 0; i < TB / 2; ++i) {
                  if (i < half) {
                    const red_t keep = upper ? p[i + half] : p[i];
                    const red_t give = upper ? p[i] : p[i + half];
                    p[i] = keep + __shfl_xor_sync(kFull, give, off);
                  }
                }
                width = half;
              } else {
                p[0] += __shfl_xor_sync(kFull, p[0], off);
              }
            }
          }
          // p[0] is the squared distance of the entry this lane fetched itself
          const std::uint32_t own = cur[s];
          const std::uint32_t own_e = base + s * E + mine;
          const bool valid = own_e < total;
          const bool is_edge = own_e < lenA;
          const bool tally = valid && (r % REP == 0) && (is_edge ? u < own : own_e < endB);
          float wf = 0.0f, sf = 0.0f;
          int bin;
          if constexpr (PRECISE) {
            const double delta = sqrt(p[0]);
            bin = static_cast<int>(delta / 12.0 * 512.0);  // DistanceHistogram::record (histogram.hpp:24-29)
            if (valid) pair_terms(delta, is_edge, rm, sh_tab, wf, sf);
          } else {
            float delta = sqrt_approx(p[0]);
            // exact tallies: recompute in double the rows whose bin position is within the fp32 error bound of an edge
            const float pos = delta * (512.0f / 12.0f);
            const float frac = pos - floorf(pos);
            const float tol = 4e-6f * pos + 1e-9f;
            const bool amb = tally && pos < 513.0f && (frac < tol || frac > 1.0f - tol);
            bin = static_cast<int>(pos);
            unsigned pending = __ballot_sync(kFull, amb);
            while (pending) {  // rare: one exact pair_distance per ambiguous pair, rows re-read (they are L1/L2 hot)
              const int l = __ffs(pending) - 1;
              pending &= pending - 1;
              const std::uint32_t other = __shfl_sync(kFull, own, l);
              double acc = 0.0;
              if (lane < LPR) {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                  if (static_cast<std::uint32_t>((lane + LPR * j) * VEC) < ld) {
                    float xo[VEC], xs[VEC];
                    load_row<VEC>(a.x_cur + static_cast<std::size_t>(other) * ld + (lane + LPR * j) * VEC, xo);
                    load_row<VEC>(a.x_cur + static_cast<std::size_t>(u) * ld + (lane + LPR * j) * VEC, xs);
#pragma unroll
                    for (int c = 0; c < VEC; ++c) {
                      const double diff = static_cast<double>(xs[c]) - static_cast<double>(xo[c]);
                      acc = fma(diff, diff, acc);
                    }
                  }
                }
              }
#pragma unroll
              for (int off = 16; off >= 1; off >>= 1) acc += shfl_xor_f64(acc, off);
              if (lane == l) {
                const double exact = sqrt(acc);
                bin = static_cast<int>(exact / 12.0 * 512.0);
                delta = static_cast<float>(exact);
              }
            }
            if (valid) pair_terms_f(delta, is_edge, mf, rm.exact, sh_tab, wf, sf);
          }
          if (tally) {  // tallied before the w > 0 test (engine.cpp:221-222)
            bin = bin >= kBins ? kBins - 1 : (bin < 0 ? 0 : bin);
            atomicAdd(&sh_hist[(is_edge ? 0 : kBins) + bin], 1u);
          }
          if (r % REP == 0) zacc += wf;
          const float coef = wf * (sf - 1.0f);
          // y += wf (sf - 1) (x_u - x_v) from the resident differences
#pragma unroll
          for (int t = 0; t < TB; ++t) {
            const float ct = __shfl_sync(kFull, coef, t * REP, LPR);  // coefficient of entry grp*TB + t
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              if constexpr (VEC % 2 == 0) {
#pragma unroll
                for (int c = 0; c < VEC; c += 2) {
                  const float2 acc = ffma2(make_float2(ct, ct), make_float2(xv[s][t][j][c], xv[s][t][j][c + 1]),
                                           make_float2(y[j][c], y[j][c + 1]));
                  y[j][c] = acc.x;
                  y[j][c + 1] = acc.y;
                }
              } else {
                y[j][0] = fmaf(ct, xv[s][t][j][0], y[j][0]);
              }
            }
          }
        }
#pragma unroll
        for (int s = 0; s < U; ++s) {
          cur[s] = nxt[s];
          nxt[s] = nn[s];
        }
      }

      // Consolidation (the reference sums its replicas in double, engine.cpp:88-107) and the update, spread over the
      // WHOLE warp: vector j of the row is finalised by lane group j % G, so every lane handles JF = ceil(NV / G) vectors
      // instead of group 0 handling all NV.  The groups' fp32 partial sums (and the own row) change hands through shared
      // memory; y_u = z_u x_u + sum of the weighted differences.
      constexpr int JF = (NV + G - 1) / G;
      double zs = static_cast<double>(zacc);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) zs += shfl_xor_f64(zs, off);
      double ys[JF][VEC];
      float xo[JF][VEC];
      bool fin[JF];
      std::uint32_t fcol[JF];
      if constexpr (G == 1) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          fin[j] = act[j];
          fcol[j] = static_cast<std::uint32_t>((r + LPR * j) * VEC);
#pragma unroll
          for (int c = 0; c < VEC; ++c) {
            xo[j][c] = xu[j][c];
            ys[j][c] = fma(zs, static_cast<double>(xu[j][c]), static_cast<double>(y[j][c]));
          }
        }
      } else {
        static_assert(G == 1 || VEC == 4, "the exchange moves 16-byte vectors");
        __shared__ float4 sh_part[THREADS / 32][G][NV * LPR];
        __shared__ float4 sh_own[THREADS / 32][NV * LPR];
        const int w = threadIdx.x >> 5;
        __syncwarp();  // the previous item's readers are done
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          sh_part[w][grp][j * LPR + r] = make_float4(y[j][0], y[j][1], y[j][2], y[j][3]);
          if (grp == 0) sh_own[w][j * LPR + r] = make_float4(xu[j][0], xu[j][1], xu[j][2], xu[j][3]);
        }
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < JF; ++jj) {
          const int j = grp + jj * G;
          fcol[jj] = static_cast<std::uint32_t>((r + LPR * j) * VEC);
          fin[jj] = j < NV && (FULL || fcol[jj] < ld);
          const int at = (j < NV ? j : 0) * LPR + r;
          double sum[VEC] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float4 v = sh_part[w][g][at];
            sum[0] += static_cast<double>(v.x);
            sum[1] += static_cast<double>(v.y);
            sum[2] += static_cast<double>(v.z);
            sum[3] += static_cast<double>(v.w);
          }
          const float4 own = sh_own[w][at];
          xo[jj][0] = own.x; xo[jj][1] = own.y; xo[jj][2] = own.z; xo[jj][3] = own.w;
#pragma unroll
          for (int c = 0; c < VEC; ++c) ys[jj][c] = fma(zs, static_cast<double>(xo[jj][c]), sum[c]);
        }
      }

      bool finalize = true;
      if (hub != kNoHub) {
        const std::uint32_t p0 = __ldg(a.hub_first + hub), q = __ldg(a.hub_items + hub);
        const std::uint32_t slot = p0 + d1.w;
#pragma unroll
        for (int jj = 0; jj < JF; ++jj) {
          if (!fin[jj]) continue;
#pragma unroll
          for (int c = 0; c < VEC; ++c) a.part_y[static_cast<std::size_t>(slot) * ld + fcol[jj] + c] = ys[jj][c];
        }
        if (lane == 0) a.part_z[slot] = zs;
        __threadfence();
        __syncwarp();
        std::uint32_t arrived = 0;
        if (lane == 0) arrived = atomicAdd(a.hub_arrived + hub, 1u);
        arrived = __shfl_sync(kFull, arrived, 0);
        finalize = arrived == q - 1;
        if (finalize) {  // last slice of the hub: consolidate the partials in slot order
          __threadfence();
          zs = 0.0;
#pragma unroll
          for (int jj = 0; jj < JF; ++jj)
#pragma unroll
            for (int c = 0; c < VEC; ++c) ys[jj][c] = 0.0;
          for (std::uint32_t sl = p0; sl < p0 + q; ++sl) {
            zs += __ldcg(a.part_z + sl);
#pragma unroll
            for (int jj = 0; jj < JF; ++jj) {
              if (!fin[jj]) continue;
#pragma unroll
              for (int c = 0; c < VEC; ++c) ys[jj][c] += __ldcg(a.part_y + static_cast<std::size_t>(sl) * ld + fcol[jj] + c);
            }
          }
          if (lane == 0) a.hub_arrived[hub] = 0;
        }
      }

      if (finalize) {
        // reduce_and_update (engine.cpp:261-272): z <= 0 holds position, else x = float(y / z) -- as y * (1 / z) in
        // double, one division per item (the quotient differs from y / z by at most one double ulp before the rounding
        // to float)
        bool bad = false;
        const double inv_z = zs > 0.0 ? 1.0 / zs : 0.0;
#pragma unroll
        for (int jj = 0; jj < JF; ++jj) {
          if (!fin[jj]) continue;
          float out[VEC];
#pragma unroll
          for (int c = 0; c < VEC; ++c) {
            out[c] = xo[jj][c];
            if (zs > 0.0) {
              out[c] = static_cast<float>(ys[jj][c] * inv_z);
              bad |= !isfinite(out[c]);
            }
          }
          store_row_everywhere<VEC>(a, static_cast<std::size_t>(u) * ld + fcol[jj], out);
          if (a.cap_y) {
#pragma unroll
            for (int c = 0; c < VEC; ++c)
              if (fcol[jj] + c < a.dim) a.cap_y[static_cast<std::size_t>(u) * a.dim + fcol[jj] + c] = ys[jj][c];
          }
        }
        if (a.cap_z && lane == 0) a.cap_z[u] = zs;
        if (bad) atomicOr(a.status + kStatNonFinite, 1u);
      }
    }
  }

  __syncthreads();
  for (int i = threadIdx.x; i < 2 * kBins; i += THREADS) {
    const unsigned int c = sh_hist[i];
    if (c) atomicAdd(a.hist + i, static_cast<unsigned long long>(c));
  }
  if (a.n_peers) __threadfence_system();  // peer stores are performed before the grid retires
}

// ---------------------------------------------------------------------------------- gather, one thread per work item
//
// d <= 4 (graph drawing): a row is one 4..16-byte vector, so a whole work item fits one thread -- 32 different
// vertices per warp keep 4 x 32 independent row gathers in flight, and there is no warp-serial latency chain per
// item.  Same arithmetic and the same hub protocol as gather_batched_kernel; items are capped at 32 adjacency
// positions (context.cpp) to bound divergence on hubs.
template <int VEC, bool PRECISE>
__global__ void __launch_bounds__(kThreads) gather_thread_kernel(const GatherArgs a, std::uint32_t item_lo,
                                                                 std::uint32_t item_hi) {
#ifndef GEMPE_INFLIGHT
#define GEMPE_INFLIGHT 4
#endif
  constexpr int kInflight = GEMPE_INFLIGHT;
  if (a.run && run_stopped(a.run)) return;  // a queued round after the run has stopped
  __shared__ unsigned int sh_hist[2 * kBins];
  using tab_t = typename std::conditional<PRECISE, SmemTables, SmemTablesF>::type;
  __shared__ tab_t sh_tab;
  for (int i = threadIdx.x; i < 2 * kBins; i += kThreads) sh_hist[i] = 0;
  load_tables<kThreads>(sh_tab, a);
  const RoundMath rm = a.math_dev ? *a.math_dev : a.math;
  const RoundMathF mf{static_cast<float>(rm.mu), static_cast<float>(rm.inv_sqrt2_sigma),
                      static_cast<float>(rm.A), static_cast<float>(rm.B), static_cast<float>(rm.C)};
  __syncthreads();

  const std::uint32_t item = item_lo + blockIdx.x * kThreads + threadIdx.x;
  if (item < item_hi) {
    const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(a.items + item));
    const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(a.items + item) + 1);
    const std::uint32_t u = d0.x, begin = d0.y, lenA = d0.z, offB = d0.w, lenB = d1.x, hub = d1.z;
    std::uint32_t offC = 0, lenC = 0, offD = 0, lenD = 0;
    if (d1.y) {  // first item of the vertex
      if (a.in_stride) {  // slotted buckets (see gather_batched_kernel)
        offC = u * a.in_stride;
        lenC = min(a.in_cnt[u], a.in_stride);
        if (*a.spill_count) {
          offD = a.spill_off[u];
          lenD = a.spill_off[u + 1] - offD;
        }
      } else {
        offC = __ldg(a.in_off + u);
        lenC = __ldg(a.in_off + u + 1) - offC;
      }
    }
    const std::uint32_t endB = lenA + lenB, endC = endB + lenC, total = endC + lenD;
    const std::uint32_t ld = a.ld;

    float xu[VEC], y[VEC];
    load_row<VEC>(a.x_cur + static_cast<std::size_t>(u) * ld, xu);
#pragma unroll
    for (int c = 0; c < VEC; ++c) y[c] = 0.0f;
    float zacc = 0.0f;

    for (std::uint32_t base = 0; base < total; base += kInflight) {
      std::uint32_t other[kInflight];
      float xv[kInflight][VEC];
#pragma unroll
      for (int q = 0; q < kInflight; ++q) {
        const std::uint32_t e = base + q;
        other[q] = u;
        if (e < total) {
          other[q] = __ldg(e < lenA ? a.nbr + begin + e
                                    : (e < endB ? a.neg_own + offB + (e - lenA)
                                                : (e < endC ? a.in_anchor + offC + (e - endB) : a.spill_anchor + offD + (e - endC))));
        }
      }
#pragma unroll
      for (int q = 0; q < kInflight; ++q) load_row<VEC>(a.x_cur + static_cast<std::size_t>(other[q]) * ld, xv[q]);
#pragma unroll
      for (int q = 0; q < kInflight; ++q) {
        const std::uint32_t e = base + q;
        if (e >= total) break;
        const bool is_edge = e < lenA;
        const bool tally = is_edge ? u < other[q] : e < endB;
        float diff[VEC];
        double exact2 = 0.0;
        float d2 = 0.0f;
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          diff[c] = xu[c] - xv[q][c];
          d2 = fmaf(diff[c], diff[c], d2);
          const double dd = static_cast<double>(xu[c]) - static_cast<double>(xv[q][c]);
          exact2 = fma(dd, dd, exact2);  // pair_distance (engine.cpp:45-52); dead code in the fast path unless needed below
        }
        float wf = 0.0f, sf = 0.0f;
        int bin;
        if constexpr (PRECISE) {
          const double delta = sqrt(exact2);
          bin = static_cast<int>(delta / 12.0 * 512.0);
          pair_terms(delta, is_edge, rm, sh_tab, wf, sf);
        } else {
          float delta = sqrt_approx(d2);
          const float pos = delta * (512.0f / 12.0f);
          const float frac = pos - floorf(pos);
          const float tol = 4e-6f * pos + 1e-9f;
          bin = static_cast<int>(pos);
          if (tally && pos < 513.0f && (frac < tol || frac > 1.0f - tol)) {  // exact tally near a bin edge
            const double ex = sqrt(exact2);
            bin = static_cast<int>(ex / 12.0 * 512.0);
            delta = static_cast<float>(ex);
          }
          pair_terms_f(delta, is_edge, mf, rm.exact, sh_tab, wf, sf);
        }
        if (tally) {
          bin = bin >= kBins ? kBins - 1 : (bin < 0 ? 0 : bin);
          atomicAdd(&sh_hist[(is_edge ? 0 : kBins) + bin], 1u);
        }
        zacc += wf;
        const float coef = wf * (sf - 1.0f);
#pragma unroll
        for (int c = 0; c < VEC; ++c) y[c] = fmaf(coef, diff[c], y[c]);
      }
    }

    double zs = static_cast<double>(zacc);
    double ys[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) ys[c] = fma(zs, static_cast<double>(xu[c]), static_cast<double>(y[c]));
    bool finalize = true;
    if (hub != kNoHub) {
      const std::uint32_t p0 = __ldg(a.hub_first + hub), q = __ldg(a.hub_items + hub);
      const std::uint32_t slot = p0 + d1.w;
#pragma unroll
      for (int c = 0; c < VEC; ++c) a.part_y[static_cast<std::size_t>(slot) * ld + c] = ys[c];
      a.part_z[slot] = zs;
      __threadfence();
      finalize = atomicAdd(a.hub_arrived + hub, 1u) == q - 1;
      if (finalize) {  // last slice of the hub: consolidate the partials in slot order
        __threadfence();
        zs = 0.0;
#pragma unroll
        for (int c = 0; c < VEC; ++c) ys[c] = 0.0;
        for (std::uint32_t sl = p0; sl < p0 + q; ++sl) {
          zs += __ldcg(a.part_z + sl);
#pragma unroll
          for (int c = 0; c < VEC; ++c) ys[c] += __ldcg(a.part_y + static_cast<std::size_t>(sl) * ld + c);
        }
        a.hub_arrived[hub] = 0;
      }
    }
    if (finalize) {
      bool bad = false;
      float out[VEC];
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        out[c] = xu[c];
        if (zs > 0.0) {
          out[c] = static_cast<float>(ys[c] / zs);
          bad |= !isfinite(out[c]);
        }
      }
      store_row_everywhere<VEC>(a, static_cast<std::size_t>(u) * ld, out);
      if (a.cap_y) {
#pragma unroll
        for (int c = 0; c < VEC; ++c)
          if (static_cast<std::uint32_t>(c) < a.dim) a.cap_y[static_cast<std::size_t>(u) * a.dim + c] = ys[c];
      }
      if (a.cap_z) a.cap_z[u] = zs;
      if (bad) atomicOr(a.status + kStatNonFinite, 1u);
    }
  }

  __syncthreads();
  for (int i = threadIdx.x; i < 2 * kBins; i += kThreads) {
    const unsigned int c = sh_hist[i];
    if (c) atomicAdd(a.hist + i, static_cast<unsigned long long>(c));
  }
  if (a.n_peers) __threadfence_system();  // peer stores are performed before the grid retires
}

// ---------------------------------------------------------------------------------- sigma search on the device
//
// optimize_sigma_detail + the growth cap + the PE estimate of run_single_iteration (slope.cpp:75-125,
// engine.cpp:293-314) on the round's 2x512 tallies: one block, thread b owns bin b of both tallies, every objective
// evaluation is one block-wide double sum.  Removes the host round trip (8 KiB D2H + ~0.3 ms of libm) between
// rounds; the next round's gather reads the folded RoundMath straight from device memory.
namespace sigma {

constexpr double kLn2 = 0.693147180559945309417232121458176568;
constexpr double kSqrt2 = 1.41421356237309504880168872420969808;
constexpr double kSqrtPi = 1.77245385090551602729816748334;

__device__ __forceinline__ double tail_ratio(double x) {  // gauss_over_erfc, sigmoid.hpp:39-45
  if (x <= 6.0) return exp(-x * x) / erfc(x);
  const double r = 1.0 / (x * x);
  return x * kSqrtPi / (1.0 + r * (-0.5 + r * (0.75 + r * (-1.875 + 6.5625 * r))));
}
__device__ __forceinline__ double cost_tail(double mid, double mu, double s, bool edge) {  // sigmoid.hpp:50-59
  const double u = (mid - mu) / (kSqrt2 * s);
  const double x = edge ? u : -u;
  if (x <= 6.0) return 1.0 - log2(erfc(x));
  const double r = 1.0 / (x * x);
  const double series = 1.0 + r * (-0.5 + r * (0.75 + r * (-1.875 + 6.5625 * r)));
  return 1.0 - (-x * x - log(x * kSqrtPi) + log(series)) / kLn2;
}
__device__ __forceinline__ double cost_floor(double mid, double mu, double s, bool edge) {  // sigmoid.hpp:69-81
  const double e = erf((mid - mu) / (kSqrt2 * s));
  double pr = edge ? 0.5 - 0.5 * e : 0.5 + 0.5 * e;
  pr = fmin(fmax(pr, 1e-12), 1.0 - 1e-12);
  return -log2(pr);
}
__device__ __forceinline__ double cost_dsigma(double mid, double mu, double s, bool edge) {  // sigmoid.hpp:108-113
  const double u = (mid - mu) / (kSqrt2 * s);
  const double v = 2.0 / (kSqrtPi * kLn2) * u * tail_ratio(edge ? u : -u) / s;
  return edge ? -v : v;
}

__device__ __forceinline__ double block_sum(double v, double* scratch) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kBins / 32; ++w) t += scratch[w];
  return t;
}

// Run bookkeeping after a completed round (one block; see RunState): PE / sigma trace, best PE, the convergence window of
// EmbeddingEngine::run (engine.cpp:353-367: the last `window` rounds brought no minimum beating the earlier best by
// tol), failure flags, the round's tallies.
__device__ __forceinline__ void record_round(RunState* run, double* pe_trace, double* sigma_trace, double pe, double sigma_new,
                                             double nonedge_weight, const std::uint32_t* status,
                                             const unsigned long long* hist) {
  for (int i = threadIdx.x; i < 2 * kBins; i += blockDim.x) run->last_hist[i] = hist[i];
  if (threadIdx.x != 0) return;
  const unsigned long long k = run->count;
  std::uint32_t bad = 0;
  for (int i = 0; i < 8; ++i) {
    const std::uint32_t w = status[i];
    if (i == kStatDrawsLo || i == kStatDrawsHi) continue;
    run->sticky_status[i] |= w;
    bad |= w;
  }
  run->draws = static_cast<unsigned long long>(status[kStatDrawsLo]) | (static_cast<unsigned long long>(status[kStatDrawsHi]) << 32);
  run->last_nonedge_weight = nonedge_weight;
  if (k < run->trace_cap) {
    pe_trace[k] = pe;
    sigma_trace[k] = sigma_new;
  }
  if (pe < run->best_pe) {
    run->best_pe = pe;
    run->improved_at = k + 1;
  }
  const unsigned long long have = k + 1;
  const unsigned long long window = static_cast<unsigned long long>(run->window);
  if (have > window && have <= run->trace_cap) {
    double best_before = pe_trace[0], best_recent = pe_trace[have - window];
    for (unsigned long long i = 1; i < have - window; ++i) best_before = fmin(best_before, pe_trace[i]);
    for (unsigned long long i = have - window + 1; i < have; ++i) best_recent = fmin(best_recent, pe_trace[i]);
    if (best_before - best_recent < run->tol * fabs(best_before)) run->converged = 1;
  }
  if (bad && !run->failed) {
    run->failed = 1;
    run->fail_iter = k;
  }
  __threadfence();
  run->count = have;
}

}  // namespace sigma

// ---------------------------------------------------------------------------------- quality scoring: pe_sampled
//
// metrics.cpp:166-213 on the device: the edge distances exactly, the non-edge sum estimated from sampled partners
// reweighted by (N - m) / #samples; the (mu, sigma) minimisation of metrics.cpp:73-127 is driven from the host over the
// two distance arrays.  The sample stream is counter-based (not the reference's sequential SplitMix), and the edge test
// is the run's hash set (false positives reject a distance-independent few per cent of the non-edges), so the
// estimate agrees with the reference statistically, not draw for draw.

// distance() of metrics.cpp:16-25: double differences, double accumulation, rounded to float like the reference's arrays
__device__ __forceinline__ float pe_distance(const float* __restrict__ x, std::uint32_t ld, std::uint32_t dim,
                                             std::uint32_t i, std::uint32_t j) {
  const float* a = x + static_cast<std::size_t>(i) * ld;
  const float* b = x + static_cast<std::size_t>(j) * ld;
  double acc = 0.0;
  for (std::uint32_t k = 0; k < dim; ++k) {
    const double diff = static_cast<double>(__ldg(a + k)) - static_cast<double>(__ldg(b + k));
    acc = fma(diff, diff, acc);
  }
  return static_cast<float>(sqrt(acc));
}

__global__ void __launch_bounds__(kThreads) pe_collect_kernel(const PeCollectArgs p) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  const std::uint64_t per_edge = 1 + static_cast<std::uint64_t>(p.samples_per_edge);
  const float nan = __int_as_float(0x7fc00000);
  for (std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < p.m * per_edge; t += stride) {
    const std::uint64_t e = t / per_edge;
    const std::uint32_t s = static_cast<std::uint32_t>(t % per_edge);
    const std::uint32_t u = __ldg(p.src + e), v = __ldg(p.dst + e);
    if (s == 0) {
      p.edge_dist[e] = pe_distance(p.x, p.ld, p.dim, u, v);
      continue;
    }
    const std::uint32_t k = s - 1;
    std::uint32_t anchor = (k % 2 == 0) ? u : v, other = (k % 2 == 0) ? v : u;
    const std::uint64_t slot = e * p.samples_per_edge + k;
    auto degree = [&](std::uint32_t w) { return __ldg(p.rowptr + w + 1) - __ldg(p.rowptr + w); };
    if (degree(anchor) >= p.n - 1) {  // saturated anchors cannot have a non-edge partner (metrics.cpp:188-190)
      const std::uint32_t tmp = anchor;
      anchor = other;
      other = tmp;
    }
    float d = nan;
    if (degree(anchor) < p.n - 1) {
      const std::uint64_t key = mix(p.seed, slot);
      for (std::uint32_t tries = 0; tries < 100000u; ++tries) {
        const std::uint64_t r = mix(key, tries);
        const std::uint32_t g = static_cast<std::uint32_t>(((r >> 32) * p.n) >> 32);
        if (g == anchor) continue;
        if (hash_test(p.hash_words, p.hash_summary, p.hash_mask, p.n, anchor, g)) continue;
        d = pe_distance(p.x, p.ld, p.dim, anchor, g);
        break;
      }
    }
    p.nonedge_dist[slot] = d;  // NaN = skipped
  }
}

// sum over a distance array of description_length (which = 0) or dl_sigma_derivative (which = 1); NaN entries are
// skipped and counted out
__global__ void __launch_bounds__(kThreads) pe_sum_kernel(const float* __restrict__ dist, std::uint64_t count, double mu,
                                                          double sg, int is_edge, int which, double* __restrict__ total,
                                                          unsigned long long* __restrict__ valid) {
  using namespace sigma;
  __shared__ double warp_sum[kThreads / 32];
  __shared__ unsigned long long warp_cnt[kThreads / 32];
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  double acc = 0.0;
  unsigned long long cnt = 0;
  for (std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += stride) {
    const float d = dist[t];
    if (d != d) continue;
    ++cnt;
    acc += which == 0 ? cost_floor(static_cast<double>(d), mu, sg, is_edge != 0)
                      : cost_dsigma(static_cast<double>(d), mu, sg, is_edge != 0);
  }
  for (int off = 16; off > 0; off >>= 1) {
    acc += __shfl_xor_sync(kFull, acc, off);
    cnt += __shfl_xor_sync(kFull, cnt, off);
  }
  if ((threadIdx.x & 31) == 0) {
    warp_sum[threadIdx.x >> 5] = acc;
    warp_cnt[threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    unsigned long long c = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      t += warp_sum[w];
      c += warp_cnt[w];
    }
    atomicAdd(total, t);
    if (valid) atomicAdd(valid, c);
  }
}

__global__ void __launch_bounds__(kBins) sigma_update_kernel(const unsigned long long* __restrict__ hist, double mu,
                                                             double pairs, double edges, int exact_math,
                                                             SigmaState* __restrict__ state,
                                                             std::uint32_t* __restrict__ status, RunState* run,
                                                             double* pe_trace, double* sigma_trace) {
  using namespace sigma;
  if (run && run_stopped(run)) return;  // a queued round after the run has stopped
  __shared__ double scratch[kBins / 32];
  const int b = threadIdx.x;
  const double ec = static_cast<double>(hist[b]), nc = static_cast<double>(hist[kBins + b]);
  const double mid = (b + 0.5) * 12.0 / kBins;  // histogram.hpp:52
  const double samples = block_sum(nc, scratch);
  if (block_sum(ec, scratch) + samples == 0.0) {  // optimize_sigma on an empty histogram is a config_error (slope.cpp:76)
    if (b == 0) atomicOr(status + kStatEmptyTallies, 1u);
    if (run) {
      __syncthreads();
      record_round(run, pe_trace, sigma_trace, 0.0, state->sigma, 1.0, status, hist);
    }
    return;  // sigma stays what it was
  }
  const double nw = samples > 0.0 ? (pairs - edges) / samples : 1.0;  // engine.cpp:296-300
  auto total = [&](double s, int which) {
    double v = 0.0;
    if (which == 0) {
      if (ec != 0.0) v += ec * cost_tail(mid, mu, s, true);
      if (nc != 0.0) v += nw * nc * cost_tail(mid, mu, s, false);
    } else if (which == 1) {
      if (ec != 0.0) v += ec * cost_dsigma(mid, mu, s, true);
      if (nc != 0.0) v += nw * nc * cost_dsigma(mid, mu, s, false);
    } else {
      if (ec != 0.0) v += ec * cost_floor(mid, mu, s, true);
      if (nc != 0.0) v += nw * nc * cost_floor(mid, mu, s, false);
    }
    return block_sum(v, scratch);
  };
  // coarse geometric scan of the unfloored cost (all 17 candidates in ONE pass: 17 partial sums per thread, reduced
  // together), then bisection on dF/dsigma inside the best cell
  constexpr int kGrid = 17;
  __shared__ double grid_scratch[kBins / 32][kGrid];
  double grid[kGrid], cost[kGrid], best_cost = 0.0;
  int best = 0;
#pragma unroll 1
  for (int i = 0; i < kGrid; ++i) {
    grid[i] = 1e-3 * pow(16.0 / 1e-3, static_cast<double>(i) / (kGrid - 1));
    double v = 0.0;
    if (ec != 0.0) v += ec * cost_tail(mid, mu, grid[i], true);
    if (nc != 0.0) v += nw * nc * cost_tail(mid, mu, grid[i], false);
    cost[i] = v;
  }
#pragma unroll
  for (int i = 0; i < kGrid; ++i) {
    double v = cost[i];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    cost[i] = v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int i = 0; i < kGrid; ++i) grid_scratch[threadIdx.x >> 5][i] = cost[i];
  }
  __syncthreads();
  for (int i = 0; i < kGrid; ++i) {
    double t = 0.0;
    for (int w = 0; w < kBins / 32; ++w) t += grid_scratch[w][i];
    if (i == 0 || t < best_cost) best_cost = t, best = i;
  }
  double sigma_opt = grid[best];
  double lo = grid[best > 0 ? best - 1 : 0], hi = grid[best < kGrid - 1 ? best + 1 : kGrid - 1];
  double f_lo = total(lo, 1);
  const double f_hi = total(hi, 1);
  int steps = 0;
  if (f_lo < 0.0 && f_hi > 0.0) {
    while (hi - lo > 1e-4 && steps < 60) {
      ++steps;
      const double m = 0.5 * (lo + hi);
      const double f_mid = total(m, 1);
      if (f_mid == 0.0) {
        lo = hi = m;
        break;
      }
      if ((f_mid > 0.0) == (f_lo > 0.0)) {
        lo = m;
        f_lo = f_mid;
      } else {
        hi = m;
      }
    }
    const double refined = 0.5 * (lo + hi);
    if (total(refined, 0) <= best_cost) sigma_opt = refined;
  }
  const double sigma_new = fmin(sigma_opt, state->sigma * 1.5);  // growth cap, engine.cpp:302-307
  const double pe = total(sigma_new, 2) / pairs;
  if (b == 0) {
    const double c1 = 2.0 / (3.14159265358979323846264338327950288 * kLn2);
    const double c2 = 1.0 / (2.50662827463100050241576528481 * kLn2);
    state->sigma = sigma_new;
    state->pe_estimate = pe;
    state->nonedge_weight = nw;
    state->bisection_steps = steps;
    state->math.mu = mu;
    state->math.inv_sqrt2_sigma = 1.0 / (kSqrt2 * sigma_new);
    state->math.A = c1 / (sigma_new * sigma_new);
    state->math.B = c2 / (sigma_new * sigma_new * sigma_new);
    state->math.C = c2 / sigma_new;
    state->math.exact = exact_math;
  }
  if (run) record_round(run, pe_trace, sigma_trace, pe, sigma_new, nw, status, hist);
}

// The same search on a cluster of 8 CTAs (8 SMs): one evaluation of the objective is bound by the FP64 throughput of
// ONE SM, and the search is ~38 of them in a row.  Here every CTA owns all 512 bins and evaluates a DIFFERENT candidate:
// the 17-point scan takes one round of <= 3 evaluations per CTA, and the bisection is walked speculatively, the 7 nodes
// of the next three levels at once (each CTA derives its node's interval with the same arithmetic the sequential walk
// uses, so every visited midpoint and therefore sigma is bit-identical to sigma_update_kernel).  Results travel
// through distributed shared memory: thread 0 stores its block sum into every CTA's mailbox, cluster.sync() orders it.
constexpr int kSigmaCtas = 8;
__global__ void __cluster_dims__(kSigmaCtas, 1, 1) __launch_bounds__(kBins)
    sigma_update_cluster_kernel(const unsigned long long* __restrict__ hist, double mu, double pairs, double edges,
                                int exact_math, SigmaState* __restrict__ state, std::uint32_t* __restrict__ status,
                                RunState* run, double* pe_trace, double* sigma_trace) {
  using namespace sigma;
  namespace cg = cooperative_groups;
  // a queued round after the run has stopped: every CTA sees the same state (it only changes at the very end of this
  // kernel, after the last cluster.sync), so the whole cluster leaves together
  if (run && run_stopped(run)) return;
  cg::cluster_group cluster = cg::this_cluster();
  const int cta = static_cast<int>(cluster.block_rank());
  __shared__ double scratch[kBins / 32];
  __shared__ double mailbox[2][24];
  const int b = threadIdx.x;
  const double ec = static_cast<double>(hist[b]), nc = static_cast<double>(hist[kBins + b]);
  const double mid = (b + 0.5) * 12.0 / kBins;
  const double cap = state->sigma * 1.5;  // read before anybody writes the state (CTA 0, after the last sync)
  const double samples = block_sum(nc, scratch);
  const bool empty = block_sum(ec, scratch) + samples == 0.0;  // the same in every CTA: all return together
  // every CTA of the cluster is running (and its shared memory exists) before anybody stores into a peer's mailbox
  cluster.sync();
  if (empty) {  // optimize_sigma on an empty histogram is a config_error (slope.cpp:76); sigma stays what it was
    if (cta == 0 && b == 0) atomicOr(status + kStatEmptyTallies, 1u);
    if (cta == 0 && run) {
      __syncthreads();
      record_round(run, pe_trace, sigma_trace, 0.0, state->sigma, 1.0, status, hist);
    }
    return;
  }
  const double nw = samples > 0.0 ? (pairs - edges) / samples : 1.0;
  auto total = [&](double s, int which) {
    double v = 0.0;
    if (which == 0) {
      if (ec != 0.0) v += ec * cost_tail(mid, mu, s, true);
      if (nc != 0.0) v += nw * nc * cost_tail(mid, mu, s, false);
    } else if (which == 1) {
      if (ec != 0.0) v += ec * cost_dsigma(mid, mu, s, true);
      if (nc != 0.0) v += nw * nc * cost_dsigma(mid, mu, s, false);
    } else {
      if (ec != 0.0) v += ec * cost_floor(mid, mu, s, true);
      if (nc != 0.0) v += nw * nc * cost_floor(mid, mu, s, false);
    }
    return block_sum(v, scratch);
  };
  int parity = 0;
  auto post = [&](int slot, double v) {
    if (b == 0) {
      for (int r = 0; r < kSigmaCtas; ++r) *cluster.map_shared_rank(&mailbox[parity][slot], r) = v;
    }
  };

  // round 0: coarse geometric scan
  constexpr int kGrid = 17;
  double grid[kGrid];
#pragma unroll 1
  for (int i = 0; i < kGrid; ++i) grid[i] = 1e-3 * pow(16.0 / 1e-3, static_cast<double>(i) / (kGrid - 1));
#pragma unroll 1
  for (int i = cta; i < kGrid; i += kSigmaCtas) post(i, total(grid[i], 0));
  cluster.sync();
  double best_cost = 0.0;
  int best = 0;
  for (int i = 0; i < kGrid; ++i) {
    const double t = mailbox[parity][i];
    if (i == 0 || t < best_cost) best_cost = t, best = i;
  }
  parity ^= 1;
  double sigma_opt = grid[best];
  double lo = grid[best > 0 ? best - 1 : 0], hi = grid[best < kGrid - 1 ? best + 1 : kGrid - 1];

  // interval of heap node k (children of k: 2k+1 = left half, 2k+2 = right half) below (lo, hi)
  auto node_mid = [&](int k) {
    int path[3], depth = 0;
    for (int q = k; q > 0; q = (q - 1) >> 1) path[depth++] = (q & 1) ? 0 : 1;
    double nlo = lo, nhi = hi;
    for (int d = depth - 1; d >= 0; --d) {
      const double m = 0.5 * (nlo + nhi);
      if (path[d]) nlo = m; else nhi = m;
    }
    return 0.5 * (nlo + nhi);
  };
  int steps = 0;
  bool open = true;  // the bisection loop of optimize_sigma_detail is still running
  // consumes up to `levels` levels of the posted tree (slots base .. base + 2^levels - 2)
  auto walk = [&](int levels, int base) {
    int k = 0;
    for (int l = 0; l < levels && open; ++l) {
      if (!(hi - lo > 1e-4 && steps < 60)) {
        open = false;
        break;
      }
      ++steps;
      const double m = 0.5 * (lo + hi);
      const double f_mid = mailbox[parity][base + k];
      if (f_mid == 0.0) {
        lo = hi = m;
        open = false;
        break;
      }
      if ((f_mid > 0.0) == false) {  // same sign as f_lo (< 0 throughout): move the lower end
        lo = m;
        k = 2 * k + 2;
      } else {
        hi = m;
        k = 2 * k + 1;
      }
    }
  };

  // round 1: the derivative at both ends and the first two levels
  if (cta == 0) post(0, total(lo, 1));
  else if (cta == 1) post(1, total(hi, 1));
  else if (cta < 5) post(cta, total(node_mid(cta - 2), 1));
  cluster.sync();
  const bool bisect = mailbox[parity][0] < 0.0 && mailbox[parity][1] > 0.0;
  if (bisect) walk(2, 2); else open = false;
  parity ^= 1;
  while (open && hi - lo > 1e-4 && steps < 60) {
    if (cta < 7) post(cta, total(node_mid(cta), 1));
    cluster.sync();
    walk(3, 0);
    parity ^= 1;
  }

  // last round: acceptance test and the PE estimate of either outcome
  const double refined = 0.5 * (lo + hi);
  if (cta == 0) post(0, bisect ? total(refined, 0) : 0.0);
  else if (cta == 1) post(1, total(fmin(refined, cap), 2));
  else if (cta == 2) post(2, total(fmin(grid[best], cap), 2));
  cluster.sync();
  double pe_sum = mailbox[parity][2];
  if (bisect && mailbox[parity][0] <= best_cost) {
    sigma_opt = refined;
    pe_sum = mailbox[parity][1];
  }
  const double sigma_new = fmin(sigma_opt, cap);  // growth cap, engine.cpp:302-307
  if (cta == 0 && b == 0) {
    const double c1 = 2.0 / (3.14159265358979323846264338327950288 * kLn2);
    const double c2 = 1.0 / (2.50662827463100050241576528481 * kLn2);
    state->sigma = sigma_new;
    state->pe_estimate = pe_sum / pairs;
    state->nonedge_weight = nw;
    state->bisection_steps = steps;
    state->math.mu = mu;
    state->math.inv_sqrt2_sigma = 1.0 / (kSqrt2 * sigma_new);
    state->math.A = c1 / (sigma_new * sigma_new);
    state->math.B = c2 / (sigma_new * sigma_new * sigma_new);
    state->math.C = c2 / sigma_new;
    state->math.exact = exact_math;
  }
  if (cta == 0 && run) record_round(run, pe_trace, sigma_trace, pe_sum / pairs, sigma_new, nw, status, hist);
}

// best-PE snapshot (engine.cpp:316-319) without the host: see launch_snapshot_if_improved
__global__ void __launch_bounds__(kThreads) snapshot_if_improved_kernel(const float4* __restrict__ x0,
                                                                        const float4* __restrict__ x1,
                                                                        float4* __restrict__ dst, std::size_t floats,
                                                                        const RunState* __restrict__ run) {
  const unsigned long long count = run->count;
  if (run->improved_at != count) return;
  const float4* src = ((run->parity_base + count) & 1ull) ? x1 : x0;
  const std::size_t count4 = floats / 4, stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  const std::size_t t = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (std::size_t i = t; i < count4; i += stride) dst[i] = src[i];
  if (t < floats % 4) {  // tail of a buffer whose length is not a multiple of four floats (d <= 2)
    reinterpret_cast<float*>(dst)[4 * count4 + t] = reinterpret_cast<const float*>(src)[4 * count4 + t];
  }
}

__global__ void __launch_bounds__(kThreads) sum_tallies_kernel(const TallySources srcs, unsigned long long* __restrict__ dst) {
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= 2 * kBins) return;
  unsigned long long total = 0;
  for (int r = 0; r < srcs.count; ++r) total += srcs.hist[r][i];
  dst[i] = total;
}

__global__ void __launch_bounds__(kThreads) permute_rows_kernel(const float* __restrict__ in, std::uint32_t in_ld,
                                                                float* __restrict__ out, std::uint32_t out_ld,
                                                                std::uint32_t dim, std::uint32_t n,
                                                                const std::uint32_t* __restrict__ map, bool scatter) {
  const std::uint64_t total = static_cast<std::uint64_t>(n) * dim;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const std::uint32_t v = static_cast<std::uint32_t>(i / dim), col = static_cast<std::uint32_t>(i % dim);
    const std::uint32_t w = __ldg(map + v);
    const std::size_t from = static_cast<std::size_t>(scatter ? v : w) * in_ld + col;
    const std::size_t to = static_cast<std::size_t>(scatter ? w : v) * out_ld + col;
    out[to] = in[from];
  }
}

// exclusive scan of in[0..n) into out[0..n], out[n] = total: one 1024-thread block, 4 elements per thread and pass
constexpr std::uint32_t kScanSingleBlockMax = 1u << 14;  // beyond that the three-kernel scan wins (c2, n = 1e5: 50 vs 82 us)
__global__ void __launch_bounds__(1024) scan_single_block_kernel(std::uint32_t* __restrict__ in,
                                                                 std::uint32_t* __restrict__ out, std::uint32_t n,
                                                                 bool clear_input) {
  __shared__ std::uint32_t warp_tot[32];
  __shared__ std::uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (std::uint32_t base = 0; base < n; base += 4096) {
    const std::uint32_t i0 = base + threadIdx.x * 4;
    std::uint32_t v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = i0 + q < n ? in[i0 + q] : 0u;
      if (clear_input && i0 + q < n) in[i0 + q] = 0;
    }
    const std::uint32_t mine = v[0] + v[1] + v[2] + v[3];
    std::uint32_t inc = mine;
    for (int off = 1; off < 32; off <<= 1) {
      const std::uint32_t o = __shfl_up_sync(kFull, inc, off);
      if (lane >= off) inc += o;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const std::uint32_t w = warp_tot[lane];
      std::uint32_t winc = w;
      for (int off = 1; off < 32; off <<= 1) {
        const std::uint32_t o = __shfl_up_sync(kFull, winc, off);
        if (lane >= off) winc += o;
      }
      warp_tot[lane] = winc - w;
    }
    __syncthreads();
    std::uint32_t run = carry + warp_tot[warp] + inc - mine;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i0 + q < n) out[i0 + q] = run;
      run += v[q];
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = run;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

inline unsigned blocks_for(std::uint64_t work, unsigned per_block) {
  return static_cast<unsigned>((work + per_block - 1) / per_block);
}

// SM count of the CURRENT device (a process may drive contexts on several GPUs from several threads: nothing about a
// device is cached in a plain static)
constexpr int kMaxDevices = 64;
inline int current_device() {
  int device = 0;
  cudaGetDevice(&device);
  return device;
}
inline unsigned sm_count() {
  static std::atomic<int> cached[kMaxDevices] = {};
  const int device = current_device();
  int sms = device < kMaxDevices ? cached[device].load(std::memory_order_relaxed) : 0;
  if (sms == 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    sms = std::max(1, sms);
    if (device < kMaxDevices) cached[device].store(sms, std::memory_order_relaxed);
  }
  return static_cast<unsigned>(sms);
}
// grid-stride kernels: enough blocks for `work`, at most `per_sm` per SM
inline unsigned capped_blocks(std::uint64_t work, unsigned per_block, unsigned per_sm) {
  return static_cast<unsigned>(std::min<std::uint64_t>((work + per_block - 1) / per_block,
                                                       static_cast<std::uint64_t>(sm_count()) * per_sm));
}

}  // namespace

// ---------------------------------------------------------------------------------- launchers

int launch_validate_edges(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t m, std::uint32_t n,
                          std::uint32_t* flags, cudaStream_t stream) {
  if (m == 0) return 0;
  const unsigned blocks = capped_blocks(m, kThreads, 32);
  validate_edges_kernel<<<blocks, kThreads, 0, stream>>>(src, dst, m, n, flags);
  return 1;
}

int launch_hash_build(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t m, std::uint32_t n,
                      std::uint32_t hash_mask, std::uint32_t* hash_words, cudaStream_t stream) {
  if (m == 0) return 0;
  const unsigned blocks = capped_blocks(m, kThreads, 32);
  hash_build_kernel<<<blocks, kThreads, 0, stream>>>(src, dst, m, n, hash_mask, hash_words);
  return 1;
}

int launch_hash_popcount(const std::uint32_t* hash_words, std::uint64_t nwords, unsigned long long* total, cudaStream_t stream) {
  cudaMemsetAsync(total, 0, sizeof(unsigned long long), stream);
  const unsigned blocks = capped_blocks(nwords, kThreads, 16);
  hash_popcount_kernel<<<blocks, kThreads, 0, stream>>>(hash_words, nwords, total);
  return 1;
}

int launch_hash_summary(const std::uint32_t* hash_words, std::uint64_t nsummary, std::uint32_t* summary, cudaStream_t stream) {
  const unsigned blocks = capped_blocks(nsummary, kThreads, 16);
  hash_summary_kernel<<<blocks, kThreads, 0, stream>>>(hash_words, nsummary, summary);
  return 1;
}

int launch_probe(const std::uint32_t* hash_words, std::uint32_t hash_mask, std::uint32_t n, const std::uint32_t* i,
                 const std::uint32_t* j, std::uint64_t count, std::uint8_t* out, cudaStream_t stream) {
  if (count == 0) return 0;
  probe_kernel<<<blocks_for(count, kThreads), kThreads, 0, stream>>>(hash_words, hash_mask, n, i, j, count, out);
  return 1;
}

int launch_relabel_apply(std::uint32_t* src, std::uint32_t* dst, std::uint64_t m, const std::uint32_t* forward,
                         cudaStream_t stream) {
  if (m == 0) return 0;
  relabel_apply_kernel<<<capped_blocks(m, kThreads, 32), kThreads, 0, stream>>>(src, dst, m, forward);
  return 1;
}

int launch_csr_build(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t m, std::uint32_t n,
                     std::uint32_t* deg, std::uint32_t* rowptr, std::uint32_t* scratch, std::uint32_t* nbr,
                     std::uint32_t* eid_role, std::uint32_t* csr_src, cudaStream_t stream) {
  const unsigned blocks = capped_blocks(m, kThreads, 32);
  cudaMemsetAsync(deg, 0, static_cast<std::size_t>(n) * sizeof(std::uint32_t), stream);
  degree_count_kernel<<<blocks, kThreads, 0, stream>>>(src, dst, m, deg);
  const int scans = launch_scan(deg, rowptr, n, scratch, stream);
  cudaMemsetAsync(deg, 0, static_cast<std::size_t>(n) * sizeof(std::uint32_t), stream);  // reused as the row cursors
  csr_fill_kernel<<<blocks, kThreads, 0, stream>>>(src, dst, m, rowptr, deg, nbr, eid_role, csr_src);
  return 2 + scans;
}

int launch_sample(const SampleArgs& a, cudaStream_t stream) {
  if (a.slots == 0) return 0;
  sample_kernel<<<blocks_for(a.slots, kThreads * kSampleIlp), kThreads, 0, stream>>>(a);
  return 1;
}

int launch_spill_index(const SpillIndexArgs& a, cudaStream_t stream) {
  spill_index_kernel<<<1, 1024, 0, stream>>>(a);
  return 1;
}

int launch_sample_pack(const SampleArgs& a, const ExchangeArgs& x, cudaStream_t stream) {
  cudaMemsetAsync(x.send_count, 0, x.regions * sizeof(std::uint32_t), stream);
  if (x.spill) cudaMemsetAsync(x.spill_count, 0, sizeof(std::uint32_t), stream);
  if (x.own_slots == 0) return 0;
  sample_pack_kernel<<<blocks_for(x.own_slots, kThreads), kThreads, 2 * x.regions * sizeof(std::uint32_t), stream>>>(a, x);
  return 1;
}

int launch_publish_counts(const ExchangeArgs& x, cudaStream_t stream) {
  publish_counts_kernel<<<1, 32, 0, stream>>>(x);
  return 1;
}

int launch_bucket_records(const ExchangeArgs& x, std::uint32_t sources, std::uint32_t n, std::uint32_t* in_cnt,
                          std::uint32_t* in_off, std::uint32_t* rec_rank, std::uint32_t* in_anchor, std::uint32_t* scratch,
                          cudaStream_t stream) {
  cudaMemsetAsync(in_cnt, 0, static_cast<std::size_t>(n) * sizeof(std::uint32_t), stream);
  int launches = 0;
  const dim3 grid(blocks_for(x.capacity, kThreads * kRecIlp), sources);
  std::uint32_t* spill_rank = rec_rank + static_cast<std::size_t>(sources) * x.capacity;
  if (x.capacity) {
    count_records_kernel<<<grid, kThreads, 0, stream>>>(x, in_cnt, rec_rank);
    ++launches;
  }
  if (x.spill) {
    count_spill_kernel<<<sm_count() * 4, kThreads, 0, stream>>>(x, in_cnt, spill_rank);
    ++launches;
  }
  launches += launch_scan(in_cnt, in_off, n, scratch, stream);
  if (x.capacity) {
    scatter_records_kernel<<<grid, kThreads, 0, stream>>>(x, rec_rank, in_off, in_anchor);
    ++launches;
  }
  if (x.spill) {
    scatter_spill_kernel<<<sm_count() * 4, kThreads, 0, stream>>>(x, spill_rank, in_off, in_anchor);
    ++launches;
  }
  return launches;
}

std::uint32_t partition_grid(std::uint64_t slots) {
  return capped_blocks(slots, kPartThreads, 4);
}

int launch_sample_partition(const SampleArgs& a, const PartitionArgs& p, std::uint32_t* in_off, std::uint32_t* in_anchor,
                            cudaStream_t stream) {
  if (a.slots == 0) return 0;
  const std::uint32_t grid = p.grid;
  const std::size_t hist_smem = static_cast<std::size_t>(p.buckets) * sizeof(std::uint32_t);
  const std::size_t vert_smem = (static_cast<std::size_t>(1) << p.shift) * sizeof(std::uint32_t);
  {  // the attribute is per device: set it once on every device this process launches on
    static std::atomic<bool> configured[kMaxDevices] = {};
    const int device = current_device();
    if (device >= kMaxDevices || !configured[device].load(std::memory_order_relaxed)) {
      cudaFuncSetAttribute(bucket_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      if (device < kMaxDevices) configured[device].store(true, std::memory_order_relaxed);
    }
  }
  sample_count_kernel<<<grid, kPartThreads, hist_smem, stream>>>(a, p);
  bucket_column_scan_kernel<<<blocks_for(p.buckets, 128), 128, 0, stream>>>(p, grid);
  bucket_offsets_kernel<<<1, 1024, 0, stream>>>(p, in_off, a.n);
  partition_kernel<<<std::min<std::uint32_t>(grid, sm_count()), 1024, hist_smem, stream>>>(a, p);
  bucket_finalize_kernel<<<p.buckets, kPartThreads, vert_smem, stream>>>(p, a.n, in_off, in_anchor);
  return 5;
}

int launch_scan(std::uint32_t* in_cnt, std::uint32_t* in_off, std::uint32_t n, std::uint32_t* scratch,
                cudaStream_t stream, bool clear_input) {
  if (n <= kScanSingleBlockMax) {  // small graphs are launch-bound: one block walks the array with a running carry
    scan_single_block_kernel<<<1, 1024, 0, stream>>>(in_cnt, in_off, n, clear_input);
    return 1;
  }
  const unsigned tiles = blocks_for(n, kScanTile);
  scan_tile_sums_kernel<<<tiles, kThreads, 0, stream>>>(in_cnt, n, scratch);
  scan_tile_offsets_kernel<<<1, 1024, 0, stream>>>(scratch, tiles);
  scan_apply_kernel<<<tiles, kThreads, 0, stream>>>(in_cnt, n, scratch, in_off, clear_input);
  return 3;
}

int launch_scatter(const SampleArgs& a, const std::uint32_t* in_off, std::uint32_t* in_anchor, cudaStream_t stream) {
  if (a.slots == 0) return 0;
  // parts of at most 64 MB of in_anchor each (half of L2; every extra walk re-reads the index streams).  Measured on c4:
  // 84 MB window (k = 20 per vertex) 264 / 236 / 250 / 248 us with 1 / 2 / 3 / 4 parts, 125 MB window (2 per edge)
  // 716 / 376 / 425 / 494 us.  GEMPE_SCATTER_PARTS overrides (A/B hook)
  static const int forced = [] { const char* e = std::getenv("GEMPE_SCATTER_PARTS"); return e ? std::atoi(e) : 0; }();
  std::uint64_t parts = forced > 0 ? static_cast<std::uint64_t>(forced) : (a.slots * 4 + (64ull << 20) - 1) / (64ull << 20);
  parts = std::min<std::uint64_t>(std::max<std::uint64_t>(parts, 1), 8);
  const std::uint32_t part_rows = static_cast<std::uint32_t>((static_cast<std::uint64_t>(a.n) + parts - 1) / parts);
  const dim3 grid(blocks_for(a.slots, kThreads * kScatterIlp), static_cast<unsigned>(parts));
  scatter_kernel<<<grid, kThreads, 0, stream>>>(a, in_off, in_anchor, part_rows);
  return 1;
}

int launch_sort_buckets(const std::uint32_t* in_off, std::uint32_t* in_anchor, std::uint32_t n, cudaStream_t stream) {
  sort_buckets_kernel<<<blocks_for(static_cast<std::uint64_t>(n) * 32, kThreads), kThreads, 0, stream>>>(in_off, in_anchor, n);
  return 1;
}

int launch_permute_rows(const float* in, std::uint32_t in_ld, float* out, std::uint32_t out_ld, std::uint32_t dim,
                        std::uint32_t n, const std::uint32_t* map, bool scatter, cudaStream_t stream) {
  const std::uint64_t total = static_cast<std::uint64_t>(n) * dim;
  if (total == 0) return 0;
  const unsigned blocks = capped_blocks(total, kThreads, 64);
  permute_rows_kernel<<<blocks, kThreads, 0, stream>>>(in, in_ld, out, out_ld, dim, n, map, scatter);
  return 1;
}

int launch_unpermute_partners(const std::uint32_t* neg_own, const std::uint32_t* eid_role, std::uint64_t slots,
                              std::uint32_t* out, cudaStream_t stream) {
  if (slots == 0) return 0;
  unpermute_kernel<<<blocks_for(slots, kThreads), kThreads, 0, stream>>>(neg_own, eid_role, slots, out);
  return 1;
}

int launch_init_coords(float* x, std::uint32_t n, std::uint32_t dim, std::uint32_t ld, int rule, std::uint64_t seed,
                       double stddev, cudaStream_t stream) {
  const std::uint64_t total = static_cast<std::uint64_t>(n) * ld;
  if (total == 0) return 0;
  // SplitMix(mix_seed(seed, 0x1217)) for the reference rule (engine.cpp:121); other rules use their own key
  const std::uint64_t state0 = mix(seed, rule == 0 ? 0x1217ull : 0x1217ull + 0x100ull * rule);
  init_coords_kernel<<<blocks_for(total, kThreads), kThreads, 0, stream>>>(x, n, dim, ld, rule, state0, stddev);
  return 1;
}

namespace {
template <int LPR, int NV, int VEC, int TB, int U, bool PRECISE, bool FULL, int THREADS, int MINB>
void gather_batched_launch(const GatherArgs& a, std::uint32_t lo, std::uint32_t hi, cudaStream_t stream) {
  // persistent grid: as many blocks as fit on the device at once (occupancy query cached per instantiation)
  static std::atomic<int> cached[kMaxDevices] = {};  // per device: GPUs of one process need not be alike
  auto kernel = gather_batched_kernel<LPR, NV, VEC, TB, U, PRECISE, FULL, THREADS, MINB>;
  const int device = current_device();
  int resident_blocks = device < kMaxDevices ? cached[device].load(std::memory_order_relaxed) : 0;
  if (resident_blocks == 0) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, THREADS, 0);
    resident_blocks = static_cast<int>(sm_count()) * std::max(1, per_sm);
    if (device < kMaxDevices) cached[device].store(resident_blocks, std::memory_order_relaxed);
  }
  const unsigned needed = blocks_for(blocks_for(hi - lo, kGrab), THREADS / 32);
  const unsigned blocks = std::min<unsigned>(needed, static_cast<unsigned>(resident_blocks));
  cudaMemsetAsync(a.work_cursor, 0, sizeof(std::uint32_t), stream);
  kernel<<<blocks, THREADS, 0, stream>>>(a, lo, hi);
}
template <int LPR, int NV, int VEC, int TB, int U, int THREADS = 256, int MINB = 2>
void gather_batched_go(const GatherArgs& a, std::uint32_t lo, std::uint32_t hi, bool precise, cudaStream_t stream) {
  const bool full = a.ld == static_cast<std::uint32_t>(LPR * NV * VEC);
  if (precise) {  // the double chain needs the registers: never more than 4 blocks per SM
    constexpr int kMinB = MINB > 4 ? 4 : MINB;
    if (full) gather_batched_launch<LPR, NV, VEC, TB, U, true, true, THREADS, kMinB>(a, lo, hi, stream);
    else gather_batched_launch<LPR, NV, VEC, TB, U, true, false, THREADS, kMinB>(a, lo, hi, stream);
  } else {
    if (full) gather_batched_launch<LPR, NV, VEC, TB, U, false, true, THREADS, MINB>(a, lo, hi, stream);
    else gather_batched_launch<LPR, NV, VEC, TB, U, false, false, THREADS, MINB>(a, lo, hi, stream);
  }
}
}  // namespace

int launch_gather(const GatherArgs& a, std::uint32_t lo, std::uint32_t hi, bool precise, cudaStream_t stream) {
  if (hi <= lo) return 0;
  const std::uint32_t ld = a.ld;
  if (ld <= 4) {  // one thread per work item
    const unsigned blocks = blocks_for(hi - lo, kThreads);
    if (ld == 1) {
      if (precise) gather_thread_kernel<1, true><<<blocks, kThreads, 0, stream>>>(a, lo, hi);
      else gather_thread_kernel<1, false><<<blocks, kThreads, 0, stream>>>(a, lo, hi);
    } else if (ld == 2) {
      if (precise) gather_thread_kernel<2, true><<<blocks, kThreads, 0, stream>>>(a, lo, hi);
      else gather_thread_kernel<2, false><<<blocks, kThreads, 0, stream>>>(a, lo, hi);
    } else {
      if (precise) gather_thread_kernel<4, true><<<blocks, kThreads, 0, stream>>>(a, lo, hi);
      else gather_thread_kernel<4, false><<<blocks, kThreads, 0, stream>>>(a, lo, hi);
    }
    return 1;
  }
  //                          LPR NV VEC TB U
  // narrow rows need few registers: 128-thread blocks at 8-12 per SM (c3 graph, dimension overridden: d = 8 -40 %,
  // d = 16 -24 %, d = 32 -24 %, d = 64 -13 % against 256-thread blocks at 2 per SM / 16 rows at 5 per SM)
  if (ld <= 8) gather_batched_go<2, 1, 4, 2, 2, 128, 12>(a, lo, hi, precise, stream);
  else if (ld <= 16) gather_batched_go<4, 1, 4, 4, 2, 128, 8>(a, lo, hi, precise, stream);
  else if (ld <= 32) gather_batched_go<8, 1, 4, 8, 1, 128, 8>(a, lo, hi, precise, stream);
  // d = 64 (c3, gather ms): 16 lanes per row, 8 rows per group, 64 registers 0.269; 8 lanes per row, 4 groups x 4 rows, 80
  // registers 0.289 (-DGEMPE_D64_ROW_LANES=8)
#ifndef GEMPE_D64_ROW_LANES
#define GEMPE_D64_ROW_LANES 16
#endif
#if GEMPE_D64_ROW_LANES == 16
  else if (ld <= 64) gather_batched_go<16, 1, 4, 8, 1, 128, 8>(a, lo, hi, precise, stream);  // 8 rows per group, 32 warps/SM
#else
  else if (ld <= 64) gather_batched_go<8, 2, 4, 4, 1, 128, 6>(a, lo, hi, precise, stream);
#endif
#ifndef GEMPE_D128_ROW_LANES
#define GEMPE_D128_ROW_LANES 32
#endif
  // d = 128 on c4 / c5 (40-round / 3-round runs under the power cap, gather ms): one warp per row at 96 registers and 20
  // warps/SM 4.43 / 86.5 (alone: 4.17, 2.19 G warp instructions); 8 lanes per row at 128 registers and 16 warps/SM 4.59 /
  // 89.3 (alone: 4.26, 1.75 G); 16 lanes per row 5.12 / 97.8.  The kernel wants warps more than it wants fewer
  // instructions (3 instead of 4 resident blocks of the 8-lane shape: 5.12), so one warp per row is the default.
#if GEMPE_D128_ROW_LANES == 32
  else if (ld <= 128) gather_batched_go<32, 1, 4, 16, 1, 128, 5>(a, lo, hi, precise, stream);
#elif GEMPE_D128_ROW_LANES == 16
  else if (ld <= 128) gather_batched_go<16, 2, 4, 8, 1, 128, 5>(a, lo, hi, precise, stream);
#else  // 8 lanes per row, 4 rows per group: fewest instructions, but own row + accumulator take 32 registers -> 16 warps/SM
  else if (ld <= 128) gather_batched_go<8, 4, 4, 4, 1, 128, 4>(a, lo, hi, precise, stream);
#endif
  // wider rows: 64 row registers per lane as well (8 / 4 rows per batch), 16 warps/SM (d = 256: -19 %, d = 512: -10 %
  // against 4 / 2 rows in 256-thread blocks)
  else if (ld <= 192) gather_batched_go<16, 3, 4, 8, 1, 128, 4>(a, lo, hi, precise, stream);  // 2 half-warps x 8 rows
  else if (ld <= 256) gather_batched_go<32, 2, 4, 8, 1, 128, 4>(a, lo, hi, precise, stream);
  else if (ld <= 384) gather_batched_go<32, 3, 4, 4, 1, 128, 4>(a, lo, hi, precise, stream);
  else if (ld <= 512) gather_batched_go<32, 4, 4, 4, 1, 128, 4>(a, lo, hi, precise, stream);
  else gather_batched_go<32, 8, 4, 1, 1>(a, lo, hi, precise, stream);  // own row + accumulator already take 64 registers
  return 1;
}

int launch_pe_collect(const PeCollectArgs& p, cudaStream_t stream) {
  if (p.m == 0) return 0;
  const std::uint64_t work = p.m * (1 + static_cast<std::uint64_t>(p.samples_per_edge));
  const unsigned blocks = capped_blocks(work, kThreads, 64);
  pe_collect_kernel<<<blocks, kThreads, 0, stream>>>(p);
  return 1;
}

int launch_pe_sum(const float* dist, std::uint64_t count, double mu, double sigma, bool is_edge, int which, double* total,
                  unsigned long long* valid, cudaStream_t stream) {
  if (count == 0) return 0;
  const unsigned blocks = capped_blocks(count, kThreads * 4, 8);
  pe_sum_kernel<<<blocks, kThreads, 0, stream>>>(dist, count, mu, sigma, is_edge ? 1 : 0, which, total, valid);
  return 1;
}

int launch_sigma_update(const unsigned long long* hist, double mu, double pairs, double edges, int exact_math,
                        SigmaState* state, std::uint32_t* status, bool single_block, RunState* run, double* pe_trace,
                        double* sigma_trace, cudaStream_t stream) {
  if (single_block) {
    sigma_update_kernel<<<1, kBins, 0, stream>>>(hist, mu, pairs, edges, exact_math, state, status, run, pe_trace, sigma_trace);
  } else {
    sigma_update_cluster_kernel<<<kSigmaCtas, kBins, 0, stream>>>(hist, mu, pairs, edges, exact_math, state, status, run,
                                                                  pe_trace, sigma_trace);
  }
  return 1;
}

int launch_sum_tallies(const TallySources& srcs, unsigned long long* dst, cudaStream_t stream) {
  sum_tallies_kernel<<<blocks_for(2 * kBins, kThreads), kThreads, 0, stream>>>(srcs, dst);
  return 1;
}

int launch_snapshot_if_improved(const float* x0, const float* x1, float* dst, std::size_t floats, const RunState* run,
                                cudaStream_t stream) {
  if (floats == 0) return 0;
  snapshot_if_improved_kernel<<<capped_blocks(floats / 4 + 1, kThreads, 8), kThreads, 0, stream>>>(
      reinterpret_cast<const float4*>(x0), reinterpret_cast<const float4*>(x1), reinterpret_cast<float4*>(dst), floats, run);
  return 1;
}

}  // namespace gempe
