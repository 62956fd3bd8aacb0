// Launch interface between the context (host) and the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gempe {

constexpr int kBins = 512;
constexpr std::uint32_t kNoHub = 0xffffffffu;
constexpr std::uint32_t kNotLocal = 0xffffffffu;

// status word layout (device u32[8])
enum StatusSlot { kStatNonFinite = 0, kStatRetryCap = 1, kStatDrawsLo = 2, kStatDrawsHi = 3, kStatExchangeOverflow = 4,
                  kStatEmptyTallies = 5 };

// Per-round scalars of parabola_impl (sigmoid.hpp:88-101), folded on the host in double:
//   u = (delta - mu) * inv_sqrt2_sigma,  w = A g^2 + sign B (delta-mu) g,  d = delta + sign C g / w.
struct RoundMath {
  double mu;
  double inv_sqrt2_sigma;  // 1 / (sqrt(2) sigma)
  double A;                // 2 / (pi ln2 sigma^2)
  double B;                // 1 / (sqrt(2 pi) ln2 sigma^3)
  double C;                // 1 / (sqrt(2 pi) ln2 sigma)
  int exact;               // 1: exp(-x^2)/erfc(x), 0: piecewise tables
};

// Device-resident sigma feedback (sigma_update_kernel): the state after the latest round's tallies.
struct SigmaState {
  double sigma;
  double pe_estimate;
  double nonedge_weight;
  int bisection_steps;
  int pad;
  RoundMath math;  // folded constants of `sigma` for the next round's gather
};

// Device-resident bookkeeping of a run of iterations queued without host round trips (EmbeddingEngine::run,
// engine.cpp:349-373): the sigma kernel of every completed round appends the PE estimate, tracks the best PE and evaluates
// the convergence window; a round whose turn comes after the run has stopped (converged, failed, or `stop_at` rounds
// done) does nothing.  One instance per context, read back by the host every few rounds.
struct RunState {
  unsigned long long count;        // rounds completed == PE values recorded == index of the next round's sample streams
  unsigned long long stop_at;      // rounds with count >= stop_at are skipped (max_iters / relabel boundary / batch end)
  unsigned long long batch_base;   // rounds done when the current batch was queued: round r of the batch samples the streams
                                   // of iteration first_iter + batch_base + r (set by the host, stable while the batch runs)
  unsigned long long fail_iter;    // round that raised the first failure flag
  unsigned long long draws;        // LCG draws of the last completed round
  double best_pe;                  // minimum of the trace so far (engine.cpp:316-319)
  double tol;                      // convergence_tol
  int window;                      // convergence_window
  int converged;                   // engine.cpp:353-367 held after some round
  int failed;                      // a completed round left a failure flag in sticky_status
  int parity_base;                 // the current coordinates are buffer (parity_base + count) & 1
  unsigned long long improved_at;  // value of `count` after the latest round that set a new PE minimum (0: none yet)
  std::uint32_t sticky_status[8];  // OR of the rounds' status words
  std::uint32_t trace_cap;         // capacity of pe_trace / sigma_trace
  std::uint32_t pad;
  double last_nonedge_weight;      // of the last completed round
  unsigned long long last_hist[2 * kBins];  // tallies of the last completed round
};
// true when the round whose kernels read this must not run
#if defined(__CUDACC__)
__device__ __forceinline__ bool run_stopped(const RunState* r) {
  return r->converged || r->failed || r->count >= r->stop_at;
}
#endif

// knots[17] a[16] b[16] c[16] per table (the lo/hi clamps are the first/last knot).
struct DeviceTables {
  double erf[65];
  double ratio[65];
};

// Vertex ownership under sharding: block-cyclic over work ids, block = block_rows rows:
// owner(v) = (v / block_rows) % world.  world == 1 => everything is local.
struct Ownership {
  std::uint32_t block_rows;
  std::uint32_t world;
  std::uint32_t rank;
};

struct SampleArgs {
  std::uint32_t n;
  std::uint64_t slots;            // S
  int neg_mode;                   // 0 PER_EDGE_2 (slot = CSR position), 1 PER_VERTEX_K (slot = v*k+draw)
  std::uint32_t k;
  int rng;                        // 0 reference replay, 1 philox
  std::uint64_t stream_base;      // mix(seed, iter)  (reference) / seed (philox)
  std::uint64_t iter;
  // iteration index on the device (RunState::count): when non-null the round's index is iter + *iter_dev and the
  // stream base is derived from `seed` in the kernel, so one captured launch sequence serves every round
  std::uint64_t seed;
  const unsigned long long* iter_dev;
  const std::uint32_t* csr_src;   // PER_EDGE_2: anchor of each CSR position
  const std::uint32_t* eid_role;  // PER_EDGE_2: 2*edge + role (role 0: anchor is src[e], 1: dst[e])
  const std::uint32_t* hash_words;  // bit-packed direct-mapped table, 2^bits bits
  const std::uint32_t* hash_summary;  // optional: one bit per 4 cells ("any set"), null when the table itself fits L2
  std::uint32_t hash_mask;        // 2^bits - 1
  std::uint32_t* neg_own;         // out: accepted partner per slot
  std::uint32_t* in_cnt;          // in/out: per-vertex count of incoming samples (zeroed before)
  std::uint32_t* in_rank;         // out: arrival rank of the slot inside its partner's bucket
  std::uint32_t* status;
  Ownership own;
  // slotted buckets (bucket_mode 4): every vertex owns `in_stride` slots of in_anchor; the sampler stores the anchor at
  // slot (partner * in_stride + arrival rank) itself -- no scan, no scatter pass.  The few samples whose partner's slots are
  // full go to the spill list, indexed afterwards by launch_spill_index.  in_stride == 0: off.
  std::uint32_t in_stride;
  std::uint32_t* in_anchor;
  uint2* spill;                   // (partner, anchor)
  std::uint32_t* spill_count;
  std::uint32_t spill_capacity;
};

// Slotted buckets, overflow side: `spill_count` records (partner, anchor) that did not fit their partner's slots.
struct SpillIndexArgs {
  std::uint32_t n;
  const uint2* spill;
  const std::uint32_t* spill_count;
  std::uint32_t spill_capacity;
  std::uint32_t* cnt;     // [n] scratch, zero on entry and on exit
  std::uint32_t* off;     // [n + 1] exclusive offsets of the spilled anchors per partner (valid when spill_count > 0)
  std::uint32_t* anchor;  // [spill_capacity] spilled anchors grouped by partner
};
int launch_spill_index(const SpillIndexArgs& a, cudaStream_t stream);

constexpr int kMaxPeers = 15;  // other ranks whose X_{t+1} copy this rank writes directly (world <= 16)

// Sharded sampling with an exchange step: this rank samples the streams of the anchors it owns and packs
// (partner, anchor) records by destination rank; after the all-to-all it buckets the records it received.
struct ExchangeArgs {
  std::uint64_t own_slots;           // sample streams anchored at vertices this rank owns
  std::uint32_t ranges;              // owned blocks (comm chunks)
  const std::uint64_t* first_slot;   // [ranges] global slot id of the first own slot of block c
  const std::uint64_t* prefix;       // [ranges + 1] own slots before block c
  std::uint32_t regions;             // destinations: the ranks (exchange), or contiguous vertex ranges of one rank
  std::uint32_t region_rows;         // 0: destination = owner rank of the partner; else destination = partner / region_rows
  std::uint32_t capacity;            // records per (source, destination) region
  uint2* send;                       // [world][capacity]
  std::uint32_t* send_count;         // [world]
  const uint2* recv;                 // [world][capacity]
  const std::uint32_t* recv_count;   // [world]
  // one rank, vertex ranges as destinations: records that do not fit their range's region (partners far from uniform
  // over the ranges, e.g. structured ids without the random relabelling) go to a common spill area, bucketed after
  // the regions -- correct for any input, only slower.  Null across ranks (a record must reach its owner).
  uint2* spill;
  std::uint32_t* spill_count;
  std::uint32_t spill_capacity;
  // direct exchange (every peer's receive buffers opened in this process): the pack kernel stores a record for rank d
  // straight into the region reserved for THIS rank in d's receive buffer -- no all-to-all follows.  Null otherwise.
  int direct;
  uint2* dest_region[kMaxPeers + 1];          // [world] region `rank` of rank d's receive buffer (current parity)
  std::uint32_t* dest_count[kMaxPeers + 1];   // [world] slot `rank` of rank d's receive counts (current parity)
};

// Two-level counting sort of the accepted samples by partner (large n).
struct PartitionArgs {
  std::uint32_t shift;          // coarse bucket = partner >> shift (2^shift vertices per bucket)
  std::uint32_t buckets;        // ceil(n / 2^shift) <= 8192
  std::uint32_t grid;           // persistent blocks of the sampling / partition passes
  std::uint32_t* block_hist;    // [grid][buckets] per-block bucket counts, then run bases
  std::uint32_t* bucket_off;    // [buckets + 1]
  uint2* records;               // [S] (partner, anchor), grouped by coarse bucket
};


// One work item of the gather: a vertex, or one slice of a hub's adjacency.  32 bytes, written once per graph build, so
// an item starts with two 16-byte loads instead of a chain of dependent ones (items -> rowptr -> ...); the four items
// of a claim share one 128-byte line.
struct ItemDesc {
  std::uint32_t u;       // vertex (work id)
  std::uint32_t off_a;   // first adjacency position of the slice (index into nbr)
  std::uint32_t len_a;   // adjacency positions in the slice
  std::uint32_t off_b;   // first own-sample slot (index into neg_own): u*k, or off_a in PER_EDGE_2
  std::uint32_t len_b;   // own samples taken by this item: k on a vertex's first item (0 on later slices), len_a in PER_EDGE_2
  std::uint32_t first;   // 1: first item of the vertex -- it also takes the incoming samples (in_off[u] .. in_off[u+1])
  std::uint32_t hub;     // hub id, kNoHub for an unsplit vertex
  std::uint32_t sub;     // slice index inside the hub
};
static_assert(sizeof(ItemDesc) == 32, "two 16-byte loads per item");

// fp32 view of the FastMath tables for the default (non-PRECISE) kernels, laid out for direct indexing: the ratio table's
// knots (-1 ... 8) are all multiples of 0.05, so every cell [-1 + 0.05 i, -1 + 0.05 (i+1)) lies inside ONE segment and
// carries that segment's quadratic {a, b, c}; the erf table's 16 segments are uniform (width 0.375).
constexpr int kRatioCells = 180;
constexpr int kErfSegments = 16;
constexpr int kTableF32Entries = kRatioCells + kErfSegments;  // float4 {a, b, c, 0} each

struct GatherArgs {
  const float* x_cur;
  float* x_next;
  // fused update + broadcast: every updated row is also stored into the X_{t+1} buffer of each peer rank (peer
  // device memory over NVLink, opened through CUDA IPC), so no all-gather follows the kernel
  int n_peers;
  float* peer_next[kMaxPeers];
  std::uint32_t n, dim, ld;
  const std::uint32_t* nbr;        // 2m, both directions
  const std::uint32_t* neg_own;
  const std::uint32_t* in_off;     // n+1
  const std::uint32_t* in_anchor;
  // slotted buckets (in_stride != 0): incoming samples of u are in_anchor[u*in_stride .. + min(in_cnt[u], in_stride)), plus,
  // when *spill_count != 0, spill_anchor[spill_off[u] .. spill_off[u+1])
  std::uint32_t in_stride;
  const std::uint32_t* in_cnt;
  const std::uint32_t* spill_count;
  const std::uint32_t* spill_off;
  const std::uint32_t* spill_anchor;
  const ItemDesc* items;
  const std::uint32_t* hub_first;  // first partial slot of hub h
  const std::uint32_t* hub_items;  // number of items of hub h
  std::uint32_t* hub_arrived;      // arrival counters (zero between rounds)
  double* part_y;                  // partial slots x ld
  double* part_z;
  unsigned long long* hist;        // [2*kBins]: edge tallies then non-edge tallies
  std::uint32_t* status;
  std::uint32_t* work_cursor;      // persistent-warp work queue head (reset before every launch)
  double* cap_y;                   // optional capture (n*dim, n), null when off
  double* cap_z;
  RoundMath math;
  const RoundMath* math_dev;       // non-null: read the round's constants from device memory (device sigma feedback)
  const RunState* run;             // non-null: the launch does nothing once the run has stopped
  DeviceTables tab;                // double tables (PRECISE kernels)
  const float4* tab_f32;           // kTableF32Entries cells in device memory (default kernels), see above
};

// ---- launchers (all asynchronous on `stream`; return the number of kernels launched) ---------------
// flags |= 1 when an endpoint is >= n, |= 2 on a self-loop
int launch_validate_edges(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t m, std::uint32_t n,
                          std::uint32_t* flags, cudaStream_t stream);
int launch_hash_build(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t m, std::uint32_t n,
                      std::uint32_t hash_mask, std::uint32_t* hash_words, cudaStream_t stream);
int launch_hash_popcount(const std::uint32_t* hash_words, std::uint64_t nwords, unsigned long long* total, cudaStream_t stream);
// summary bit g = some cell of cells 4g .. 4g+3 is set; nsummary = words / 4
int launch_hash_summary(const std::uint32_t* hash_words, std::uint64_t nsummary, std::uint32_t* summary, cudaStream_t stream);
constexpr int kHashSummaryShift = 2;  // cells per summary bit = 4 (kernels.cu: kSummaryShift)
// construction on the device: relabel application and the both-direction CSR (row order = atomic arrival order)
int launch_relabel_apply(std::uint32_t* src, std::uint32_t* dst, std::uint64_t m, const std::uint32_t* forward,
                         cudaStream_t stream);
int launch_csr_build(const std::uint32_t* src, const std::uint32_t* dst, std::uint64_t m, std::uint32_t n,
                     std::uint32_t* deg, std::uint32_t* rowptr, std::uint32_t* scratch, std::uint32_t* nbr,
                     std::uint32_t* eid_role, std::uint32_t* csr_src, cudaStream_t stream);
int launch_probe(const std::uint32_t* hash_words, std::uint32_t hash_mask, std::uint32_t n,
                 const std::uint32_t* i, const std::uint32_t* j, std::uint64_t count, std::uint8_t* out,
                 cudaStream_t stream);
int launch_sample(const SampleArgs& a, cudaStream_t stream);
int launch_sample_pack(const SampleArgs& a, const ExchangeArgs& x, cudaStream_t stream);
// direct exchange: fill counts of this rank's regions on every destination (after launch_sample_pack, same stream)
int launch_publish_counts(const ExchangeArgs& x, cudaStream_t stream);
int launch_bucket_records(const ExchangeArgs& x, std::uint32_t sources, std::uint32_t n, std::uint32_t* in_cnt,
                          std::uint32_t* in_off, std::uint32_t* rec_rank, std::uint32_t* in_anchor, std::uint32_t* scratch,
                          cudaStream_t stream);
std::uint32_t partition_grid(std::uint64_t slots);
// sampling + bucketing by partner with streaming traffic only (fills neg_own, in_off[n+1], in_anchor)
int launch_sample_partition(const SampleArgs& a, const PartitionArgs& p, std::uint32_t* in_off, std::uint32_t* in_anchor,
                            cudaStream_t stream);
// exclusive scan of in_cnt[n] into in_off[n+1]; scratch must hold ceil(n/4096)+1 words
// exclusive scan, in_off[n] = total; clear_input zeroes in_cnt behind the read (per-round counters)
int launch_scan(std::uint32_t* in_cnt, std::uint32_t* in_off, std::uint32_t n, std::uint32_t* scratch,
                cudaStream_t stream, bool clear_input = false);
int launch_scatter(const SampleArgs& a, const std::uint32_t* in_off, std::uint32_t* in_anchor,
                   cudaStream_t stream);
// sorts every incoming bucket ascending (deterministic mode)
int launch_sort_buckets(const std::uint32_t* in_off, std::uint32_t* in_anchor, std::uint32_t n,
                        cudaStream_t stream);
// reorders neg_own (CSR order) into reference slot order 2e+draw (test hook)
// Row permutation of a coordinate matrix: gather (out[v] = in[map[v]]) or scatter (out[map[v]] = in[v]); dim floats
// per row, row pitches in floats.
int launch_permute_rows(const float* in, std::uint32_t in_ld, float* out, std::uint32_t out_ld, std::uint32_t dim,
                        std::uint32_t n, const std::uint32_t* map, bool scatter, cudaStream_t stream);
int launch_unpermute_partners(const std::uint32_t* neg_own, const std::uint32_t* eid_role, std::uint64_t slots,
                              std::uint32_t* out, cudaStream_t stream);
// gradient + update of work items [item_lo, item_hi).  precise: reference-exact double pair_distance.
int launch_gather(const GatherArgs& a, std::uint32_t item_lo, std::uint32_t item_hi, bool precise, cudaStream_t stream);
// optimize_sigma + growth cap + PE estimate on the device tallies; updates *state (and state->math)
// pe_sampled (metrics.cpp:166-213): distances of all edges and of samples_per_edge sampled non-edges per edge
struct PeCollectArgs {
  const float* x;
  std::uint32_t n, dim, ld;
  std::uint64_t m;
  const std::uint32_t* src;  // work edge list
  const std::uint32_t* dst;
  const std::uint32_t* rowptr;
  const std::uint32_t* hash_words;
  const std::uint32_t* hash_summary;
  std::uint32_t hash_mask;
  std::uint32_t samples_per_edge;
  std::uint64_t seed;
  float* edge_dist;     // [m]
  float* nonedge_dist;  // [m * samples_per_edge], NaN where no sample could be drawn
};
int launch_pe_collect(const PeCollectArgs& p, cudaStream_t stream);
int launch_pe_sum(const float* dist, std::uint64_t count, double mu, double sigma, bool is_edge, int which, double* total,
                  unsigned long long* valid, cudaStream_t stream);
// (an empty histogram sets status[kStatEmptyTallies] and leaves the state alone); single_block selects the one-CTA
// kernel instead of the 8-CTA cluster (A/B switch)
// run / pe_trace / sigma_trace (optional): device-side run bookkeeping, see RunState
int launch_sigma_update(const unsigned long long* hist, double mu, double pairs, double edges, int exact_math,
                        SigmaState* state, std::uint32_t* status, bool single_block, RunState* run, double* pe_trace,
                        double* sigma_trace, cudaStream_t stream);
// best-PE snapshot on the device (engine.cpp:316-319): when the latest completed round set a new PE minimum, copies the
// current coordinates -- buffer (parity_base + count) & 1 of {x0, x1} -- to dst.  `floats` is a multiple of 4.
int launch_snapshot_if_improved(const float* x0, const float* x1, float* dst, std::size_t floats, const RunState* run,
                                cudaStream_t stream);
// job-wide tallies of a sharded round inside one process: dst[i] = sum over `count` ranks of srcs[r][i] (2*kBins counters;
// the sources are the ranks' device tallies, peer memory included)
struct TallySources {
  const unsigned long long* hist[kMaxPeers + 1];
  int count;
};
int launch_sum_tallies(const TallySources& srcs, unsigned long long* dst, cudaStream_t stream);
int launch_init_coords(float* x, std::uint32_t n, std::uint32_t dim, std::uint32_t ld, int rule,
                       std::uint64_t seed, double stddev, cudaStream_t stream);

}  // namespace gempe
