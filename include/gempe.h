/* gempe.h -- C ABI of the B200-native GEMPE hot path (libgempe_b200.so).
 *
 * Drop-in boundary for ONE path of the reference library "entropy-embed"
 * (/root/reference/proj; file:line citations below are relative to it): one Jacobi round of
 * EmbeddingEngine::run_single_iteration (src/engine.cpp:278-325) -- edge terms, hash-verified
 * sampled non-edge terms, per-vertex reduction of (y, z) and the update x = y / z -- plus the
 * one-time preparation that defines its inputs (relabel, initial coordinates, edge hash set).
 *
 * The reference has no FFI layer; its boundary is the C++ surface of
 * include/entropy_embed/engine.hpp:112-171.  Every entry point below names the reference
 * interface it replaces.  Plain pointers and sizes only; all host pointers are caller-owned and
 * copied.  One context per GPU and per host thread; contexts are not re-entrant (same contract
 * as the reference engine).
 *
 * Return codes mirror the CLI's exit codes (tools/embed_main.cpp:214-230):
 *   0 ok, 1 config_error, 2 data_error (incl. near_complete_graph_error), 3 divergence_error,
 *   4 CUDA runtime failure (no reference analogue; there is NO CPU fallback).
 */
#ifndef GEMPE_H_
#define GEMPE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEMPE_OK 0
#define GEMPE_ERR_CONFIG 1
#define GEMPE_ERR_DATA 2
#define GEMPE_ERR_DIVERGENCE 3
#define GEMPE_ERR_CUDA 4

#define GEMPE_HIST_BINS 512 /* include/entropy_embed/histogram.hpp:15-16: 512 bins over [0,12) */

/* negative-sampling scheme */
#define GEMPE_NEG_PER_EDGE_2 0   /* reference: 2 draws per edge (src/engine.cpp:227-249) */
#define GEMPE_NEG_PER_VERTEX_K 1 /* BASELINE.json: k draws per vertex, stream key (seed,iter,v,draw) */
/* math policy for e^{-x^2}/erfc(x) */
#define GEMPE_MATH_TABLES 0 /* FastMath piecewise tables (include/entropy_embed/piecewise.hpp:72-79) */
#define GEMPE_MATH_EXACT 1  /* ExactMath (include/entropy_embed/sigmoid.hpp:61-65) */
/* sample-stream generator */
#define GEMPE_RNG_REFERENCE 0 /* expand_seed32 + LCG replay (include/entropy_embed/rng.hpp:31-34,82-86) */
#define GEMPE_RNG_PHILOX 1    /* Philox4x32-10 keyed (seed,iter), counter (slot,try); not a parity mode */
/* initial-coordinate rule */
#define GEMPE_INIT_REFERENCE 0 /* init_embedding: U[0,1) SplitMix stream (src/engine.cpp:116-124) */
#define GEMPE_INIT_UNIFORM_PM1 1 /* U(-1,1)  (BASELINE.json configs 1-2) */
#define GEMPE_INIT_NORMAL 2      /* N(0, std^2) (BASELINE.json configs 3-5, std = 0.01) */

typedef struct gempe_ctx gempe_ctx;

typedef struct gempe_options {
  uint32_t dim;           /* embedding dimension d >= 1 (EmbeddingEngine ctor, src/engine.cpp:152) */
  int32_t hash_bits;      /* 0 = auto (next pow2 >= 64 m, cap 2^31), else [1,31] (src/hash_set.cpp:13-24) */
  uint64_t seed;          /* run seed */
  int32_t neg_mode;       /* GEMPE_NEG_* */
  uint32_t negatives;     /* k for PER_VERTEX_K (ignored for PER_EDGE_2) */
  int32_t math;           /* GEMPE_MATH_* */
  int32_t rng;            /* GEMPE_RNG_* */
  int32_t relabel;        /* 1 = apply random_relabel(mix_seed(seed,0xA11BE11)) as the reference ctor does
                             (src/engine.cpp:161-163); 0 = ids are used as work ids */
  int32_t device;         /* CUDA device ordinal */
  int32_t rank, world;    /* vertex sharding, one process per GPU; world = 1 for a single GPU */
  int32_t comm_chunks;    /* all-gather pipeline depth (>= 1): ownership blocks per rank */
  uint32_t chunk_entries; /* hub split: max adjacency entries per work item (0 = default) */
  int32_t deterministic;  /* 1 = sort incoming-sample buckets so the fp32 sums are run-to-run identical */
  int32_t precise_distance; /* 1 = pair_distance exactly as src/engine.cpp:45-52 (double differences); 0 = fp32
                             differences with double cross-lane sum and exact-tally recheck (default) */
  int32_t kernel_variant; /* must be 0 (one gather kernel per row width: thread per item for d <= 4, batched warp per
                             item above); the A/B variants of round 1 are retired, the field keeps the layout */
  int32_t bucket_mode;    /* incoming-sample bucketing: 0 = auto, 1 = per-partner atomics + scan + scatter,
                             2 = two-level counting sort (streaming traffic only),
                             3 = one radix pass by contiguous vertex range, then per-partner atomics range by range
                                 (auto for n >= 2^22 on one rank),
                             4 = slotted buckets: S/n + 6 sigma + 8 slots per vertex, the sampler places each anchor at
                                 its arrival rank itself (no scan, no scatter pass; overflow goes to an indexed spill
                                 list).  Auto on one rank while the slot array fits L2 (<= 48 MB), unless `deterministic`
                                 (sorted buckets: mode 1) */
  int32_t exchange;       /* sharded sampling: 0 = every rank enumerates all sample streams and keeps the partners it
                             owns (no exchange step); 1 = a rank samples only the streams of its own anchors, packs
                             (partner, anchor) records per destination rank and the ranks exchange them with one
                             equal-split all-to-all per round (gempe_exchange_layout / gempe_bucket_received);
                             2 = as 1, and a single rank (world = 1) also leaves the exchange to the caller */
} gempe_options;

/* Fills *opt with defaults (dim must still be set). */
void gempe_default_options(gempe_options* opt);

/* Replaces EmbeddingEngine::EmbeddingEngine (src/engine.cpp:143-180): copies the graph (ORIGINAL ids),
 * relabels, builds the edge hash set, the both-direction CSR and the work-item table on `device`, and
 * initialises coordinates with the reference rule.  n <= 1 or m == 0 yields a degenerate context
 * (gempe_is_degenerate) on which gempe_iterate returns GEMPE_ERR_CONFIG, as the reference does. */
int gempe_create(gempe_ctx** out, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                 const gempe_options* opt);
void gempe_destroy(gempe_ctx* ctx);
/* Message of the last failure on this context (ctx == NULL: last failure of gempe_create on this thread). */
const char* gempe_last_error(const gempe_ctx* ctx);

int gempe_is_degenerate(const gempe_ctx* ctx);              /* EmbeddingEngine::degenerate() */
int gempe_hash_bits(const gempe_ctx* ctx);                  /* EdgeHashSet::bits() */
uint64_t gempe_sample_slots(const gempe_ctx* ctx);          /* S: 2m (PER_EDGE_2) or n*k */
uint64_t gempe_pair_terms(const gempe_ctx* ctx);            /* m + S: pair-terms per iteration */
uint64_t gempe_algorithmic_bytes(const gempe_ctx* ctx);     /* B_alg of SURVEY.md 8(d) with p = 1 */

/* EmbeddingEngine::work_graph() and the original->work permutation (src/engine.cpp:182-194).
 * Any pointer may be NULL. */
int gempe_get_work_graph(const gempe_ctx* ctx, uint32_t* src, uint32_t* dst, uint32_t* to_work);

/* Coordinates in WORK indexing, n*dim row-major fp32 (EmbeddingEngine::work_coords()).  The reference has
 * no setter; set_coords exists for teacher-forced parity runs and custom initial layouts. */
int gempe_set_coords(gempe_ctx* ctx, const float* x_work);
int gempe_get_coords(gempe_ctx* ctx, float* x_work);
int gempe_init_coords(gempe_ctx* ctx, int rule, uint64_t seed, double std);

/* Re-relabel (EmbeddingEngine::apply_relabel, src/engine.cpp:182-194): permutes the work graph and the
 * coordinates with random_relabel(relabel_seed) and rebuilds hash set, CSR and work items. */
int gempe_relabel(gempe_ctx* ctx, uint64_t relabel_seed);

/* One Jacobi round = accumulate_worker + reduce_and_update (src/engine.cpp:196-276) for the stream index
 * `iter_index` (the reference's iter_), with the (mu, sigma) of SigmoidParams.  Blocks until the round is
 * complete; fills the 2 x 512 distance tallies (DistanceHistogram::record, histogram.hpp:24-29; either may
 * be NULL).  Returns GEMPE_ERR_DIVERGENCE on a non-finite coordinate (src/engine.cpp:273-275, the state is
 * then undefined) and GEMPE_ERR_DATA when a sample stream hit the 10^4 retry cap (src/sampler.cpp:18-21). */
int gempe_iterate(gempe_ctx* ctx, double mu, double sigma, uint64_t iter_index,
                  uint64_t* hist_edge, uint64_t* hist_nonedge);

/* The round as a pure function on HOST buffers (what a caller that keeps the coordinates on the host pays):
 * x_in (X_t, n*dim, WORK indexing; page-locked memory is fastest, pageable memory takes the library's staged path) is
 * copied in while the sampling passes run, the gradient/update
 * kernel runs in slices, and each finished slice of X_{t+1} is copied to x_out while the next slice is computed.
 * Equivalent to gempe_set_coords + gempe_iterate + gempe_get_coords.  Unsharded contexts only. */
int gempe_step_host(gempe_ctx* ctx, const float* x_in, float* x_out, double mu, double sigma, uint64_t iter_index,
                    uint64_t* hist_edge, uint64_t* hist_nonedge);

/* Same round, enqueue-only: no host synchronisation.  gempe_sync waits, checks the status word and
 * returns the tallies of the LAST round. */
int gempe_iterate_async(gempe_ctx* ctx, double mu, double sigma, uint64_t iter_index);
/* Quality scoring on the device: pe_sampled (src/metrics.cpp:166-213) of the context's CURRENT coordinates.  Edge sum
 * exact; non-edge sum from samples_per_edge sampled partners per edge, reweighted by (N - m) / #samples; the
 * predictive entropy is minimised over (mu, sigma) exactly as minimize_pe does (21-point mu grid, sigma by bisection
 * on d/dsigma, golden-section refinement; src/metrics.cpp:73-127) with the exact-erf description length.  The sample
 * stream is counter-based and the edge test is the run's hash set, so the result agrees with the reference's
 * pe_sampled / pe_exact statistically (sampling noise), not draw for draw. */
typedef struct gempe_pe_report {
  double pe;                /* bits per pair */
  double mu_star, sigma_star;
  double h_basic;           /* basic_entropy of the graph (src/graph.cpp:208-217) */
  double compression_ratio; /* pe / h_basic */
  double grid_pe;           /* grid minimum before the refinement */
  uint64_t nonedge_samples; /* samples that entered the estimate */
} gempe_pe_report;
int gempe_pe_sampled(gempe_ctx* ctx, int samples_per_edge, uint64_t seed, gempe_pe_report* out);

/* `count` consecutive rounds (iteration indices first_iter .. first_iter + count - 1, fixed mu and sigma) captured
 * into one CUDA graph and replayed with one launch: small graphs (BASELINE configs 1-2) are bound by the gaps
 * between their ~5 kernels per round, not by the kernels.  gempe_graph_launch is asynchronous (gempe_sync waits and
 * returns the tallies of the LAST round); a replay repeats the same sample streams from the current coordinates.
 * Capture again after anything that swaps the coordinate buffers an odd number of times, after gempe_relabel, and
 * to change sigma.  Single-rank contexts only. */
int gempe_graph_capture(gempe_ctx* ctx, double mu, double sigma, uint64_t first_iter, int count);
int gempe_graph_launch(gempe_ctx* ctx);
int gempe_sync(gempe_ctx* ctx, uint64_t* hist_edge, uint64_t* hist_nonedge);

/* Device-resident sigma feedback: optimize_sigma_detail, the 1.5x growth cap and the PE
 * estimate of run_single_iteration (src/slope.cpp:75-125, src/engine.cpp:293-314) evaluated on the GPU from the
 * round's tallies, so that consecutive rounds need no host round trip.  gempe_set_sigma seeds the device state;
 * gempe_iterate_auto runs one round with the device's sigma, updates it, and returns the new sigma, the PE
 * estimate and the non-edge reweighting (any output pointer may be NULL).  The _async form only enqueues;
 * gempe_get_sigma_state waits and reads the state.  gempe_sigma_update_async applies the update to the current
 * device tallies (used after a cross-rank reduction of gempe_device_tallies, 1024 x u64). */
int gempe_set_sigma(gempe_ctx* ctx, double mu, double sigma);
int gempe_iterate_auto(gempe_ctx* ctx, uint64_t iter_index, double* sigma, double* pe_estimate,
                       double* nonedge_weight, uint64_t* hist_edge, uint64_t* hist_nonedge);
int gempe_iterate_auto_async(gempe_ctx* ctx, uint64_t iter_index);
int gempe_get_sigma_state(gempe_ctx* ctx, double* sigma, double* pe_estimate, double* nonedge_weight);
int gempe_sigma_update_async(gempe_ctx* ctx);
void* gempe_device_tallies(gempe_ctx* ctx);

/* ---- Runs queued without host round trips: the loop of EmbeddingEngine::run (src/engine.cpp:349-373) on the device.
 * gempe_run_begin arms the device-side bookkeeping for a run that starts at the current coordinates: sigma feedback
 * (src/engine.cpp:293-314), PE / sigma trace of up to max_rounds rounds, best-PE snapshot (:316-319) and the
 * convergence window (:353-367).  gempe_run_enqueue queues `rounds` whole iterations -- sampling, gradient + update,
 * sigma search, bookkeeping, snapshot -- that turn into no-ops once `stop_at` rounds of the run are done, the window
 * criterion holds or a round failed; with use_graph != 0 the sequence is captured once and replayed as ONE CUDA graph
 * launch (small graphs are launch-bound).  Round r of the run uses the sample streams of iteration first_iter + r.
 * gempe_run_poll waits for what was queued, moves the context to the coordinates actually reached, returns the traces
 * (first min(rounds_done, trace_cap) entries) and the last completed round's tallies, and raises the error of a failed
 * round (non-finite coordinate -> GEMPE_ERR_DIVERGENCE, ...).  Queue -> poll -> queue ...; single-rank contexts only.
 * gempe_run_best_snapshot: device pointer to the best-PE coordinates (padded rows x row stride, WORK ids of the
 * moment they were taken; valid when improved_at > 0).  gempe_run_rebase: call after gempe_relabel inside a run. */
typedef struct gempe_run_status {
  uint64_t rounds_done;      /* completed rounds of the run */
  uint64_t improved_at;      /* rounds_done value after the round that set the best PE (0: none yet) */
  uint64_t draws;            /* LCG draws of the last completed round */
  double best_pe;
  double sigma;              /* after the last completed round */
  double pe_estimate;        /* of the last completed round */
  double last_nonedge_weight;
  int32_t converged;
  int32_t failed;
} gempe_run_status;
int gempe_run_begin(gempe_ctx* ctx, double mu, double sigma, uint64_t first_iter, int32_t window, double tol,
                    uint32_t max_rounds);
int gempe_run_enqueue(gempe_ctx* ctx, uint32_t rounds, uint64_t stop_at, int32_t use_graph);
int gempe_run_poll(gempe_ctx* ctx, gempe_run_status* out, double* pe_trace, double* sigma_trace, uint32_t trace_cap,
                   uint64_t* hist_edge, uint64_t* hist_nonedge);
void* gempe_run_best_snapshot(gempe_ctx* ctx);
int gempe_run_rebase(gempe_ctx* ctx);

/* IterationCapture (include/entropy_embed/engine.hpp:92-96): consolidated y (n*dim) and z (n) of the last
 * round, in double.  Capture must be switched on before the round. */
int gempe_set_capture(gempe_ctx* ctx, int on);
int gempe_get_yz(gempe_ctx* ctx, double* y, double* z);
/* The same for `count` selected work rows (y: count*dim, z: count), and the coordinates of selected rows
 * (x: count*dim): at BASELINE config 5 the full arrays are 17 GB / 8.6 GB, a parity check needs thousands of rows. */
int gempe_get_yz_rows(gempe_ctx* ctx, const uint32_t* rows, uint64_t count, double* y, double* z);
int gempe_get_coords_rows(gempe_ctx* ctx, const uint32_t* rows, uint64_t count, float* x);

/* Bit-exact test hooks.
 * gempe_probe  == EdgeHashSet::maybe_edge (include/entropy_embed/hash_set.hpp:28-30) on WORK ids.
 * gempe_sample == the accepted partners of sample_non_edges (src/sampler.cpp:7-31) for every stream of
 *   round `iter_index`: PER_EDGE_2 slot 2*e+draw (anchor src[e] / dst[e]); PER_VERTEX_K slot v*k+draw.
 *   total_draws (may be NULL) receives the number of LCG draws, rejected ones included. */
int gempe_probe(gempe_ctx* ctx, const uint32_t* i, const uint32_t* j, uint64_t count, uint8_t* out);
int gempe_sample(gempe_ctx* ctx, uint64_t iter_index, uint32_t* partners, uint64_t* total_draws);

/* ---- plumbing for one-process-per-GPU drivers (streams, NCCL all-gather of updated shards) ---------- */
int gempe_set_stream(gempe_ctx* ctx, void* cuda_stream);           /* cudaStream_t; NULL = context's own */
void* gempe_device_coords(gempe_ctx* ctx, int which);              /* 0 = X_t (read), 1 = X_{t+1} (written) */
uint32_t gempe_row_stride(const gempe_ctx* ctx);                   /* floats per row in device layout */
uint32_t gempe_padded_rows(const gempe_ctx* ctx);                  /* world*comm_chunks*block rows */
uint32_t gempe_block_rows(const gempe_ctx* ctx);                   /* rows per (chunk, rank) ownership block */
int gempe_begin_round(gempe_ctx* ctx, double mu, double sigma, uint64_t iter_index); /* sampling passes */
int gempe_begin_round_auto(gempe_ctx* ctx, uint64_t iter_index); /* same, sigma taken from the device state */
/* opt.exchange = 1 only.  gempe_begin_round[_auto] then samples the rank's own streams and fills the send side:
 * `send_records` holds world regions of `capacity` records {uint32 partner, uint32 anchor}, region d destined for
 * rank d, `send_counts[d]` its fill.  The caller moves region d / count d of every rank s into region s / count s of
 * rank d's `recv_records` / `recv_counts` (an equal-split all-to-all on the context's stream), then calls
 * gempe_bucket_received before the first gempe_gather_chunk.  With world = 1 and exchange = 1 the context is its
 * own peer (recv aliases send) and bucketing happens inside gempe_begin_round / gempe_iterate*. */
int gempe_exchange_layout(gempe_ctx* ctx, void** send_records, void** recv_records, uint32_t** send_counts,
                          uint32_t** recv_counts, uint32_t* capacity);
int gempe_bucket_received(gempe_ctx* ctx);
int gempe_gather_chunk(gempe_ctx* ctx, int chunk);                 /* gradient+update for one comm chunk */

/* Fused update + broadcast (replaces the all-gather of gempe_gather_chunk's rows): once peers are registered, every
 * row this rank updates is stored by the gather kernel into the X_{t+1} buffer of each peer as well (peer device
 * memory over NVLink / NVSwitch), so after all ranks have finished round t every rank holds the full X_{t+1} without
 * a collective on the coordinates.  The ranks only need a barrier between consecutive rounds (a rank must not start
 * round t+1's gather while a peer still reads or writes round t's buffers); the tally all-reduce is one.
 *   gempe_coords_ipc_handles : this rank's two coordinate buffers as CUDA IPC handles (2 x 64 bytes, parity 0 and 1)
 *   gempe_open_peer          : registers a peer from the handles it published (another process, any GPU with P2P)
 *   gempe_add_peer_pointers  : registers a peer living in THIS process (buffers of parity 0 and 1)
 *   gempe_device_coords_parity / gempe_coords_parity : the buffer of a given parity / the parity holding X_t now
 * All ranks must run their rounds in lock step (same parity).  */
#define GEMPE_IPC_HANDLE_BYTES 64
int gempe_coords_ipc_handles(gempe_ctx* ctx, void* out_2x64_bytes);
int gempe_open_peer(gempe_ctx* ctx, const void* handles_2x64_bytes);
int gempe_add_peer_pointers(gempe_ctx* ctx, void* x_parity0, void* x_parity1);
int gempe_clear_peers(gempe_ctx* ctx);
/* Direct sample exchange (opt.exchange with world > 1; replaces the all-to-all of gempe_exchange_layout): every rank
 * publishes its receive area (one allocation: records of both round parities, then the counts) and opens those of all
 * other ranks; from then on the sampling kernel of gempe_begin_round stores each record straight into the region
 * reserved for this rank in the destination's receive area, and a one-warp kernel publishes the counts.  The caller
 * only needs ONE barrier per round, between gempe_begin_round and gempe_bucket_received: it also separates the
 * previous round's gather (peer stores into X) from this round's.
 *   gempe_exchange_ipc_handle       : the receive area as a CUDA IPC handle (64 bytes)
 *   gempe_open_peer_exchange        : registers rank `peer_rank`'s receive area from its handle (another process)
 *   gempe_add_peer_exchange_pointer : the same for a context living in this process (gempe_exchange_recv_area)
 * Active as soon as all world - 1 peers are registered; gempe_clear_peers drops them. */
int gempe_exchange_ipc_handle(gempe_ctx* ctx, void* out_64_bytes);
int gempe_open_peer_exchange(gempe_ctx* ctx, int peer_rank, const void* handle_64_bytes);
int gempe_add_peer_exchange_pointer(gempe_ctx* ctx, int peer_rank, void* recv_area);
void* gempe_exchange_recv_area(gempe_ctx* ctx);
void* gempe_device_coords_parity(gempe_ctx* ctx, int parity);
int gempe_coords_parity(const gempe_ctx* ctx);
int gempe_end_round(gempe_ctx* ctx);                               /* swaps X_t / X_{t+1} */
/* Device time in ms of the last `rounds` enqueued through gempe_iterate_async since the previous call
 * (CUDA events on the context's stream), split as {total, sampling passes, gather+update}. */
int gempe_elapsed_ms(gempe_ctx* ctx, float out3[3]);
uint64_t gempe_kernel_launches(const gempe_ctx* ctx);              /* kernels launched so far */
/* slotted buckets (bucket_mode 4): samples of the last round that did not fit their partner's slots and took the
 * indexed spill list (waits for the stream); -1 when the context does not use slotted buckets.  Diagnostics / tests. */
int64_t gempe_bucket_spills(gempe_ctx* ctx);

/* Page-locked host memory for a caller without CUDA headers (cudaHostAlloc / cudaFreeHost), e.g. the coordinate vectors
 * handed to gempe_step_host every round.  BASELINE config 4, gempe_step_host: 20 ms per step on these; 35-45 ms on ordinary
 * pageable vectors, which the library moves through its own ring of pinned chunks and host threads (89 ms with the driver's
 * staging); registering the caller's own pages with cudaHostRegister is NOT offered: on the bench host the step then takes
 * 139 ms -- DMA over scattered 4 KB pages.  gempe_alloc_host returns NULL on failure (message through
 * gempe_last_error(NULL)).  No reference analogue. */
void* gempe_alloc_host(uint64_t bytes);
void gempe_free_host(void* ptr);

/* Device memory of destroyed contexts / engines is kept in a per-device cache and reused by the
 * next ones: a process that calls embed() repeatedly does not pay cudaMalloc / cudaFree for gigabytes per call.  The cache
 * holds at most GEMPE_DEVICE_CACHE_MB megabytes (environment, default 16384; 0 disables it); this call returns all of it
 * to the driver.  No reference analogue (the reference allocates host vectors). */
void gempe_trim_device_cache(void);

/* ---- Several GPUs in ONE process: the C++ multi-GPU host (`devices[], n_devices` of the proposed
 * constructor).  A group is one context per listed device (a device may be listed more than once: several ranks on one
 * GPU, used by the tests), vertices sharded contiguously over the ranks, every rank holding the full X_t, CSR and edge
 * filter.  A round is driven from the calling thread through the ranks' streams and ordered by CUDA events only.  With
 * peer access between all listed devices the sample records and the updated rows travel as stores of the pack / gather
 * kernels into the other ranks' memory (NVLink / NVSwitch); otherwise, or with GEMPE_GROUP_COPY_ENGINES, as
 * cudaMemcpyPeerAsync copies (all-to-all of the packed regions, all-gather of the owned row blocks).  Results are
 * bit-identical to a single context in deterministic mode.  gempe_options.device / rank / world / comm_chunks / exchange
 * of `opt` are set per rank by the group.
 *   gempe_group_iterate       one sharded round, job-wide tallies           (gempe_iterate)
 *   gempe_group_iterate_auto  round + sigma search on every rank's device from the summed tallies (gempe_iterate_auto)
 *   gempe_group_relabel       re-relabel on every rank                        (gempe_relabel)
 *   gempe_group_replicas_agree  1 when all ranks hold bit-identical coordinates (start-up / test check) */
typedef struct gempe_group gempe_group;
#define GEMPE_GROUP_COPY_ENGINES 1 /* flags: move records and rows with copy engines even where peer stores would work */
int gempe_group_create(gempe_group** out, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                       const gempe_options* opt, const int* devices, int n_devices, int flags);
void gempe_group_destroy(gempe_group* group);
const char* gempe_group_last_error(const gempe_group* group);   /* NULL: error of a failed gempe_group_create */
int gempe_group_world(const gempe_group* group);
gempe_ctx* gempe_group_context(gempe_group* group, int rank);   /* owned by the group */
const char* gempe_group_exchange_path(const gempe_group* group);
int gempe_group_set_coords(gempe_group* group, const float* x_work);
int gempe_group_init_coords(gempe_group* group, int rule, uint64_t seed, double std);
int gempe_group_get_coords(gempe_group* group, float* x_work);
int gempe_group_iterate(gempe_group* group, double mu, double sigma, uint64_t iter_index, uint64_t* hist_edge,
                        uint64_t* hist_nonedge);
int gempe_group_set_sigma(gempe_group* group, double mu, double sigma);
int gempe_group_iterate_auto(gempe_group* group, uint64_t iter_index, double* sigma, double* pe_estimate,
                             double* nonedge_weight, uint64_t* hist_edge, uint64_t* hist_nonedge);
int gempe_group_relabel(gempe_group* group, uint64_t relabel_seed);
int gempe_group_replicas_agree(gempe_group* group);

/* ---- host-side numerics of the path (no GPU needed) ------------------------------------------------ */
/* FastMath::build tables (src/piecewise.cpp:182-195). which: 0 erf, 1 exp_neg, 2 ratio.
 * out67 = knots[17] a[16] b[16] c[16] lo hi.  Returns odd_mirror (0/1) or a negative error. */
int gempe_host_fastmath_table(int which, double* out67);
/* optimize_sigma_detail / histogram_objective(_dsigma) (src/slope.cpp:27-51, 75-125). */
double gempe_host_optimize_sigma(const uint64_t* hist_edge, const uint64_t* hist_nonedge,
                                 double nonedge_weight, double mu, int* bisection_steps);
double gempe_host_histogram_objective(const uint64_t* hist_edge, const uint64_t* hist_nonedge,
                                      double nonedge_weight, double mu, double sigma);
double gempe_host_histogram_objective_dsigma(const uint64_t* hist_edge, const uint64_t* hist_nonedge,
                                             double nonedge_weight, double mu, double sigma);
/* random_relabel (src/graph.cpp:182-194): forward[original] = relabeled. */
int gempe_host_random_relabel(uint32_t n, uint64_t seed, uint32_t* forward);
uint64_t gempe_host_mix_seed(uint64_t seed, uint64_t component);   /* include/entropy_embed/rng.hpp:26-28 */

/* ---- graph ingest and embedding export (host side) ------------------------------ */
typedef struct gempe_graph {   /* Graph, include/entropy_embed/graph.hpp:12-23; arrays owned by the library */
  uint32_t n;
  uint64_t m;
  uint32_t* src;
  uint32_t* dst;
  uint64_t* raw_labels;        /* original input id of every compact vertex (edge lists only, else NULL) */
} gempe_graph;

/* load_edge_list (src/graph.cpp:75-133): "i<ws>j" lines; '#'/'%' comments and blank lines skipped; self-loops
 * dropped; duplicate undirected edges merged; ids compacted in first-appearance order.  A malformed line returns
 * GEMPE_ERR_DATA with *error_line set (parse_error::line()); no surviving edge returns GEMPE_ERR_DATA with
 * *error_line = 0 (data_error).  Messages through gempe_last_error(NULL). */
int gempe_parse_edge_list(const char* text, uint64_t len, gempe_graph* out, uint64_t* error_line);
/* load_graph_snapshot (src/graph.cpp:149-170): "GEMP", u32 n, u64 m, src[m], dst[m], little-endian. */
int gempe_parse_graph_snapshot(const void* bytes, uint64_t len, gempe_graph* out);
/* looks_like_snapshot ? load_graph_snapshot : load_edge_list (tools/embed_main.cpp:150-153). */
int gempe_load_graph_file(const char* path, gempe_graph* out, uint64_t* error_line);
int gempe_write_graph_snapshot(const char* path, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst);
void gempe_graph_free(gempe_graph* g);
/* write_embedding_tsv (src/io.cpp:17-46): rows in ascending label order, "%.6g" coordinates; labels NULL =
 * identity; perm_forward non-NULL reads row perm_forward[v] for vertex v. */
int gempe_write_embedding_tsv(const char* path, uint32_t n, uint32_t dim, const float* coords, const uint64_t* labels,
                              const uint32_t* perm_forward);

/* ---- run-level facade: EmbeddingEngine / embed() (include/entropy_embed/engine.hpp:112-171) ------- */
typedef struct gempe_engine gempe_engine;

typedef struct gempe_iteration_config { /* IterationConfig, engine.hpp:29-38 */
  int32_t max_iters;          /* 100 */
  uint32_t lane_width;        /* accepted for source compatibility; sample streams do not depend on it */
  uint32_t workers;           /* accepted for source compatibility; unused on the GPU */
  double convergence_tol;     /* 1e-4 */
  int32_t convergence_window; /* 5 */
  int32_t relabel_period;     /* 0 */
  int32_t fast_math;          /* 1 = tables */
  int32_t hash_bits;          /* 0 = auto */
  /* extensions (zero = reference behaviour) */
  int32_t neg_mode;
  uint32_t negatives;
  int32_t device;
  int32_t host_sigma;         /* 1 = run the sigma search on the host (hostmath.cpp) instead of the device kernel */
  int32_t deterministic;      /* 1 = sorted sample buckets: byte-identical results run to run (README.md:41-44 of the
                                 reference promises this for fixed input, seed, workers and lanes) */
  int32_t batch_rounds;       /* gempe_engine_run with the device sigma search queues this many whole iterations per host
                                 round trip (gempe_run_enqueue / gempe_run_poll; convergence, best-PE snapshot and PE
                                 trace are kept on the device): 0 = auto (16, replayed as one CUDA graph, for graphs
                                 below ~4 M pair-terms per round; 4 plain launches above), 1 = poll after every round,
                                 < 0 = the host loop of round 1 (one gempe_iterate_auto per round) */
} gempe_iteration_config;

typedef struct gempe_embed_result { /* EmbedResult, engine.hpp:98-107 */
  float* embedding;           /* n*dim, ORIGINAL indexing; caller-provided */
  double* pe_trace;           /* caller-provided, capacity pe_trace_cap */
  int32_t pe_trace_cap;
  int32_t pe_trace_len;
  double final_sigma;
  int32_t converged;
  int32_t degenerate;
  int32_t iterations;
  uint32_t* relabel_forward;  /* n, may be NULL */
  uint64_t* last_hist_edge;   /* 512, may be NULL */
  uint64_t* last_hist_nonedge;
  double last_nonedge_weight;
} gempe_embed_result;

void gempe_default_iteration_config(gempe_iteration_config* cfg);
int gempe_engine_create(gempe_engine** out, uint32_t n, uint64_t m, const uint32_t* src,
                        const uint32_t* dst, uint32_t dim, const gempe_iteration_config* cfg,
                        uint64_t seed);
/* The same engine sharded over several GPUs of this process (`devices[], n_devices` of SURVEY.md 8b; a gempe_group
 * inside): n_devices <= 1 is gempe_engine_create on devices[0] / cfg->device.  gempe_engine_context returns rank 0. */
int gempe_engine_create_multi(gempe_engine** out, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                              uint32_t dim, const gempe_iteration_config* cfg, uint64_t seed, const int* devices,
                              int n_devices);
void gempe_engine_destroy(gempe_engine* e);
const char* gempe_engine_last_error(const gempe_engine* e);
gempe_ctx* gempe_engine_context(gempe_engine* e);                   /* borrowed */
int gempe_engine_degenerate(const gempe_engine* e);
int gempe_engine_iteration(const gempe_engine* e);                  /* EmbeddingEngine::iteration() */
double gempe_engine_sigma(const gempe_engine* e);                   /* params().sigma */
/* EmbeddingEngine::run_single_iteration (src/engine.cpp:278-325). */
int gempe_engine_run_single_iteration(gempe_engine* e, double* pe_estimate, double* sigma);
/* EmbeddingEngine::run (src/engine.cpp:339-382). */
int gempe_engine_run(gempe_engine* e, gempe_embed_result* result);

#ifdef __cplusplus
}
#endif
#endif /* GEMPE_H_ */
