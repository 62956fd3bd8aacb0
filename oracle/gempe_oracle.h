/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the GEMPE hot path.
 *
 * Plain-C restatement of one iteration of the reference "entropy-embed" engine
 * (/root/reference/proj, citations are relative to that directory).  It exists so that
 * tests/ can check the CUDA path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product (paper_2011_03479_b200/) never does.
 *
 * Parity of THIS file is pinned (tests/test_oracle_pins.py) against
 *   - the reference's own frozen vectors (tests/test_graph.cpp:161-178,
 *     tests/test_rng_sampler.cpp:17-54, tests/test_sigmoid.cpp:73-87), and
 *   - outputs of the unmodified reference compiled here (oracle/_ref), committed as
 *     tests/golden/ *.json by tools/make_golden.py.
 */
#ifndef GEMPE_ORACLE_H_
#define GEMPE_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GO_BINS 512
#define GO_SEGMENTS 16

/* 16-segment continuous piecewise quadratic (include/entropy_embed/piecewise.hpp:17-47). */
typedef struct {
  double knots[GO_SEGMENTS + 1];
  double a[GO_SEGMENTS], b[GO_SEGMENTS], c[GO_SEGMENTS];
  double lo, hi;
  int odd_mirror;
} go_table;

/* The two tables the hot loop reads (piecewise.hpp:72-79). */
typedef struct {
  go_table erf;
  go_table ratio;
} go_fastmath;

/* negative-sampling schemes */
enum { GO_PER_EDGE_2 = 0, GO_PER_VERTEX_K = 1 };

/* ---- integer layer -------------------------------------------------------------------- */
uint64_t go_splitmix64(uint64_t z);                               /* rng.hpp:17-22 */
uint64_t go_mix_seed(uint64_t seed, uint64_t component);          /* rng.hpp:26-28 */
uint32_t go_expand_seed32(uint64_t seed, uint64_t a, uint64_t b, uint64_t c); /* rng.hpp:31-34 */
uint32_t go_lcg_next(uint32_t s);                                 /* rng.hpp:82-86 */
uint32_t go_lane_uniform_index(uint32_t state_word, uint32_t n);  /* rng.hpp:99-108 */
uint32_t go_pair_hash(uint32_t i, uint32_t j, uint32_t n, uint32_t table_size); /* hash_set.hpp:14-17 */
int go_hash_bits(uint64_t m, int bits_override);                  /* hash_set.cpp:13-24 */
/* table must hold 1<<bits zeroed bytes; hash_set.cpp:27-32 */
void go_hash_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst, int bits,
                   uint8_t* table);
/* sampler.cpp:15-29 for one lane.  Returns 0 and the partner, or 2 after 10^4 rejected draws. */
int go_sample_one(const uint8_t* table, uint32_t table_size, uint32_t n, uint32_t anchor,
                  uint32_t state, uint32_t* partner, uint32_t* draws);
void go_random_relabel(uint32_t n, uint64_t seed, uint32_t* forward);   /* graph.cpp:182-206 */
void go_init_embedding(uint32_t n, uint32_t dim, uint64_t seed, float* out); /* engine.cpp:116-124 */

/* ---- numerics ---------------------------------------------------------------------------- */
double go_table_eval(const go_table* t, double x);                /* piecewise.hpp:25-47 */
double go_gauss_over_erfc(double x);                              /* sigmoid.hpp:39-45 */
double go_ratio_fast(const go_fastmath* fm, double x);            /* piecewise.hpp:72-79 */
/* sigmoid.hpp:88-101; fm == NULL selects ExactMath (sigmoid.hpp:61-65). */
void go_parabola(double delta, double mu, double sigma, int is_edge, const go_fastmath* fm,
                 double* d_target, double* w);
int go_hist_bin(double delta);                                    /* histogram.hpp:24-29 */

/* ---- sigma optimiser (slope.cpp) -- exact math throughout ------------------------------ */
double go_histogram_objective(const uint64_t* edge, const uint64_t* nonedge, double nonedge_weight,
                              double mu, double sigma);           /* slope.cpp:27-38 */
double go_histogram_objective_dsigma(const uint64_t* edge, const uint64_t* nonedge,
                                     double nonedge_weight, double mu, double sigma); /* :40-51 */
double go_optimize_sigma(const uint64_t* edge, const uint64_t* nonedge, double nonedge_weight,
                         double mu, int* bisection_steps);        /* slope.cpp:75-125 */

/* ---- one Jacobi round (engine.cpp:196-276) ------------------------------------------------
 * Work-graph ids.  x is n*dim row-major fp32.  y (n*dim) and z (n) receive the consolidated sums in
 * double (the "independent double-precision replay" of tests/test_engine.cpp:209-266); x_next
 * (n*dim, may alias nothing) receives the updated coordinates (hold on z<=0).  partners (S slots)
 * receives the accepted samples: PER_EDGE_2 slot = 2*e+draw (anchor src[e] / dst[e], stream key
 * (seed, iter, e, draw)); PER_VERTEX_K slot = v*k+draw (anchor v, key (seed, iter, v, draw)).
 * If forced_partners != NULL the sampler is skipped and those indices are used (teacher forcing).
 * Returns 0, 2 (retry cap) or 3 (non-finite coordinate). */
int go_iterate(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst, uint32_t dim,
               const float* x, int neg_mode, uint32_t k, uint64_t seed, uint64_t iter, double mu,
               double sigma, const go_fastmath* fm, const uint8_t* table, uint32_t table_size,
               const uint32_t* forced_partners, double* y, double* z, uint64_t* hist_edge,
               uint64_t* hist_nonedge, float* x_next, uint32_t* partners, uint64_t* total_draws);

/* ---- the same pair arithmetic on an explicit pair list, accumulated for a vertex SUBSET -----
 * For sizes where a whole round is minutes of CPU work (BASELINE config 5): every pair (a[i], b[i])
 * goes through pair_distance + parabola + add_pair exactly as in go_iterate, but only endpoints with
 * sub_index[v] >= 0 receive their sums, in row sub_index[v] of y_sub (rows x dim) / z_sub.  The caller
 * lists every pair that touches a subset vertex once (edges incident to it; samples it anchors or
 * receives).  hist (GO_BINS, may be NULL) tallies the listed pairs. */
void go_pairs_accumulate(uint32_t dim, const float* x, const int32_t* sub_index, uint64_t count,
                         const uint32_t* a, const uint32_t* b, int is_edge, double mu, double sigma,
                         const go_fastmath* fm, double* y_sub, double* z_sub, uint64_t* hist);

#ifdef __cplusplus
}
#endif
#endif
