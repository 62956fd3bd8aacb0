/* TEST INFRASTRUCTURE ONLY -- see gempe_oracle.h.  Plain C11, libm only.
 * Compiled with -ffp-contract=off so that no FMA contraction changes the double results relative
 * to the reference's g++ build (x86-64 baseline, no -march: no FMA there either). */
#include "gempe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GO_GOLDEN 0x9E3779B97F4A7C15ull
#define GO_LCG_MUL 1103515245u
#define GO_PI 3.14159265358979323846264338327950288
#define GO_LN2 0.693147180559945309417232121458176568
#define GO_SQRT2 1.41421356237309504880168872420969808
#define GO_SQRT_PI 1.77245385090551602729816748334
#define GO_SQRT_2PI 2.50662827463100050241576528481

/* ------------------------------------------------------------------ integer layer */

uint64_t go_splitmix64(uint64_t z) { /* rng.hpp:17-22 */
  z += GO_GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t go_mix_seed(uint64_t seed, uint64_t component) { /* rng.hpp:26-28 */
  return go_splitmix64(seed ^ (GO_GOLDEN * (component + 1)));
}

uint32_t go_expand_seed32(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:31-34 */
  return (uint32_t)(go_mix_seed(go_mix_seed(go_mix_seed(seed, a), b), c) >> 16);
}

uint32_t go_lcg_next(uint32_t s) { return s * GO_LCG_MUL + 1u; } /* rng.hpp:82-86 */

uint32_t go_lane_uniform_index(uint32_t w, uint32_t n) { /* rng.hpp:99-108 */
  if (n <= (1u << 23)) {
    const uint32_t bits = 0x3f800000u | (w & 0x7fffffu);
    float f;
    memcpy(&f, &bits, sizeof f);
    const double v = (double)f * n - n;
    return (uint32_t)v;
  }
  return (uint32_t)((uint64_t)w % n);
}

uint32_t go_pair_hash(uint32_t i, uint32_t j, uint32_t n, uint32_t size) { /* hash_set.hpp:14-17 */
  return ((i * n + j) * GO_LCG_MUL) & (size - 1);
}

int go_hash_bits(uint64_t m, int bits_override) { /* hash_set.cpp:13-24 */
  int bits = 6;
  if (bits_override > 0) return bits_override;
  const uint64_t target = 64ull * (m > 1 ? m : 1);
  while ((1ull << bits) < target) ++bits;
  if (bits > 31) bits = 31;
  return bits;
}

void go_hash_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst, int bits,
                   uint8_t* table) { /* hash_set.cpp:27-32 */
  const uint32_t size = 1u << bits;
  for (uint64_t e = 0; e < m; ++e) {
    table[go_pair_hash(src[e], dst[e], n, size)] = 1;
    table[go_pair_hash(dst[e], src[e], n, size)] = 1;
  }
}

int go_sample_one(const uint8_t* table, uint32_t size, uint32_t n, uint32_t anchor,
                  uint32_t state, uint32_t* partner, uint32_t* draws) { /* sampler.cpp:15-29 */
  for (int tries = 0;; ++tries) {
    if (tries >= 10000) {
      if (draws) *draws = (uint32_t)tries;
      return 2;
    }
    state = go_lcg_next(state); /* advance first, then use */
    const uint32_t g = go_lane_uniform_index(state, n);
    if (g == anchor) continue;
    if (table[go_pair_hash(anchor, g, n, size)]) continue;
    *partner = g;
    if (draws) *draws = (uint32_t)tries + 1;
    return 0;
  }
}

static uint64_t bounded_u64(uint64_t r, uint64_t range) { /* rng.hpp:37-39 */
  return (uint64_t)(((unsigned __int128)r * range) >> 64);
}

void go_random_relabel(uint32_t n, uint64_t seed, uint32_t* forward) { /* graph.cpp:182-194 */
  for (uint32_t i = 0; i < n; ++i) forward[i] = i;
  uint64_t state = go_mix_seed(seed, 0x5eedu);
  for (uint32_t i = 0; i + 1 < n; ++i) {
    state = go_splitmix64(state);
    const uint32_t j = i + (uint32_t)bounded_u64(state, n - i);
    const uint32_t t = forward[i];
    forward[i] = forward[j];
    forward[j] = t;
  }
}

void go_init_embedding(uint32_t n, uint32_t dim, uint64_t seed, float* out) { /* engine.cpp:116-124 */
  uint64_t state = go_mix_seed(seed, 0x1217);
  const size_t total = (size_t)n * dim;
  for (size_t i = 0; i < total; ++i) {
    state += GO_GOLDEN; /* SplitMix::next, rng.hpp:48-54 */
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    out[i] = (float)((double)(z >> 11) * 0x1.0p-53);
  }
}

/* ------------------------------------------------------------------ numerics */

static int segment_of(const go_table* t, double x) { /* piecewise.hpp:36-47 */
  int lo = 0, hi = GO_SEGMENTS;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (x < t->knots[mid]) hi = mid; else lo = mid;
  }
  return lo;
}

double go_table_eval(const go_table* t, double x) { /* piecewise.hpp:25-34 */
  double xa = x < t->lo ? t->lo : (x > t->hi ? t->hi : x);
  double flip = 1.0;
  if (t->odd_mirror && xa < 0.0) {
    xa = -xa;
    flip = -1.0;
  }
  const int s = segment_of(t, xa);
  return flip * ((t->a[s] * xa + t->b[s]) * xa + t->c[s]);
}

double go_gauss_over_erfc(double x) { /* sigmoid.hpp:39-45 */
  if (x <= 6.0) return exp(-x * x) / erfc(x);
  const double ix2 = 1.0 / (x * x);
  const double series = 1.0 + ix2 * (-0.5 + ix2 * (0.75 + ix2 * (-1.875 + 6.5625 * ix2)));
  return x * GO_SQRT_PI / series;
}

double go_ratio_fast(const go_fastmath* fm, double x) { /* piecewise.hpp:72-79 */
  if (x >= fm->ratio.lo) {
    if (x > fm->ratio.hi) return go_gauss_over_erfc(x);
    return go_table_eval(&fm->ratio, x);
  }
  if (x < -6.0) return 0.0;
  return exp(-x * x) / (1.0 - go_table_eval(&fm->erf, x));
}

void go_parabola(double delta, double mu, double sigma, int is_edge, const go_fastmath* fm,
                 double* d_target, double* w_out) { /* sigmoid.hpp:88-101 */
  const double k_two_over_pi_ln2 = 2.0 / (GO_PI * GO_LN2);
  const double k_inv_sqrt2pi_ln2 = 1.0 / (GO_SQRT_2PI * GO_LN2);
  const double u = (delta - mu) / (GO_SQRT2 * sigma);
  const double sign = is_edge ? -1.0 : 1.0;
  const double xarg = is_edge ? u : -u;
  const double ratio = fm ? go_ratio_fast(fm, xarg) : go_gauss_over_erfc(xarg);
  const double s2 = sigma * sigma;
  const double w = k_two_over_pi_ln2 * ratio * ratio / s2 +
                   sign * k_inv_sqrt2pi_ln2 * (delta - mu) * ratio / (s2 * sigma);
  if (!(w > 0.0)) {
    *d_target = delta;
    *w_out = 0.0;
    return;
  }
  *d_target = delta + sign * k_inv_sqrt2pi_ln2 * ratio / (w * sigma);
  *w_out = w;
}

int go_hist_bin(double delta) { /* histogram.hpp:24-29 */
  int b = (int)(delta / 12.0 * GO_BINS);
  if (b >= GO_BINS) b = GO_BINS - 1;
  if (b < 0) b = 0;
  return b;
}

/* ------------------------------------------------------------------ sigma optimiser */

static double bin_mid(int b) { return (b + 0.5) * 12.0 / GO_BINS; } /* histogram.hpp:52 */

static double description_length(double delta, double mu, double sigma, int is_edge) {
  /* sigmoid.hpp:69-81 with ExactMath */
  const double u = (delta - mu) / (GO_SQRT2 * sigma);
  const double e = erf(u);
  double s = is_edge ? 0.5 - 0.5 * e : 0.5 + 0.5 * e;
  if (s < 1e-12) s = 1e-12;
  if (s > 1.0 - 1e-12) s = 1.0 - 1e-12;
  return -log2(s);
}

static double dl_tail_exact(double delta, double mu, double sigma, int is_edge) { /* sigmoid.hpp:50-59 */
  const double u = (delta - mu) / (GO_SQRT2 * sigma);
  const double x = is_edge ? u : -u;
  if (x <= 6.0) return 1.0 - log2(erfc(x));
  const double ix2 = 1.0 / (x * x);
  const double series = 1.0 + ix2 * (-0.5 + ix2 * (0.75 + ix2 * (-1.875 + 6.5625 * ix2)));
  const double log_erfc = -x * x - log(x * GO_SQRT_PI) + log(series);
  return 1.0 - log_erfc / GO_LN2;
}

static double dl_sigma_derivative(double delta, double mu, double sigma, int is_edge) {
  /* sigmoid.hpp:108-113 with ExactMath */
  const double k = 2.0 / (GO_SQRT_PI * GO_LN2);
  const double u = (delta - mu) / (GO_SQRT2 * sigma);
  const double v = k * u * go_gauss_over_erfc(is_edge ? u : -u) / sigma;
  return is_edge ? -v : v;
}

typedef double (*go_dl_fn)(double, double, double, int);

static double hist_sum(const uint64_t* edge, const uint64_t* nonedge, double nw, double mu,
                       double sigma, go_dl_fn f) { /* slope.cpp:27-38, 40-51, 58-71 */
  double total = 0.0;
  for (int b = 0; b < GO_BINS; ++b) {
    const uint64_t ec = edge[b], nc = nonedge[b];
    if (ec == 0 && nc == 0) continue;
    const double mid = bin_mid(b);
    if (ec) total += (double)ec * f(mid, mu, sigma, 1);
    if (nc) total += nw * (double)nc * f(mid, mu, sigma, 0);
  }
  return total;
}

double go_histogram_objective(const uint64_t* e, const uint64_t* ne, double nw, double mu, double s) {
  return hist_sum(e, ne, nw, mu, s, description_length);
}

double go_histogram_objective_dsigma(const uint64_t* e, const uint64_t* ne, double nw, double mu,
                                     double s) {
  return hist_sum(e, ne, nw, mu, s, dl_sigma_derivative);
}

double go_optimize_sigma(const uint64_t* edge, const uint64_t* nonedge, double nw, double mu,
                         int* steps_out) { /* slope.cpp:75-125 */
  const double smin = 1e-3, smax = 16.0, tol = 1e-4;
  enum { kGrid = 17, kMaxSteps = 60 };
  double grid[kGrid];
  int best = 0;
  double best_cost = 0.0;
  for (int i = 0; i < kGrid; ++i) {
    grid[i] = smin * pow(smax / smin, (double)i / (kGrid - 1));
    const double cost = hist_sum(edge, nonedge, nw, mu, grid[i], dl_tail_exact);
    if (i == 0 || cost < best_cost) {
      best_cost = cost;
      best = i;
    }
  }
  double sigma = grid[best];
  int steps = 0;
  double lo = grid[best > 0 ? best - 1 : 0];
  double hi = grid[best < kGrid - 1 ? best + 1 : kGrid - 1];
  double f_lo = hist_sum(edge, nonedge, nw, mu, lo, dl_sigma_derivative);
  const double f_hi = hist_sum(edge, nonedge, nw, mu, hi, dl_sigma_derivative);
  if (!(f_lo < 0.0) || !(f_hi > 0.0)) {
    if (steps_out) *steps_out = 0;
    return sigma;
  }
  while (hi - lo > tol && steps < kMaxSteps) {
    ++steps;
    const double mid = 0.5 * (lo + hi);
    const double f_mid = hist_sum(edge, nonedge, nw, mu, mid, dl_sigma_derivative);
    if (f_mid == 0.0) {
      lo = hi = mid;
      break;
    }
    if ((f_mid > 0.0) == (f_lo > 0.0)) {
      lo = mid;
      f_lo = f_mid;
    } else {
      hi = mid;
    }
  }
  const double refined = 0.5 * (lo + hi);
  if (hist_sum(edge, nonedge, nw, mu, refined, dl_tail_exact) <= best_cost) sigma = refined;
  if (steps_out) *steps_out = steps;
  return sigma;
}

/* ------------------------------------------------------------------ one Jacobi round */

static double pair_distance(const float* xa, const float* xb, uint32_t dim) { /* engine.cpp:45-52 */
  double acc = 0.0;
  for (uint32_t k = 0; k < dim; ++k) {
    const double diff = (double)xa[k] - (double)xb[k];
    acc += diff * diff;
  }
  return sqrt(acc);
}

/* add_pair (engine.cpp:54-73) carried in double, as the reference's own replay test does
 * (tests/test_engine.cpp:228-240). */
static void add_pair_f64(const float* x, uint32_t dim, uint32_t u, uint32_t v, double delta,
                         double d_target, double w, double* y, double* z) {
  if (!(w > 0.0)) return;
  const double target = d_target > 0.0 ? d_target : 0.0;
  const double s = delta > 0.0 ? target / delta : 0.0;
  const float* xu = x + (size_t)u * dim;
  const float* xv = x + (size_t)v * dim;
  double* yu = y + (size_t)u * dim;
  double* yv = y + (size_t)v * dim;
  for (uint32_t k = 0; k < dim; ++k) {
    const double a = xu[k], b = xv[k];
    const double diff = a - b;
    yu[k] += w * (b + s * diff);
    yv[k] += w * (a - s * diff);
  }
  z[u] += w;
  z[v] += w;
}

static void process_pair(const float* x, uint32_t dim, uint32_t u, uint32_t v, int is_edge,
                         double mu, double sigma, const go_fastmath* fm, double* y, double* z,
                         uint64_t* hist) {
  const double delta = pair_distance(x + (size_t)u * dim, x + (size_t)v * dim, dim);
  hist[go_hist_bin(delta)]++; /* tallied before the w>0 test, engine.cpp:221-222,244-245 */
  double d_target, w;
  go_parabola(delta, mu, sigma, is_edge, fm, &d_target, &w);
  add_pair_f64(x, dim, u, v, delta, d_target, w, y, z);
}

int go_iterate(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst, uint32_t dim,
               const float* x, int neg_mode, uint32_t k, uint64_t seed, uint64_t iter, double mu,
               double sigma, const go_fastmath* fm, const uint8_t* table, uint32_t table_size,
               const uint32_t* forced, double* y, double* z, uint64_t* hist_edge,
               uint64_t* hist_nonedge, float* x_next, uint32_t* partners, uint64_t* total_draws) {
  memset(y, 0, sizeof(double) * (size_t)n * dim);
  memset(z, 0, sizeof(double) * n);
  memset(hist_edge, 0, sizeof(uint64_t) * GO_BINS);
  memset(hist_nonedge, 0, sizeof(uint64_t) * GO_BINS);
  uint64_t draws_total = 0;

  for (uint64_t e = 0; e < m; ++e) { /* engine.cpp:215-225 */
    process_pair(x, dim, src[e], dst[e], 1, mu, sigma, fm, y, z, hist_edge);
  }

  const uint64_t slots = neg_mode == GO_PER_EDGE_2 ? 2 * m : (uint64_t)n * k;
  for (uint64_t t = 0; t < slots; ++t) { /* engine.cpp:230-248 */
    uint32_t anchor;
    uint64_t unit, draw;
    if (neg_mode == GO_PER_EDGE_2) {
      unit = t >> 1;
      draw = t & 1;
      anchor = draw == 0 ? src[unit] : dst[unit];
    } else {
      unit = t / k;
      draw = t % k;
      anchor = (uint32_t)unit;
    }
    uint32_t partner;
    if (forced) {
      partner = forced[t];
    } else {
      uint32_t draws = 0;
      const uint32_t s0 = go_expand_seed32(seed, iter, unit, draw);
      const int rc = go_sample_one(table, table_size, n, anchor, s0, &partner, &draws);
      draws_total += draws;
      if (rc) return rc;
    }
    if (partners) partners[t] = partner;
    process_pair(x, dim, anchor, partner, 0, mu, sigma, fm, y, z, hist_nonedge);
  }
  if (total_draws) *total_draws = draws_total;

  int bad = 0;
  if (x_next) { /* engine.cpp:261-272 */
    for (uint32_t v = 0; v < n; ++v) {
      const double zz = z[v];
      float* row = x_next + (size_t)v * dim;
      const float* old = x + (size_t)v * dim;
      if (zz <= 0.0) {
        for (uint32_t c = 0; c < dim; ++c) row[c] = old[c];
        continue;
      }
      for (uint32_t c = 0; c < dim; ++c) {
        const float value = (float)(y[(size_t)v * dim + c] / zz);
        if (!isfinite(value)) bad = 1;
        row[c] = value;
      }
    }
  }
  return bad ? 3 : 0;
}

/* add_pair for a vertex subset: same terms as add_pair_f64, rows of the subset only. */
void go_pairs_accumulate(uint32_t dim, const float* x, const int32_t* sub_index, uint64_t count,
                         const uint32_t* a, const uint32_t* b, int is_edge, double mu, double sigma,
                         const go_fastmath* fm, double* y_sub, double* z_sub, uint64_t* hist) {
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t u = a[i], v = b[i];
    const float* xu = x + (size_t)u * dim;
    const float* xv = x + (size_t)v * dim;
    const double delta = pair_distance(xu, xv, dim);
    if (hist) hist[go_hist_bin(delta)]++;
    double d_target, w;
    go_parabola(delta, mu, sigma, is_edge, fm, &d_target, &w);
    if (!(w > 0.0)) continue;
    const double target = d_target > 0.0 ? d_target : 0.0;
    const double s = delta > 0.0 ? target / delta : 0.0;
    const int32_t ru = sub_index[u], rv = sub_index[v];
    double* yu = ru >= 0 ? y_sub + (size_t)ru * dim : 0;
    double* yv = rv >= 0 ? y_sub + (size_t)rv * dim : 0;
    for (uint32_t c = 0; c < dim; ++c) {
      const double p = xu[c], q = xv[c];
      const double diff = p - q;
      if (yu) yu[c] += w * (q + s * diff);
      if (yv) yv[c] += w * (p - s * diff);
    }
    if (ru >= 0) z_sub[ru] += w;
    if (rv >= 0) z_sub[rv] += w;
  }
}
