// Host numerics of the GEMPE path (see hostmath.hpp).  Written from the published formulas; citations
// point at the reference implementation whose results these must reproduce (relative to
// /root/reference/proj).
#include "hostmath.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <mutex>

namespace gempe {

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr double kLn2 = 0.693147180559945309417232121458176568;
constexpr double kSqrt2 = 1.41421356237309504880168872420969808;
constexpr double kSqrtPi = 1.77245385090551602729816748334;
constexpr double kSqrt2Pi = 2.50662827463100050241576528481;
constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// ---- L2 projection onto continuous piecewise quadratics -------------------------------------------
// Hierarchical P2 basis per segment [k_s, k_{s+1}], t = (x-k_s)/h: two hats (1-t), t that carry the
// shared knot values v_s, v_{s+1}, and one bubble t(1-t) with coefficient e_s.  The normal equations
// M c = r use the exact element mass matrix and an 8-point Gauss-Legendre load vector per segment -- the
// same projection FastMath::build computes (src/piecewise.cpp:58-112), solved here by Cholesky.

struct GaussLegendre8 {
  double node[8], weight[8];
  GaussLegendre8() {
    // roots of P_8 by Newton from the Chebyshev guess; weights 2 / ((1-x^2) P_8'(x)^2)
    for (int i = 0; i < 8; ++i) {
      double x = -std::cos(kPi * (i + 0.75) / 8.5);
      double dp = 1.0;
      for (int it = 0; it < 100; ++it) {
        double p0 = 1.0, p1 = x;
        for (int k = 2; k <= 8; ++k) {
          const double pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
          p0 = p1;
          p1 = pk;
        }
        dp = 8.0 * (x * p1 - p0) / (x * x - 1.0);
        const double step = p1 / dp;
        x -= step;
        if (std::fabs(step) < 1e-16) break;
      }
      {
        double p0 = 1.0, p1 = x;
        for (int k = 2; k <= 8; ++k) {
          const double pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
          p0 = p1;
          p1 = pk;
        }
        dp = 8.0 * (x * p1 - p0) / (x * x - 1.0);
      }
      node[i] = x;
      weight[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
  }
};

// In-place Cholesky solve of the dense SPD system (dim <= 33).
void solve_spd(std::vector<double>& m, std::vector<double>& rhs, int dim) {
  for (int j = 0; j < dim; ++j) {
    double d = m[j * dim + j];
    for (int k = 0; k < j; ++k) d -= m[j * dim + k] * m[j * dim + k];
    if (!(d > 1e-300)) throw config_error("piecewise fit failed: singular system");
    const double l = std::sqrt(d);
    m[j * dim + j] = l;
    for (int i = j + 1; i < dim; ++i) {
      double s = m[i * dim + j];
      for (int k = 0; k < j; ++k) s -= m[i * dim + k] * m[j * dim + k];
      m[i * dim + j] = s / l;
    }
  }
  for (int i = 0; i < dim; ++i) {  // L y = r
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s -= m[i * dim + k] * rhs[k];
    rhs[i] = s / m[i * dim + i];
  }
  for (int i = dim - 1; i >= 0; --i) {  // L^T c = y
    double s = rhs[i];
    for (int k = i + 1; k < dim; ++k) s -= m[k * dim + i] * rhs[k];
    rhs[i] = s / m[i * dim + i];
  }
}

QuadTable project(const std::function<double(double)>& f,
                  const std::array<double, kSegments + 1>& knots, double lo, double hi,
                  bool pin_origin, bool odd_mirror, double max_abs_error) {
  static const GaussLegendre8 gl;
  // unknown order: knot value v_i at 2i, bubble e_s at 2s+1  (33 unknowns, band width 2)
  const int dim = 2 * kSegments + 1;
  std::vector<double> mass(static_cast<std::size_t>(dim) * dim, 0.0), load(dim, 0.0);
  for (int s = 0; s < kSegments; ++s) {
    const double k0 = knots[s], h = knots[s + 1] - knots[s];
    const int idx[3] = {2 * s, 2 * s + 2, 2 * s + 1};  // hat0, hat1, bubble
    const double em[3][3] = {{h / 3, h / 6, h / 12}, {h / 6, h / 3, h / 12}, {h / 12, h / 12, h / 30}};
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) mass[idx[p] * dim + idx[q]] += em[p][q];
    for (int g = 0; g < 8; ++g) {
      const double t = 0.5 * (gl.node[g] + 1.0);
      const double wf = 0.5 * h * gl.weight[g] * f(k0 + h * t);
      load[idx[0]] += wf * (1.0 - t);
      load[idx[1]] += wf * t;
      load[idx[2]] += wf * t * (1.0 - t);
    }
  }
  if (pin_origin) {  // v_0 = 0 (odd function fitted on [0, B])
    for (int k = 0; k < dim; ++k) mass[k] = mass[k * dim] = 0.0;
    mass[0] = 1.0;
    load[0] = 0.0;
  }
  solve_spd(mass, load, dim);

  QuadTable q;
  q.knots = knots;
  q.lo = lo;
  q.hi = hi;
  q.odd_mirror = odd_mirror;
  for (int s = 0; s < kSegments; ++s) {
    const double k0 = knots[s], h = knots[s + 1] - knots[s];
    const double v0 = load[2 * s], v1 = load[2 * s + 2], e = load[2 * s + 1];
    // v0 + (v1 - v0 + e) t - e t^2 expanded in x
    const double alpha = (v1 - v0 + e) / h;
    const double beta = -e / (h * h);
    q.a[s] = beta;
    q.b[s] = alpha - 2.0 * beta * k0;
    q.c[s] = v0 - alpha * k0 + beta * k0 * k0;
  }
  double worst = 0.0;  // same acceptance check as the reference build (piecewise.cpp:129-142)
  for (int i = 0; i <= 20000; ++i) {
    const double x = lo + (hi - lo) * i / 20000;
    worst = std::max(worst, std::fabs(q(x) - f(x)));
  }
  if (worst > max_abs_error) {
    throw config_error("piecewise fit failed: max abs error " + std::to_string(worst));
  }
  return q;
}

FastMathTables build_tables() {
  FastMathTables t;
  std::array<double, kSegments + 1> knots;
  // erf on [-6, 6]: odd-mirrored fit over [0, 6], uniform knots (piecewise.cpp:147-158)
  for (int k = 0; k <= kSegments; ++k) knots[k] = 6.0 * k / kSegments;
  t.erf = project([](double x) { return std::erf(x); }, knots, -6.0, 6.0, true, true, 1e-3);
  // exp(-x) on [0, 32]: geometric knots, ratio 1.35 (piecewise.cpp:161-176)
  const double rho = 1.35, denom = std::pow(rho, kSegments) - 1.0;
  for (int k = 0; k <= kSegments; ++k) knots[k] = 32.0 * (std::pow(rho, k) - 1.0) / denom;
  knots[kSegments] = 32.0;
  t.exp_neg = project([](double x) { return std::exp(-x); }, knots, 0.0, 32.0, false, false, 1e-3);
  // e^{-x^2}/erfc(x) on [-1, 8]: the published knot placement (piecewise.cpp:185-187)
  knots = {-1.0, -0.6, -0.3, 0.0, 0.3, 0.6, 0.9, 1.2, 1.6, 2.0, 2.5, 3.0, 3.75, 4.5, 5.5, 6.75, 8.0};
  t.ratio = project(gauss_over_erfc, knots, -1.0, 8.0, false, false, 5e-4);
  return t;
}

// -log2(clamped probability), exact erf (sigmoid.hpp:69-81 with ExactMath)
double description_length(double delta, double mu, double sigma, bool is_edge) {
  const double u = (delta - mu) / (kSqrt2 * sigma);
  const double e = std::erf(u);
  const double s = is_edge ? 0.5 - 0.5 * e : 0.5 + 0.5 * e;
  return -std::log2(std::clamp(s, kProbFloor, 1.0 - kProbFloor));
}

// unfloored coding cost -log2(erfc(x)/2) (sigmoid.hpp:50-59)
double coding_cost_tail(double delta, double mu, double sigma, bool is_edge) {
  const double u = (delta - mu) / (kSqrt2 * sigma);
  const double x = is_edge ? u : -u;
  if (x <= 6.0) return 1.0 - std::log2(std::erfc(x));
  const double r = 1.0 / (x * x);
  const double series = 1.0 + r * (-0.5 + r * (0.75 + r * (-1.875 + 6.5625 * r)));
  return 1.0 - (-x * x - std::log(x * kSqrtPi) + std::log(series)) / kLn2;
}

// d(dl)/d(sigma) (sigmoid.hpp:108-113 with ExactMath)
double coding_cost_dsigma(double delta, double mu, double sigma, bool is_edge) {
  const double u = (delta - mu) / (kSqrt2 * sigma);
  const double v = 2.0 / (kSqrtPi * kLn2) * u * gauss_over_erfc(is_edge ? u : -u) / sigma;
  return is_edge ? -v : v;
}

template <typename Cost>
double weighted_cost(const Tallies& h, double mu, double sigma, Cost cost) {
  double total = 0.0;
  for (int b = 0; b < kHistBins; ++b) {
    const std::uint64_t ec = h.edge[b], nc = h.nonedge[b];
    if (!ec && !nc) continue;
    const double mid = (b + 0.5) * kHistMaxDistance / kHistBins;  // histogram.hpp:52
    if (ec) total += static_cast<double>(ec) * cost(mid, mu, sigma, true);
    if (nc) total += h.nonedge_weight * static_cast<double>(nc) * cost(mid, mu, sigma, false);
  }
  return total;
}

}  // namespace

int QuadTable::segment_of(double x) const {
  int s = 0;
  for (int i = 1; i < kSegments; ++i) s += (x >= knots[i]);
  return s;
}

double QuadTable::operator()(double x) const {
  double xa = std::clamp(x, lo, hi);
  double flip = 1.0;
  if (odd_mirror && xa < 0.0) {
    xa = -xa;
    flip = -1.0;
  }
  const int s = segment_of(xa);
  return flip * ((a[s] * xa + b[s]) * xa + c[s]);
}

const FastMathTables& FastMathTables::get() {
  static const FastMathTables tables = build_tables();
  return tables;
}

double gauss_over_erfc(double x) {
  if (x <= 6.0) return std::exp(-x * x) / std::erfc(x);
  const double r = 1.0 / (x * x);
  const double series = 1.0 + r * (-0.5 + r * (0.75 + r * (-1.875 + 6.5625 * r)));
  return x * kSqrtPi / series;
}

double FastMathTables::gauss_erfc_ratio(double x) const {
  if (x >= ratio.lo) return x > ratio.hi ? gauss_over_erfc(x) : ratio(x);
  if (x < -6.0) return 0.0;
  return std::exp(-x * x) / (1.0 - erf(x));
}

Parabola parabola(double delta, double mu, double sigma, bool is_edge, const FastMathTables* tables) {
  const double u = (delta - mu) / (kSqrt2 * sigma);
  const double sign = is_edge ? -1.0 : 1.0;
  const double x = is_edge ? u : -u;
  const double g = tables ? tables->gauss_erfc_ratio(x) : gauss_over_erfc(x);
  const double s2 = sigma * sigma;
  const double c1 = 2.0 / (kPi * kLn2), c2 = 1.0 / (kSqrt2Pi * kLn2);
  const double w = c1 * g * g / s2 + sign * c2 * (delta - mu) * g / (s2 * sigma);
  if (!(w > 0.0)) return {delta, 0.0};
  return {delta + sign * c2 * g / (w * sigma), w};
}

std::uint64_t Tallies::edge_total() const {
  std::uint64_t t = 0;
  for (auto c : edge) t += c;
  return t;
}
std::uint64_t Tallies::nonedge_total() const {
  std::uint64_t t = 0;
  for (auto c : nonedge) t += c;
  return t;
}

double histogram_objective(const Tallies& h, double mu, double sigma) {
  return weighted_cost(h, mu, sigma, description_length);
}
double histogram_objective_dsigma(const Tallies& h, double mu, double sigma) {
  return weighted_cost(h, mu, sigma, coding_cost_dsigma);
}

namespace {

// Root of an increasing sign change: f(a) < 0 < f(b).  Halves [a, b] until it is no wider than `width` or `budget`
// halvings are spent (counted in *used); an exact zero ends the walk at that point.  Returns the centre of the last
// interval.  The visited midpoints are those of slope.cpp:104-120, so sigma agrees with the reference bit for bit.
template <typename F>
double centre_of_sign_change(F&& f, double a, double b, double width, int budget, int* used) {
  while (b - a > width && *used < budget) {
    ++*used;
    const double c = 0.5 * (a + b);
    const double fc = f(c);
    if (fc == 0.0) return c;
    if (fc > 0.0) b = c; else a = c;
  }
  return 0.5 * (a + b);
}

}  // namespace

// optimize_sigma_detail (slope.cpp:75-125): the derivative of the cost in sigma can change sign several times on the
// tallies of an unsettled layout, so the basin is located first -- 17 log-spaced candidates between the sigma bounds,
// scored with the unfloored cost -- and only the two cells around the cheapest candidate are searched for the zero of
// the derivative.  The refined value replaces the candidate only if it is not more expensive.
SigmaSearch optimize_sigma(const Tallies& h, double mu) {
  if (h.edge_total() == 0 && h.nonedge_total() == 0) throw config_error("cannot optimize sigma on an empty histogram");
  constexpr int kCandidates = 17;
  std::array<double, kCandidates> candidate{}, price{};
  for (int i = 0; i < kCandidates; ++i) {
    candidate[i] = kSigmaMin * std::pow(kSigmaMax / kSigmaMin, static_cast<double>(i) / (kCandidates - 1));
    price[i] = weighted_cost(h, mu, candidate[i], coding_cost_tail);
  }
  const int cheapest = static_cast<int>(std::min_element(price.begin(), price.end()) - price.begin());  // first minimum
  SigmaSearch found{candidate[cheapest], 0};
  const double left = candidate[cheapest > 0 ? cheapest - 1 : 0];
  const double right = candidate[cheapest + 1 < kCandidates ? cheapest + 1 : kCandidates - 1];
  auto slope = [&](double sigma) { return histogram_objective_dsigma(h, mu, sigma); };
  const double slope_left = slope(left), slope_right = slope(right);
  if (slope_left < 0.0 && slope_right > 0.0) {
    const double refined = centre_of_sign_change(slope, left, right, 1e-4, 60, &found.bisection_steps);
    if (weighted_cost(h, mu, refined, coding_cost_tail) <= price[cheapest]) found.sigma = refined;
  }
  return found;
}

std::uint64_t splitmix64(std::uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t component) {
  return splitmix64(seed ^ (kGolden * (component + 1)));
}

std::vector<std::uint32_t> random_relabel_forward(std::uint32_t n, std::uint64_t seed) {
  std::vector<std::uint32_t> fwd(n);
  for (std::uint32_t i = 0; i < n; ++i) fwd[i] = i;
  std::uint64_t state = mix_seed(seed, 0x5eedu);
  for (std::uint32_t i = 0; i + 1 < n; ++i) {  // Fisher-Yates, multiply-shift bounded draw
    state = splitmix64(state);
    const std::uint64_t j = i + static_cast<std::uint64_t>(
        (static_cast<unsigned __int128>(state) * (n - i)) >> 64);
    std::swap(fwd[i], fwd[j]);
  }
  return fwd;
}

int auto_hash_bits(std::uint64_t m, int bits_override) {
  if (bits_override != 0) {
    if (bits_override < 1 || bits_override > 31) throw config_error("hash table bits must be in [1,31]");
    return bits_override;
  }
  int bits = 6;
  const std::uint64_t target = 64ull * std::max<std::uint64_t>(m, 1);
  while ((1ull << bits) < target) ++bits;
  return std::min(bits, 31);
}

}  // namespace gempe
