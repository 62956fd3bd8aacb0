// Host-side numerics of the GEMPE path: the FastMath tables the device kernels evaluate, the
// per-iteration sigma search over the 2x512 distance tallies, and the relabelling permutation.
// Citations are relative to /root/reference/proj.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gempe {

// Error taxonomy of include/entropy_embed/errors.hpp:10-47, mapped onto the C-ABI return codes.
struct config_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct data_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct near_complete_graph_error : data_error { using data_error::data_error; };
struct divergence_error : std::runtime_error {
  divergence_error(const std::string& msg, int iteration)
      : std::runtime_error(msg), iteration_(iteration) {}
  int iteration() const noexcept { return iteration_; }
 private:
  int iteration_;
};
struct cuda_error : std::runtime_error { using std::runtime_error::runtime_error; };

constexpr int kSegments = 16;
constexpr int kHistBins = 512;          // histogram.hpp:15
constexpr double kHistMaxDistance = 12.0;  // histogram.hpp:16
constexpr double kDefaultMu = 1.5;      // sigmoid.hpp:9
constexpr double kSigmaMin = 1e-3, kSigmaMax = 16.0, kProbFloor = 1e-12;  // sigmoid.hpp:10-14

// Continuous 16-segment piecewise quadratic a x^2 + b x + c (piecewise.hpp:17-47).
struct QuadTable {
  std::array<double, kSegments + 1> knots{};
  std::array<double, kSegments> a{}, b{}, c{};
  double lo = 0.0, hi = 0.0;
  bool odd_mirror = false;

  double operator()(double x) const;
  int segment_of(double x) const;  // number of interior knots <= x
};

// The three tables of FastMath::build (src/piecewise.cpp:182-195).  The kernels read erf and ratio.
struct FastMathTables {
  QuadTable erf, exp_neg, ratio;
  static const FastMathTables& get();  // built once, thread-safe
  double gauss_erfc_ratio(double x) const;  // piecewise.hpp:72-79
};

double gauss_over_erfc(double x);  // sigmoid.hpp:39-45

struct Parabola { double d_target, w; };
// sigmoid.hpp:88-101; tables == nullptr selects the exact-math policy.
Parabola parabola(double delta, double mu, double sigma, bool is_edge, const FastMathTables* tables);

// Distance tallies of one round plus the non-edge reweighting (histogram.hpp, engine.cpp:293-300).
struct Tallies {
  std::array<std::uint64_t, kHistBins> edge{}, nonedge{};
  double nonedge_weight = 1.0;
  std::uint64_t edge_total() const;
  std::uint64_t nonedge_total() const;
};

double histogram_objective(const Tallies& h, double mu, double sigma);         // slope.cpp:27-38
double histogram_objective_dsigma(const Tallies& h, double mu, double sigma);  // slope.cpp:40-51
struct SigmaSearch { double sigma; int bisection_steps; };
SigmaSearch optimize_sigma(const Tallies& h, double mu);                       // slope.cpp:75-125

// rng.hpp:17-34
std::uint64_t splitmix64(std::uint64_t z);
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t component);
// graph.cpp:182-194: forward[original] = relabeled.
std::vector<std::uint32_t> random_relabel_forward(std::uint32_t n, std::uint64_t seed);
int auto_hash_bits(std::uint64_t m, int bits_override);  // hash_set.cpp:13-24

}  // namespace gempe
