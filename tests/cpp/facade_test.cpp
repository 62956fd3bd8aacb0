// C++ drop-in check: code written against the reference's interface (entropy_embed::Graph, IterationConfig,
// EmbeddingEngine, embed, the error classes) compiled unchanged against include/gempe.hpp.  The cases restate
// /root/reference/proj/tests/test_engine.cpp:115-173, 365-374 and tests/test_rng_sampler.cpp:121-129.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include <gempe.hpp>
namespace entropy_embed = gempe;
using namespace entropy_embed;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("CHECK failed at %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

static Graph graph_from_edges(std::uint32_t n, const std::vector<std::pair<std::uint32_t, std::uint32_t>>& edges) {
  Graph g;
  g.n = n;
  for (auto [a, b] : edges) {
    g.src.push_back(a);
    g.dst.push_back(b);
  }
  return g;
}

static Graph clique_pair(std::uint32_t k) {
  std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;
  for (std::uint32_t off : {0u, k})
    for (std::uint32_t i = 0; i < k; ++i)
      for (std::uint32_t j = i + 1; j < k; ++j) edges.emplace_back(off + i, off + j);
  edges.emplace_back(0u, k);
  return graph_from_edges(2 * k, edges);
}

int main() {
  {  // untouched vertices hold position
    Graph g = graph_from_edges(40, {{0, 1}});
    IterationConfig cfg;
    cfg.workers = 1;
    EmbeddingEngine engine(g, 2, cfg, 3);
    IterationCapture capture;
    engine.set_capture(&capture);
    const std::vector<float> before = engine.work_coords().coords;
    engine.run_single_iteration();
    const std::vector<float> after = engine.work_coords().coords;
    int untouched = 0;
    for (std::uint32_t v = 0; v < 40; ++v) {
      CHECK(capture.z[v] >= 0.0);
      if (capture.z[v] == 0.0) {
        ++untouched;
        CHECK(after[v * 2] == before[v * 2]);
        CHECK(after[v * 2 + 1] == before[v * 2 + 1]);
      }
    }
    CHECK(untouched >= 30);
  }
  {  // every edge and exactly two samples per edge are tallied; embed() returns finite coordinates
    Graph g = clique_pair(10);
    IterationConfig cfg;
    cfg.max_iters = 30;
    EmbedResult res = embed(g, 2, cfg, 4);
    std::uint64_t e = 0, ne = 0;
    for (auto c : res.last_histogram.edge) e += c;
    for (auto c : res.last_histogram.nonedge) ne += c;
    CHECK(e == g.edge_count());
    CHECK(ne == 2 * g.edge_count());
    CHECK(res.iterations >= 1 && res.iterations <= 30);
    CHECK(res.pe_trace.size() == static_cast<std::size_t>(res.iterations));
    for (float c : res.embedding.coords) CHECK(std::isfinite(c));
    // the two cliques separate: mean intra-clique distance well below the inter-clique one
    auto dist = [&](std::uint32_t a, std::uint32_t b) {
      const float* x = res.embedding.row(a);
      const float* y = res.embedding.row(b);
      return std::hypot(x[0] - y[0], x[1] - y[1]);
    };
    double intra = 0, inter = 0;
    int ci = 0, cx = 0;
    for (std::uint32_t a = 0; a < 20; ++a)
      for (std::uint32_t b = a + 1; b < 20; ++b) {
        if ((a < 10) == (b < 10)) intra += dist(a, b), ++ci;
        else inter += dist(a, b), ++cx;
      }
    CHECK(intra / ci < inter / cx);
    CHECK(res.relabel.forward.size() == 20 && res.relabel.inverse[res.relabel.forward[7]] == 7);
  }
  {  // the engine sharded over a device list (two ranks on device 0) reproduces the single-GPU engine bit for bit
    Graph g = clique_pair(12);
    IterationConfig cfg;
    cfg.max_iters = 12;
    cfg.deterministic = true;
    EmbedResult one = embed(g, 4, cfg, 9);
    cfg.devices = {0, 0};
    EmbedResult two = embed(g, 4, cfg, 9);
    CHECK(one.iterations == two.iterations && one.final_sigma == two.final_sigma);
    CHECK(one.embedding.coords == two.embedding.coords);
  }
  {  // two-body system settles (one edge inside a 3-vertex graph)
    Graph g = graph_from_edges(3, {{0, 1}});
    IterationConfig cfg;
    cfg.max_iters = 20;
    EmbeddingEngine engine(g, 2, cfg, 11);
    for (int it = 0; it < 20; ++it) engine.run_single_iteration();
    CHECK(engine.iteration() == 20 && engine.pe_trace().size() == 20);
    CHECK(std::isfinite(engine.sigma()));
    const auto report = engine.pe_sampled(4, 1);  // metrics.hpp pe_sampled of the current layout, on the device
    CHECK(report.pe > 0.0 && report.pe <= report.grid_pe && report.h_basic > 0.0);
  }
  {  // degenerate inputs return the initial layout
    Graph g;
    g.n = 5;
    IterationConfig cfg;
    EmbeddingEngine engine(g, 3, cfg, 11);
    CHECK(engine.degenerate());
    bool threw = false;
    try {
      engine.run_single_iteration();
    } catch (const config_error&) {
      threw = true;
    }
    CHECK(threw);
    EmbedResult res = engine.run();
    CHECK(res.degenerate && res.iterations == 0 && !res.converged && res.embedding.coords.size() == 15);
  }
  {  // error taxonomy
    Graph g = graph_from_edges(3, {{0, 1}});
    IterationConfig bad;
    bad.max_iters = 0;
    bool threw = false;
    try {
      EmbeddingEngine e(g, 2, bad, 1);
    } catch (const config_error&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      EmbeddingEngine e(g, 0, IterationConfig{}, 1);
    } catch (const config_error&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {  // K3: no non-edge exists
      Graph k3 = graph_from_edges(3, {{0, 1}, {0, 2}, {1, 2}});
      EmbeddingEngine e(k3, 2, IterationConfig{}, 3);
      e.run_single_iteration();
    } catch (const near_complete_graph_error&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      Graph oob = graph_from_edges(3, {{0, 7}});
      EmbeddingEngine e(oob, 2, IterationConfig{}, 3);
    } catch (const data_error&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // BASELINE convenience form: embed(dim, iterations, negatives, seed)
    EmbedResult res = embed(clique_pair(8), 2, 10, 5, 1);
    std::uint64_t ne = 0;
    for (auto c : res.last_histogram.nonedge) ne += c;
    CHECK(ne == 16u * 5u);
  }
  if (failures == 0) std::printf("facade_test: OK\n");
  return failures == 0 ? 0 : 1;
}
