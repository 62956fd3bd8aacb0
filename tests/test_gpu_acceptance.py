"""The reference's acceptance criteria that concern this path (/root/reference/proj/tests/acceptance.cpp), run against
the GPU engine through the same public surface (`embed`, `EmbeddingEngine`): c1 two-clique separation (:68-101), c2 ring
ordering (:104-141), c8 sigma optimiser on the final tallies (:358-377), c9 linear scaling of the iteration in m at
d = 128 (:380-456; sizes scaled up to what a GPU iteration needs to be more than launch overhead).  c4-c7 (reduction
equivalence, sampler soundness, hash contract, approximation quality) are the parity tests of test_gpu_parity.py and
test_oracle_pins.py; c3 is red by design in the reference; c10 is the CLI (out of scope)."""
import numpy as np
import pytest

from conftest import clique_pair, ring

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2011_03479_b200 as P
    return P


def _row_distance(x, i, j):
    return float(np.sqrt(((x[i].astype(np.float64) - x[j].astype(np.float64)) ** 2).sum()))


def test_criterion1_two_cliques_separate(G, ref):
    n, src, dst = clique_pair(10)
    assert n == 20 and len(src) == 91
    good, worst_pe = 0, 0.0
    for seed in range(1, 11):
        res = G.embed(G.Graph(n, src, dst), 2, G.IterationConfig(), seed)
        max_intra, min_inter = 0.0, 1e300
        for i in range(20):
            for j in range(i + 1, 20):
                d = _row_distance(res.embedding, i, j)
                same = (i < 10) == (j < 10)
                if same:
                    max_intra = max(max_intra, d)
                elif not (i == 0 and j == 10):
                    min_inter = min(min_inter, d)
        pe = ref.pe_exact(n, src, dst, res.embedding)
        worst_pe = max(worst_pe, pe)
        good += max_intra < min_inter and pe <= 0.10
    assert good >= 9, (good, worst_pe)


def test_criterion2_ring_orders_edges_before_non_edges(G):
    n, src, dst = ring(100)
    edges = set(zip(src.tolist(), dst.tolist())) | set(zip(dst.tolist(), src.tolist()))
    worst_ratio, trace_ok = 0.0, 0
    for seed in range(1, 11):
        res = G.embed(G.Graph(n, src, dst), 2, G.IterationConfig(), seed)
        trace_ok += res.pe_trace[-1] < res.pe_trace[0]
        edge_mean = np.mean([_row_distance(res.embedding, a, b) for a, b in zip(src.tolist(), dst.tolist())])
        rng = np.random.default_rng(seed)
        dists = []
        while len(dists) < 10000:
            i, j = (int(v) for v in rng.integers(0, n, 2))
            if i != j and (i, j) not in edges:
                dists.append(_row_distance(res.embedding, i, j))
        worst_ratio = max(worst_ratio, edge_mean / np.mean(dists))
    assert worst_ratio < 0.5 and trace_ok == 10, (worst_ratio, trace_ok)


def test_criterion8_sigma_of_the_final_tallies_is_a_minimum(G):
    from paper_2011_03479_b200 import engine as E
    n, src, dst = clique_pair(10)
    res = G.embed(G.Graph(n, src, dst), 2, G.IterationConfig(), 1)
    he, hn, w = res.last_hist_edge, res.last_hist_nonedge, res.last_nonedge_weight
    sigma, steps = E.optimize_sigma(he, hn, w, 1.5)
    assert steps <= 60
    f_star = E.histogram_objective(he, hn, w, 1.5, sigma)
    for candidate in (sigma / 2.0, 2.0 * sigma):
        clipped = min(max(candidate, 1e-3), 16.0)
        assert f_star <= E.histogram_objective(he, hn, w, 1.5, clipped) + 1e-6


def test_criterion9_iteration_time_is_linear_in_m(G):
    """Doubling m doubles the device time of an iteration (factor in [1.6, 2.6], the reference's band) at d = 128."""
    import torch
    from paper_2011_03479_b200 import graphgen
    times = []
    for scale in (17, 18, 19):  # ~1.9 M / 3.9 M / 7.8 M edges
        n, src, dst = graphgen.rmat(scale=scale, edge_factor=16, seed=scale, device=torch.device("cuda", 0))
        ctx = G.Context(G.Graph(n, src, dst), 128, 3)
        for it in range(3):
            ctx.iterate_async(1.5, 1.0, it)
        ctx.sync()
        ctx.elapsed_ms()
        for it in range(3, 13):
            ctx.iterate_async(1.5, 1.0, it)
        ctx.sync()
        times.append((len(src), ctx.elapsed_ms()[0] / 10))
        ctx.close()
    for (m0, t0), (m1, t1) in zip(times, times[1:]):
        factor = (t1 / t0) / (m1 / m0) * 2.0  # normalised to an exact doubling of m
        assert 1.6 <= factor <= 2.6, times
