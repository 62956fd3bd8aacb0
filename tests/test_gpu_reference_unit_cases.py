"""The reference's unit tests on the path that are statistical or behavioural rather than golden-value (those are in
test_oracle_pins.py / test_gpu_parity.py), restated against the GPU path through the C-ABI:

  edge hash set: false positives near the occupancy bound, one-sided agreement with exact membership
      (/root/reference/proj/tests/test_graph.cpp:197-231)
  sampler: uniform partners on a prime range, almost no retries on a sparse graph
      (/root/reference/proj/tests/test_rng_sampler.cpp:56-70, 84-101)
  engine: a run cut off early returns its best-PE snapshot, a fixed seed reproduces the run
      (/root/reference/proj/tests/test_engine.cpp:314-360)
"""
import numpy as np
import pytest

from conftest import clique_pair, er_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2011_03479_b200 as P
    return P


def test_hash_false_positives_stay_near_the_occupancy_bound(G):
    n, src, dst = er_graph(2000, 10000, 5)
    ctx = G.Context(G.Graph(n, src, dst), 2, 1, relabel=False)
    edges = set(zip(src.tolist(), dst.tolist())) | set(zip(dst.tolist(), src.tolist()))
    rng = np.random.default_rng(123)
    i = rng.integers(0, n, 130000).astype(np.uint32)
    j = rng.integers(0, n, 130000).astype(np.uint32)
    keep = np.array([a != b and (a, b) not in edges for a, b in zip(i.tolist(), j.tolist())])
    i, j = i[keep][:100000], j[keep][:100000]
    rate = float(ctx.probe(i, j).mean())
    assert rate <= 4.0 * (2.0 * len(src) / (1 << ctx.hash_bits))
    ctx.close()


def test_hash_is_one_sided(G):
    n, src, dst = er_graph(300, 2000, 3)
    ctx = G.Context(G.Graph(n, src, dst), 2, 1, relabel=False)
    edges = set(zip(src.tolist(), dst.tolist())) | set(zip(dst.tolist(), src.tolist()))
    rng = np.random.default_rng(77)
    i = rng.integers(0, n, 100000).astype(np.uint32)
    j = rng.integers(0, n, 100000).astype(np.uint32)
    out = ctx.probe(i, j)
    for a, b, hit in zip(i.tolist(), j.tolist(), out.tolist()):
        if not hit:
            assert (a, b) not in edges
    ctx.close()


def test_partners_are_roughly_uniform_on_a_prime_range(G):
    n = 97
    ctx = G.Context(G.Graph(n, [0], [1]), 2, 2024, neg_mode=G.NEG_PER_VERTEX_K, negatives=1000, hash_bits=20)
    partners, _ = ctx.sample(0)
    counts = np.bincount(partners, minlength=n).astype(np.float64)
    expect = partners.size / n
    sd = np.sqrt(expect * (1.0 - 1.0 / n))
    assert (np.abs(counts - expect) <= 6.0 * sd).all()
    ctx.close()


def test_sparse_graph_needs_almost_no_retries(G):
    # hash_bits = 14 as in the reference's test: the contract is about rejection, not table collisions
    ctx = G.Context(G.Graph(1000, [0], [1]), 2, 77, neg_mode=G.NEG_PER_VERTEX_K, negatives=100, hash_bits=14)
    partners, draws = ctx.sample(0)
    mean = draws / partners.size
    assert 1.0 <= mean < 1.01
    ctx.close()


@pytest.mark.parametrize("queued", [False, True])
def test_a_run_cut_off_early_returns_its_best_pe_snapshot(G, queued):
    n, src, dst = er_graph(30, 60, 2)
    g = G.Graph(n, src, dst)
    exercised = False
    for seed in range(1, 31):
        cfg = G.IterationConfig(max_iters=12, deterministic=True)
        engine = G.EmbeddingEngine(g, 2, cfg, seed)
        states, trace = [], []
        for _ in range(cfg.max_iters):
            trace.append(engine.run_single_iteration().pe_estimate)
            states.append(engine.work_coords())
        best = int(np.argmin(trace))  # first minimum, like the strict `<` of the reference's loop
        if trace[best] >= trace[-1]:
            engine.close()
            continue  # want an interior minimum
        exercised = True
        if queued:  # the same run with the loop on the device: the snapshot is taken by the device
            engine.close()
            res = G.embed(g, 2, cfg, seed)
        else:       # budget exhausted: run() finalises immediately
            res = engine.run()
            engine.close()
        assert not res.converged
        assert np.array_equal(res.pe_trace, np.array(trace))
        for v in range(n):
            w = int(res.relabel_forward[v])
            assert np.array_equal(res.embedding[v].view(np.uint32), states[best][w].view(np.uint32))
        break
    assert exercised


def test_fixed_seed_reproduces_the_run(G):
    n, src, dst = clique_pair(8)
    cfg = G.IterationConfig(deterministic=True)
    a = G.embed(G.Graph(n, src, dst), 2, cfg, 6)
    b = G.embed(G.Graph(n, src, dst), 2, cfg, 6)
    assert np.array_equal(a.embedding.view(np.uint32), b.embedding.view(np.uint32))
    assert np.array_equal(a.pe_trace, b.pe_trace)


def test_result_download_through_the_staging_ring(G, monkeypatch):
    """embed() exports the embedding through a ring of pinned chunks drained by host threads (large results); with a tiny
    chunk size a small result takes the same path, ring wrap-around and ragged last chunk included."""
    n, src, dst = er_graph(1201, 6000, 4)
    cfg = G.IterationConfig(max_iters=6, deterministic=True)
    plain = G.embed(G.Graph(n, src, dst), 7, cfg, 2)
    monkeypatch.setenv("GEMPE_DOWNLOAD_CHUNK", "1000")  # 1201 * 7 * 4 bytes = 33.6 chunks, ring of 6
    staged = G.embed(G.Graph(n, src, dst), 7, cfg, 2)
    assert np.array_equal(plain.embedding.view(np.uint32), staged.embedding.view(np.uint32))
    assert np.isfinite(staged.embedding).all() and np.abs(staged.embedding).sum() > 0
