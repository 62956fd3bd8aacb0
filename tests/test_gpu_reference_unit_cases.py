"""The reference's unit tests on the path that are statistical or behavioural rather than golden-value (those are in
test_oracle_pins.py / test_gpu_parity.py), restated against the GPU path through the C-ABI:

  edge hash set: false positives near the occupancy bound, one-sided agreement with exact membership
      (/root/reference/proj/tests/test_graph.cpp:197-231)
  sampler: uniform partners on a prime range, almost no retries on a sparse graph
      (/root/reference/proj/tests/test_rng_sampler.cpp:56-70, 84-101)
  engine: a run cut off early returns its best-PE snapshot, a fixed seed reproduces the run
      (/root/reference/proj/tests/test_engine.cpp:314-360); a two-body system settles at its parabola target (:160-173);
      the PE trace trends down over 10-iteration windows (:376-396); coincident points contribute w * other (:57-61)
  sampler: accepted pairs are never true edges (test_rng_sampler.cpp:103-119)
  sigma search on the device tallies: separated masses drive sigma to the bracket floor, a symmetric histogram terminates
      (test_histogram_slope.cpp:68-123)
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


def test_two_body_system_settles_at_its_parabola_target(G, oracle, golden_fastmath):
    # one edge inside a 3-vertex graph so that non-edge sampling stays feasible
    g = G.Graph(3, [0], [1])
    engine = G.EmbeddingEngine(g, 2, G.IterationConfig(max_iters=20), 11)
    for _ in range(20):
        engine.run_single_iteration()
    ws, wd, _ = engine.work_graph()
    x = engine.work_coords().astype(np.float64)
    delta = float(np.sqrt(((x[ws[0]] - x[wd[0]]) ** 2).sum()))
    d_target, _ = oracle.parabola(delta, 1.5, engine.sigma(), True, golden_fastmath)
    assert abs(delta - abs(d_target)) <= 0.05 * abs(d_target)
    engine.close()


def test_pe_trace_trends_down_over_ten_iteration_windows(G):
    n, src, dst = clique_pair(10)
    cfg = G.IterationConfig(max_iters=60, convergence_window=61)  # run all iterations
    res = G.embed(G.Graph(n, src, dst), 2, cfg, 2)
    assert len(res.pe_trace) >= 30
    med = [float(np.median(res.pe_trace[s:s + 10])) for s in range(len(res.pe_trace) - 9)]
    for prev, cur in zip(med, med[1:]):
        assert cur <= prev + max(1e-6, 0.002 * prev)  # sampling noise allows hairline upticks once the trace is flat


def test_coincident_points_contribute_weight_times_the_other_point(G, oracle, golden_fastmath):
    """delta = 0: no direction to move along, add_pair's scale factor is 0 and the pair adds w * x_other (engine.cpp:58-72)."""
    n, src, dst = 4, [0, 2], [1, 3]
    for dim in (2, 16, 128):
        ctx = G.Context(G.Graph(n, src, dst), dim, 5, relabel=False, neg_mode=G.NEG_PER_VERTEX_K, negatives=0)
        ctx.set_capture(True)
        x = np.zeros((n, dim), np.float32)
        x[0] = x[1] = np.linspace(0.25, 1.0, dim, dtype=np.float32)  # the edge (0, 1) joins coincident points
        x[2], x[3] = 0.5, -0.5
        ctx.set_coords(x)
        ctx.iterate(1.5, 1.0, 0)
        y, z = ctx.get_yz()
        _, w = oracle.parabola(0.0, 1.5, 1.0, True, golden_fastmath)
        assert w > 0
        assert np.allclose(z[:2], np.float32(w), rtol=1e-6)
        assert np.allclose(y[0], np.float32(w) * x[1].astype(np.float64), rtol=1e-5)
        assert np.array_equal(ctx.get_coords()[:2], x[:2])  # y / z = the common point: nobody moves
        ctx.close()


def test_accepted_pairs_are_never_true_edges(G):
    n, src, dst = er_graph(400, 12000, 8)  # dense enough for frequent rejections
    for mode, k in ((G.NEG_PER_EDGE_2, 0), (G.NEG_PER_VERTEX_K, 30)):
        ctx = G.Context(G.Graph(n, src, dst), 2, 9, neg_mode=mode, negatives=k)
        ws, wd, _ = ctx.work_graph()
        edges = set(zip(ws.tolist(), wd.tolist())) | set(zip(wd.tolist(), ws.tolist()))
        anchors = np.stack([ws, wd], 1).ravel() if mode == G.NEG_PER_EDGE_2 else np.repeat(np.arange(n), k)
        for it in range(3):
            partners, draws = ctx.sample(it)
            assert anchors.size == partners.size and draws > 1.05 * partners.size  # many draws were rejected
            bad = [(a, p) for a, p in zip(anchors.tolist(), partners.tolist()) if a == p or (a, p) in edges]
            assert not bad, bad[:5]
        ctx.close()


def test_device_sigma_search_on_special_tallies(G):
    """optimize_sigma on tallies written by hand into the device histogram: well separated masses (edges short, non-edges
    long) drive sigma to the bracket floor 1e-3; a histogram symmetric about mu terminates; both equal the host search."""
    import torch
    from paper_2011_03479_b200 import engine as E
    from paper_2011_03479_b200.sharded import _DeviceArray
    n, src, dst = er_graph(50, 100, 1)
    ctx = G.Context(G.Graph(n, src, dst), 2, 1)
    pairs, m = n * (n - 1) // 2, len(src)
    tallies = torch.as_tensor(_DeviceArray(ctx.device_tallies(), (1024,), "<i8"), device="cuda:0")

    def device_search(he, hn, sigma_prev):
        ctx.set_sigma(1.5, sigma_prev)
        ctx.sync()
        tallies.copy_(torch.from_numpy(np.r_[he, hn].astype(np.int64)))
        torch.cuda.synchronize()
        ctx.sigma_update_async()
        return ctx.sigma_state()

    he, hn = np.zeros(512, np.uint64), np.zeros(512, np.uint64)
    he[int(0.3 / 12.0 * 512)] = 1000   # edges at 0.3
    hn[int(4.0 / 12.0 * 512)] = 1000   # non-edges at 4.0: mu = 1.5 separates them perfectly
    nw = (pairs - m) / 1000.0
    sigma, steps = E.optimize_sigma(he, hn, nw, 1.5)
    assert steps <= 60 and sigma <= 2e-3
    s_dev, pe_dev, nw_dev = device_search(he, hn, 1.0)
    assert abs(s_dev - sigma) <= 1e-9 and abs(nw_dev - nw) <= 1e-12 * nw
    assert abs(pe_dev - E.histogram_objective(he, hn, nw, 1.5, sigma) / pairs) <= 1e-9

    sym_e, sym_n = np.zeros(512, np.uint64), np.zeros(512, np.uint64)
    for off in (-20, -10, 10, 20):
        sym_e[64 + off] += 500   # bin 64 starts at delta = 1.5
        sym_n[64 + off] += 500
    nw = (pairs - m) / 2000.0
    s2, steps2 = E.optimize_sigma(sym_e, sym_n, nw, 1.5)
    assert steps2 <= 60 and 1e-3 <= s2 <= 16.0
    s_dev, _, _ = device_search(sym_e, sym_n, 16.0)  # previous sigma at the ceiling: the growth cap does not bind
    assert abs(s_dev - s2) <= 1e-9 * s2
    ctx.close()


def test_device_memory_cache_reuses_blocks_without_changing_results(G):
    """Device memory of a destroyed engine is kept and handed to the next one (context.hpp: device_alloc): same results,
    no growth of the process's device memory on the second call, everything back at the driver after a trim."""
    import torch
    n, src, dst = er_graph(20000, 200000, 3)
    g = G.Graph(n, src, dst)
    cfg = G.IterationConfig(max_iters=4, deterministic=True)
    G.trim_device_cache()
    a = G.embed(g, 32, cfg, 5)
    free_after_first = torch.cuda.mem_get_info()[0]
    b = G.embed(g, 32, cfg, 5)
    assert np.array_equal(a.embedding.view(np.uint32), b.embedding.view(np.uint32)) and np.array_equal(a.pe_trace, b.pe_trace)
    assert torch.cuda.mem_get_info()[0] >= free_after_first - (8 << 20)
    G.trim_device_cache()
    assert torch.cuda.mem_get_info()[0] >= free_after_first + (16 << 20)
    c = G.embed(g, 32, cfg, 5)  # and from a cold cache again
    assert np.array_equal(a.embedding.view(np.uint32), c.embedding.view(np.uint32))


def test_page_locked_buffers_through_the_abi(G):
    """gempe_alloc_host / gempe_free_host: a caller without CUDA headers gets page-locked coordinate vectors; the round on
    them gives the same bits as on pageable memory."""
    n, src, dst = er_graph(3000, 20000, 6)
    ctx = G.Context(G.Graph(n, src, dst), 32, 3, deterministic=True)
    x0 = ctx.get_coords()
    plain_in, plain_out = x0.copy(), np.zeros_like(x0)
    he0, hn0 = ctx.step_host(plain_in, plain_out, 1.5, 1.0, 0)
    pin_in, pin_out = G.alloc_host(x0.shape), G.alloc_host(x0.shape)
    try:
        pin_in[:] = x0
        pin_out[:] = 0
        he1, hn1 = ctx.step_host(pin_in, pin_out, 1.5, 1.0, 0)
        assert np.array_equal(he0, he1) and np.array_equal(hn0, hn1)
        assert np.array_equal(plain_out.view(np.uint32), pin_out.view(np.uint32))
    finally:
        G.free_host(pin_in)
        G.free_host(pin_out)
    ctx.close()


@pytest.mark.parametrize("dim", [2, 32, 128])
def test_step_host_on_pageable_vectors_through_the_staging_ring(G, monkeypatch, dim):
    """gempe_step_host with ordinary (pageable) numpy arrays and a tiny ring chunk: upload and slice-by-slice download both
    go through the pinned ring and its host threads; same bits as set_coords + iterate + get_coords."""
    n, src, dst = er_graph(2500, 15000, 12)
    g = G.Graph(n, src, dst)
    ref_ctx = G.Context(g, dim, 4, deterministic=True)
    x0 = ref_ctx.get_coords()
    he0, hn0 = ref_ctx.iterate(1.5, 1.0, 0)
    x1 = ref_ctx.get_coords()
    ref_ctx.close()
    monkeypatch.setenv("GEMPE_DOWNLOAD_CHUNK", "4096")
    ctx = G.Context(g, dim, 4, deterministic=True)
    x_in, x_out = x0.copy(), np.full_like(x0, np.nan)
    he1, hn1 = ctx.step_host(x_in, x_out, 1.5, 1.0, 0)
    assert np.array_equal(he0, he1) and np.array_equal(hn0, hn1)
    assert np.array_equal(x_out.view(np.uint32), x1.view(np.uint32))
    assert np.array_equal(ctx.get_coords().view(np.uint32), x1.view(np.uint32))
    ctx.close()
