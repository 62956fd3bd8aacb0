"""The C++ multi-GPU host (gempe_group, csrc/group.cpp) through the C-ABI: several ranks in ONE process.  Only one GPU
is available to the tests, so every rank lives on device 0 -- the ranks' kernels run on their own streams, ordered by
CUDA events only (no kernel waits on another rank), and move their data exactly as on several GPUs: as stores into the
other ranks' buffers (peer path) or as cudaMemcpyPeerAsync copies (copy-engine path).  The bar is the single context:
bit-identical coordinates and tallies in deterministic mode."""
import numpy as np
import pytest

from conftest import er_graph, star_plus_ring

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2011_03479_b200 as P
    return P


def _single_rounds(G, g, dim, seed, rounds, **kw):
    ctx = G.Context(g, dim, seed, deterministic=True, **kw)
    out, sigma = [], 1.0
    for it in range(rounds):
        he, hn = ctx.iterate(1.5, sigma, it)
        out.append((he.tolist(), hn.tolist()))
        sigma = min(sigma * 1.4, 2.5)
    x = ctx.get_coords()
    ctx.close()
    return out, x


@pytest.mark.parametrize("copy_engines", [False, True])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_group_rounds_are_bit_identical_to_one_context(G, world, copy_engines):
    cases = [(er_graph(700, 4000, 3), 2, dict()), (er_graph(500, 2500, 4), 128, dict(neg_mode=1, negatives=7)),
             (star_plus_ring(600, hubs=2), 64, dict(chunk_entries=16))]
    for (n, src, dst), dim, kw in cases:
        g = G.Graph(n, src, dst)
        want, x_want = _single_rounds(G, g, dim, 11, 4, **kw)
        grp = G.Group(g, dim, 11, devices=[0] * world, copy_engines=copy_engines, deterministic=True, **kw)
        assert grp.world == world
        assert ("copy engines" in grp.exchange_path) == copy_engines
        sigma = 1.0
        for it in range(4):
            he, hn = grp.iterate(1.5, sigma, it)
            assert (he.tolist(), hn.tolist()) == want[it], (dim, it)
            sigma = min(sigma * 1.4, 2.5)
        assert grp.replicas_agree()
        assert np.array_equal(grp.get_coords().view(np.uint32), x_want.view(np.uint32))
        grp.close()


@pytest.mark.parametrize("copy_engines", [False, True])
def test_group_sigma_feedback_and_relabel_follow_one_context(G, copy_engines):
    n, src, dst = er_graph(900, 5000, 7)
    g = G.Graph(n, src, dst)
    one = G.Context(g, 16, 3, deterministic=True)
    grp = G.Group(g, 16, 3, devices=[0, 0, 0], copy_engines=copy_engines, deterministic=True)
    one.set_sigma(1.5, 1.0)
    grp.set_sigma(1.5, 1.0)
    for it in range(6):
        if it == 3:  # periodic re-relabel (engine.cpp:281-283): every rank rebuilds, the peers are registered again
            one.relabel(12345)
            grp.relabel(12345)
        s1, pe1, nw1, he1, hn1 = one.iterate_auto(it)
        s2, pe2, nw2, he2, hn2 = grp.iterate_auto(it)
        assert (s1, pe1, nw1) == (s2, pe2, nw2), it
        assert np.array_equal(he1, he2) and np.array_equal(hn1, hn2)
    assert grp.replicas_agree()
    assert np.array_equal(grp.get_coords().view(np.uint32), one.get_coords().view(np.uint32))
    one.close()
    grp.close()


def test_group_of_one_and_errors(G):
    n, src, dst = er_graph(300, 1200, 2)
    g = G.Graph(n, src, dst)
    grp = G.Group(g, 4, 5, devices=[0], deterministic=True)
    want, x_want = _single_rounds(G, g, 4, 5, 2)
    assert [tuple(map(list, grp.iterate(1.5, s, it))) for it, s in ((0, 1.0), (1, 1.4))] == [tuple(w) for w in want]
    assert np.array_equal(grp.get_coords().view(np.uint32), x_want.view(np.uint32))
    grp.close()
    with pytest.raises(G.ConfigError):
        G.Group(g, 4, 5, devices=[0, 99])
    # a failing round on one rank is raised for the whole group after every rank has been drained
    grp = G.Group(g, 4, 5, devices=[0, 0])
    x = grp.get_coords()
    x[7, 2] = np.nan
    grp.set_coords(x)
    with pytest.raises(G.DivergenceError):
        grp.iterate(1.5, 1.0, 0)
    grp.close()


def test_engine_sharded_over_a_device_list_equals_the_single_gpu_engine(G):
    """gempe_engine_create_multi (the `devices[], n_devices` constructor): embed() on three ranks == embed() on one."""
    from dataclasses import replace
    n, src, dst = er_graph(600, 3500, 9)
    g = G.Graph(n, src, dst)
    cfg = G.IterationConfig(max_iters=25, deterministic=True, relabel_period=10, batch_rounds=-1)
    one = G.embed(g, 8, cfg, 4)
    many = G.embed(g, 8, replace(cfg, devices=[0, 0, 0]), 4)
    assert many.iterations == one.iterations and many.converged == one.converged
    assert np.array_equal(many.pe_trace, one.pe_trace) and many.final_sigma == one.final_sigma
    assert np.array_equal(many.embedding.view(np.uint32), one.embedding.view(np.uint32))
    assert np.array_equal(many.last_hist_nonedge, one.last_hist_nonedge)


@pytest.mark.parametrize("case", range(16))
def test_randomized_groups_are_bit_identical_to_one_context(G, case):
    """Seeded random draws over world size (1-7 ranks), exchange path, graph shape, dimension, sampling scheme and hub
    split: three rounds of the group equal three rounds of one context bit for bit (deterministic mode)."""
    rng = np.random.default_rng(7000 + case)
    n = int(rng.choice([40, 300, 1500, 5000]))
    n, src, dst = er_graph(n, int(n * rng.choice([2, 6, 15])), int(rng.integers(1, 1000)))
    if rng.integers(0, 3) == 0:
        n, src, dst = star_plus_ring(max(n // 4, 30), hubs=int(rng.integers(1, 4)))
    dim = int(rng.choice([2, 3, 16, 64, 100, 128]))
    mode = int(rng.integers(0, 2))
    kw = dict(neg_mode=mode, negatives=int(rng.choice([1, 4, 11])) if mode else 0)
    if rng.integers(0, 2):
        kw["chunk_entries"] = int(rng.choice([8, 32]))
    world, copy_engines, seed = int(rng.integers(1, 8)), bool(rng.integers(0, 2)), int(rng.integers(1, 1 << 20))
    g = G.Graph(n, src, dst)
    want, x_want = _single_rounds(G, g, dim, seed, 3, **kw)
    grp = G.Group(g, dim, seed, devices=[0] * world, copy_engines=copy_engines, deterministic=True, **kw)
    sigma = 1.0
    for it in range(3):
        he, hn = grp.iterate(1.5, sigma, it)
        assert (he.tolist(), hn.tolist()) == want[it], (case, it)
        sigma = min(sigma * 1.4, 2.5)
    assert grp.replicas_agree()
    assert np.array_equal(grp.get_coords().view(np.uint32), x_want.view(np.uint32))
    grp.close()
