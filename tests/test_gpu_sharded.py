"""Sharded CUDA path on ONE GPU: the ranks' contexts are stepped one after another (no kernel ever waits on
another rank) and the all-gather is replaced by device copies of each owner's blocks, so the per-rank item
tables, the partner-side bucket filter (`is_local`) and the block-cyclic layout are exercised for real.
Every rank must reproduce the single-GPU context bit for bit (deterministic bucket order) and the rank
tallies must sum to the single-GPU tallies."""
import numpy as np
import pytest

from conftest import er_graph, star_plus_ring

pytestmark = pytest.mark.gpu


def _views(ctx, which):
    import torch
    from paper_2011_03479_b200.sharded import _DeviceArray
    return torch.as_tensor(_DeviceArray(ctx.device_coords(which), (ctx.padded_rows, ctx.row_stride)), device="cuda:0")


@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3), (4, 2), (8, 4)])
@pytest.mark.parametrize("mode,k,bucket_mode", [(0, 0, 1), (1, 6, 1), (1, 6, 2)])
def test_rank_contexts_reproduce_the_single_gpu_round(world, chunks, mode, k, bucket_mode):
    import torch
    import paper_2011_03479_b200 as G
    for (n, src, dst), dim in ((er_graph(1003, 6000, 3), 64), (star_plus_ring(400, hubs=2), 2)):
        g = G.Graph(n, src, dst)
        single = G.Context(g, dim, 5, neg_mode=mode, negatives=k, deterministic=True, chunk_entries=64,
                           bucket_mode=bucket_mode)
        ranks = [G.Context(g, dim, 5, neg_mode=mode, negatives=k, deterministic=True, chunk_entries=64, rank=r,
                           world=world, comm_chunks=chunks, bucket_mode=bucket_mode) for r in range(world)]
        block = ranks[0].block_rows
        assert ranks[0].padded_rows == world * chunks * block
        sigma = 1.0
        for it in range(3):
            he, hn = single.iterate(1.5, sigma, it)
            want = single.get_coords()
            tot_e, tot_n = np.zeros(512, np.uint64), np.zeros(512, np.uint64)
            for c in ranks:
                c.begin_round(1.5, sigma, it)
                for ch in range(chunks):
                    c.gather_chunk(ch)
                e, nn = c.sync()
                tot_e += e
                tot_n += nn
            assert np.array_equal(tot_e, he) and np.array_equal(tot_n, hn)
            nxt = [_views(c, 1) for c in ranks]
            for ch in range(chunks):  # the exchange: block (ch, r) travels from rank r to everybody else
                for r in range(world):
                    lo = (ch * world + r) * block
                    for other in range(world):
                        if other != r:
                            nxt[other][lo:lo + block].copy_(nxt[r][lo:lo + block])
            torch.cuda.synchronize()
            for c in ranks:
                c.end_round()
                assert np.array_equal(c.get_coords().view(np.uint32), want.view(np.uint32))
            sigma *= 1.3
        for c in ranks + [single]:
            c.close()


def _exchange_views(ctx, world):
    import torch
    from paper_2011_03479_b200.sharded import _DeviceArray
    send, recv, send_cnt, recv_cnt, cap = ctx.exchange_layout()
    t = lambda ptr, shape: torch.as_tensor(_DeviceArray(ptr, shape, "<i4"), device="cuda:0")
    return t(send, (world, cap, 2)), t(recv, (world, cap, 2)), t(send_cnt, (world,)), t(recv_cnt, (world,))


@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3), (4, 2), (8, 4)])
@pytest.mark.parametrize("mode,k", [(0, 0), (1, 6)])
def test_rank_contexts_with_sample_exchange_reproduce_the_single_gpu_round(world, chunks, mode, k):
    """opt.exchange: each rank samples only its own anchors' streams; the all-to-all is emulated by device copies
    (region d of rank s -> region s of rank d).  Coordinates bit-identical to the single context, tallies and draw
    counts sum to the single context's, and every rank does ~1/world of the sampling."""
    import torch
    import paper_2011_03479_b200 as G
    for (n, src, dst), dim in ((er_graph(1003, 6000, 3), 64), (star_plus_ring(400, hubs=2), 2)):
        g = G.Graph(n, src, dst)
        single = G.Context(g, dim, 5, neg_mode=mode, negatives=k, deterministic=True, chunk_entries=64)
        ranks = [G.Context(g, dim, 5, neg_mode=mode, negatives=k, deterministic=True, chunk_entries=64, rank=r,
                           world=world, comm_chunks=chunks, exchange=1) for r in range(world)]
        views = [_exchange_views(c, world) for c in ranks]
        block = ranks[0].block_rows
        sigma = 1.0
        for it in range(3):
            he, hn = single.iterate(1.5, sigma, it)
            want = single.get_coords()
            for c in ranks:
                c.begin_round(1.5, sigma, it)
            torch.cuda.synchronize()
            packed = 0
            for s_rank in range(world):
                packed += int(views[s_rank][2].sum())
                for d in range(world):
                    views[d][1][s_rank].copy_(views[s_rank][0][d])
                    views[d][3][s_rank] = views[s_rank][2][d]
            assert packed == single.sample_slots  # every stream sampled by exactly one rank
            torch.cuda.synchronize()
            tot_e, tot_n = np.zeros(512, np.uint64), np.zeros(512, np.uint64)
            for c in ranks:
                if it == 0 and c is ranks[0]:
                    with pytest.raises(G.ConfigError):  # packed records must be exchanged and bucketed first
                        c.gather_chunk(0)
                c.bucket_received()
                for ch in range(chunks):
                    c.gather_chunk(ch)
                e, nn = c.sync()
                tot_e += e
                tot_n += nn
            assert np.array_equal(tot_e, he) and np.array_equal(tot_n, hn)
            nxt = [_views(c, 1) for c in ranks]
            for ch in range(chunks):
                for r in range(world):
                    lo = (ch * world + r) * block
                    for other in range(world):
                        if other != r:
                            nxt[other][lo:lo + block].copy_(nxt[r][lo:lo + block])
            torch.cuda.synchronize()
            for c in ranks:
                c.end_round()
                assert np.array_equal(c.get_coords().view(np.uint32), want.view(np.uint32))
            sigma *= 1.3
        for c in ranks + [single]:
            c.close()


@pytest.mark.parametrize("world,chunks,exchange", [(2, 1, 0), (4, 1, 1), (8, 2, 1), (16, 1, 0)])
@pytest.mark.parametrize("mode,k", [(0, 0), (1, 6)])
def test_fused_update_and_broadcast_into_peer_buffers(world, chunks, exchange, mode, k):
    """Peer broadcast: the rank contexts of one process register each other's coordinate buffers (and, with the sample
    exchange on, each other's receive areas): every gather kernel stores the rows it updates into all of them and every
    pack kernel stores its records at their owners -- no copy stands in for a collective here.  Ranks are stepped one
    after another; after the last one every rank must hold the single-GPU X_{t+1} bit for bit."""
    import torch
    import paper_2011_03479_b200 as G
    for (n, src, dst), dim in ((er_graph(1003, 6000, 3), 64), (er_graph(1003, 6000, 3), 128),
                               (star_plus_ring(400, hubs=2), 2)):
        g = G.Graph(n, src, dst)
        single = G.Context(g, dim, 5, neg_mode=mode, negatives=k, deterministic=True, chunk_entries=64)
        ranks = [G.Context(g, dim, 5, neg_mode=mode, negatives=k, deterministic=True, chunk_entries=64, rank=r,
                           world=world, comm_chunks=chunks, exchange=exchange) for r in range(world)]
        for ra, a in enumerate(ranks):
            for rb, b in enumerate(ranks):
                if a is not b:
                    a.add_peer_pointers(b.device_coords_parity(0), b.device_coords_parity(1))
                    if exchange:  # direct sample exchange: the pack kernel writes into b's receive area
                        a.add_peer_exchange_pointer(rb, b.exchange_recv_area)
        sigma = 1.0
        for it in range(3):
            he, hn = single.iterate(1.5, sigma, it)
            want = single.get_coords()
            for c in ranks:
                c.begin_round(1.5, sigma, it)  # exchange: no copy stands in for an all-to-all either
            torch.cuda.synchronize()
            tot_e, tot_n = np.zeros(512, np.uint64), np.zeros(512, np.uint64)
            for c in ranks:
                assert c.coords_parity == it % 2
                if exchange:
                    c.bucket_received()
                for ch in range(chunks):
                    c.gather_chunk(ch)
                e, nn = c.sync()
                tot_e += e
                tot_n += nn
            assert np.array_equal(tot_e, he) and np.array_equal(tot_n, hn)
            for c in ranks:
                c.end_round()
                assert np.array_equal(c.get_coords().view(np.uint32), want.view(np.uint32))
            sigma *= 1.3
        for c in ranks:
            c.clear_peers()
        for c in ranks + [single]:
            c.close()


def test_exchange_and_peer_api_misuse_is_reported():
    """The sharding entry points fail loudly (config_error) when called out of order or on the wrong kind of context."""
    import paper_2011_03479_b200 as G
    n, src, dst = er_graph(500, 2000, 1)
    g = G.Graph(n, src, dst)
    plain = G.Context(g, 8, 1)
    with pytest.raises(G.ConfigError):
        plain.exchange_layout()              # no exchange buffers
    with pytest.raises(G.ConfigError):
        plain.bucket_received()              # nothing packed
    with pytest.raises(G.ConfigError):
        plain.exchange_ipc_handle()          # single rank: nothing to publish
    with pytest.raises(G.ConfigError):
        plain.add_peer_pointers(0, 0)        # null buffers
    a = G.Context(g, 8, 1, rank=0, world=2, exchange=1)
    b = G.Context(g, 8, 1, rank=1, world=2, exchange=1)
    with pytest.raises(G.ConfigError):
        a.add_peer_exchange_pointer(0, b.exchange_recv_area)   # own rank
    with pytest.raises(G.ConfigError):
        a.add_peer_exchange_pointer(2, b.exchange_recv_area)   # outside the world
    a.add_peer_exchange_pointer(1, b.exchange_recv_area)
    with pytest.raises(G.ConfigError):
        a.add_peer_exchange_pointer(1, b.exchange_recv_area)   # twice
    with pytest.raises(G.ConfigError):
        a.sample(0)                          # the hook would write into b
    a.begin_round(1.5, 1.0, 0)
    with pytest.raises(G.ConfigError):
        a.gather_chunk(0)                    # records packed but not bucketed
    with pytest.raises(G.ConfigError):
        a.gather_chunk(5)                    # no such chunk
    a.clear_peers()
    for c in (plain, a, b):
        c.close()
    with pytest.raises(G.ConfigError):
        G.Context(g, 8, 1, rank=2, world=2)  # rank outside the world
    with pytest.raises(G.ConfigError):
        G.Context(g, 8, 1, exchange=7)


def _ipc_worker(rank, world, port, exchange, results):
    """One process per rank, all on cuda:0 (time-sliced; no kernel waits on another process): gloo carries the IPC
    handles, the tallies and the barriers; the coordinates travel only through the peer stores of the gather kernel and
    (exchange) the sample records only through those of the pack kernel."""
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2011_03479_b200 as G
        from paper_2011_03479_b200 import sharded
        torch.cuda.set_device(0)
        n, src, dst = er_graph(2003, 12000, 4)
        g = G.Graph(n, src, dst)
        eng = sharded.make_cuda_engine(g, 64, 5, device=0, neg_mode=1, negatives=6, deterministic=True,
                                       exchange=exchange, peer_broadcast=True)
        assert eng.peer_broadcast and eng.chunks == 1 and eng.ops.direct_exchange == exchange
        plain = G.Context(g, 64, 5, neg_mode=1, negatives=6, deterministic=True)
        ok = True
        sigma = 1.0
        for it in range(4):
            eng.round_async(1.5, sigma, it)
            he, hn = eng.finish_round()
            he_w, hn_w = plain.iterate(1.5, sigma, it)
            ok = ok and np.array_equal(he, he_w) and np.array_equal(hn, hn_w)
            dist.barrier()
            ok = ok and np.array_equal(eng.ops.ctx.get_coords().view(np.uint32), plain.get_coords().view(np.uint32))
            dist.barrier()
            sigma *= 1.2
        eng.ops.ctx.clear_peers()
        results[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", [False, True])
def test_peer_broadcast_across_processes_over_cuda_ipc(exchange):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_ipc_worker, args=(2, port, exchange, results), nprocs=2, join=True)
    assert dict(results) == {0: True, 1: True}


@pytest.mark.parametrize("exchange", [False, True])
def test_nccl_plumbing_on_a_single_rank_group(exchange):
    """Real NCCL on one GPU: a 1-rank process group with the collectives forced on, three comm chunks.  Exercises
    the device-pointer tensor views, the in-place all_gather_into_tensor per chunk, the device-side tally all-reduce,
    the device sigma search and (exchange=True) the all_to_all_single of the packed sample records; the result must
    equal the plain engine bit for bit."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    import paper_2011_03479_b200 as G
    from paper_2011_03479_b200 import sharded
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, src, dst = er_graph(2003, 12000, 4)
        g = G.Graph(n, src, dst)
        eng = sharded.make_cuda_engine(g, 64, 5, comm_chunks=3, device=0, force_collectives=True, neg_mode=1,
                                       negatives=6, deterministic=True, exchange=exchange)
        assert eng.chunks == 3 and eng.collective
        assert (eng.ops.exchange_tensors() is not None) == exchange
        plain = G.Context(g, 64, 5, neg_mode=1, negatives=6, deterministic=True)
        plain.set_sigma(1.5, 1.0)
        for it in range(3):
            pe, sigma = eng.run_single_iteration()
            s_want, pe_want, _, _, _ = plain.iterate_auto(it)
            assert sigma == s_want and pe == pe_want
        assert np.array_equal(eng.ops.ctx.get_coords().view(np.uint32), plain.get_coords().view(np.uint32))
        # host-sigma path of the driver as well (tallies() + all_reduce + host search)
        eng.round_async(1.5, eng.sigma, eng.iter)
        he, hn = eng.finish_round()
        he_w, hn_w = plain.iterate(1.5, eng.sigma, eng.iter)
        assert np.array_equal(he, he_w) and np.array_equal(hn, hn_w)
    finally:
        dist.destroy_process_group()
