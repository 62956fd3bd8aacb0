"""World-size-2 (and 3) CPU test of the sharded round driver (paper_2011_03479_b200/sharded.py) over gloo.

The collective logic -- block-cyclic ownership, one in-place all_gather_into_tensor per comm chunk, the tally
all_reduce, the all-to-all of the packed sample records, the host sigma update on every rank -- is backend-agnostic; here the per-rank compute is supplied
by the CPU oracle (test infrastructure) instead of the CUDA context, and every rank must end each round with
exactly the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import er_graph


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleShardOps:
    """Computes this rank's owned blocks with the CPU oracle; rows it does not own are poisoned with NaN so the
    test fails unless the all-gather delivers them."""

    def __init__(self, oracle, fm, n, ws, wd, x0, seed, rank, world, chunks, exchange=False):
        from paper_2011_03479_b200.sharded import block_layout
        self.o, self.fm, self.n, self.ws, self.wd, self.seed = oracle, fm, n, ws, wd, seed
        self.rank, self.world, self.chunks = rank, world, chunks
        self.block_rows, self.rows = block_layout(n, world, chunks)
        self.dim = x0.shape[1]
        self.x = [torch.zeros(self.rows, self.dim), torch.zeros(self.rows, self.dim)]
        self.x[0][:n] = torch.from_numpy(x0)
        self.cur = 0
        self.table = oracle.hash_build(n, ws, wd)
        self.exchange, self.exchange_ok = exchange, True

    def x_next(self):
        return self.x[self.cur ^ 1]

    def begin_round(self, mu, sigma, it):
        x = self.x[self.cur][:self.n].numpy().copy()
        self.out = self.o.iterate(self.n, self.ws, self.wd, x, 0, 0, self.seed, it, mu, sigma, self.fm, self.table)
        self.x_next().fill_(float("nan"))

    # sample exchange (opt.exchange of the CUDA context): own anchors' samples packed by the partner's owner
    def exchange_tensors(self):
        if not self.exchange:
            return None
        from paper_2011_03479_b200.sharded import owner_of
        p = self.out["partners"].astype(np.int64)
        anchors = np.stack([self.ws, self.wd], 1).ravel().astype(np.int64)  # slot 2e + role
        mine = owner_of(anchors, self.block_rows, self.world) == self.rank
        dest = owner_of(p, self.block_rows, self.world)
        cap = len(p) + 1
        self.send = torch.full((self.world, cap, 2), -1, dtype=torch.int32)
        self.send_cnt = torch.zeros(self.world, dtype=torch.int32)
        for d in range(self.world):
            sel = mine & (dest == d)
            k = int(sel.sum())
            self.send[d, :k, 0] = torch.from_numpy(p[sel].astype(np.int32))
            self.send[d, :k, 1] = torch.from_numpy(anchors[sel].astype(np.int32))
            self.send_cnt[d] = k
        self.recv = torch.full((self.world, cap, 2), -7, dtype=torch.int32)
        self.recv_cnt = torch.zeros(self.world, dtype=torch.int32)
        self.expected = sorted(zip(p[dest == self.rank].tolist(), anchors[dest == self.rank].tolist()))
        return self.send, self.recv, self.send_cnt, self.recv_cnt

    def bucket_received(self):
        got = []
        for s in range(self.world):
            k = int(self.recv_cnt[s])
            got += [tuple(r) for r in self.recv[s, :k].tolist()]
        # exactly the samples whose partner this rank owns, each once
        self.exchange_ok = self.exchange_ok and sorted(got) == self.expected

    def gather_chunk(self, c):
        b = c * self.world + self.rank
        lo, hi = min(self.n, b * self.block_rows), min(self.n, (b + 1) * self.block_rows)
        self.x_next()[lo:hi] = torch.from_numpy(self.out["x_next"][lo:hi])
        self.x_next()[max(lo, self.n):(b + 1) * self.block_rows] = 0.0  # padding rows of an owned block

    def end_round(self):
        self.cur ^= 1

    def tallies(self):
        # every pair is tallied by exactly one rank: edges at the owner of min(u,v), samples at the owner of the anchor
        from paper_2011_03479_b200.sharded import owner_of
        x = self.x[self.cur ^ 1 if False else self.cur]  # noqa: F841 (state already swapped; tallies come from self.out)
        he = np.zeros(512, np.int64)
        hn = np.zeros(512, np.int64)
        if self.rank == 0:
            he += self.out["hist_edge"].astype(np.int64)
            hn += self.out["hist_nonedge"].astype(np.int64)
        return torch.from_numpy(np.concatenate([he, hn]))


def _worker(rank, world, port, chunks, exchange, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from conftest import load_golden
        from paper_2011_03479_b200.sharded import ShardedEngine
        orc = O.Oracle()
        t = load_golden("numerics.json")["tables"]
        fm = O.fastmath_from_flat([float(v) for v in t["erf"]["flat"]], [float(v) for v in t["ratio"]["flat"]])
        n, src, dst = er_graph(203, 700, 5)  # n not divisible by world*chunks: exercises the padded tail
        seed = 9
        fwd = orc.random_relabel(n, orc.lib.go_mix_seed(seed, 0xA11BE11))
        ws, wd = fwd[src], fwd[dst]
        x0 = orc.init_embedding(n, 3, seed)
        ops = OracleShardOps(orc, fm, n, ws, wd, x0, seed, rank, world, chunks, exchange)
        eng = ShardedEngine(ops, n, len(ws), world, rank, chunks)
        trace = []
        for _ in range(3):
            pe, sigma = eng.run_single_iteration()
            trace.append((pe, sigma))
        x_final = ops.x[ops.cur][:n].numpy().copy()
        # single-process truth
        x, sigma, table = x0, 1.0, orc.hash_build(n, ws, wd)
        want = []
        for it in range(3):
            out = orc.iterate(n, ws, wd, x, 0, 0, seed, it, 1.5, sigma, fm, table)
            pairs = n * (n - 1) // 2
            nw = (pairs - len(ws)) / out["hist_nonedge"].sum()
            sigma = min(orc.optimize_sigma(out["hist_edge"], out["hist_nonedge"], nw, 1.5)[0], sigma * 1.5)
            want.append((orc.lib.go_histogram_objective(out["hist_edge"], out["hist_nonedge"], nw, 1.5, sigma) / pairs,
                         sigma))
            x = out["x_next"]
        ok = np.array_equal(x_final, x) and not np.isnan(x_final).any()
        ok = ok and all(abs(a[0] - b[0]) <= 1e-12 * abs(b[0]) and a[1] == b[1] for a, b in zip(trace, want))
        results[rank] = bool(ok and ops.exchange_ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,exchange", [(2, 1, False), (2, 3, True), (3, 2, True)])
def test_sharded_rounds_match_single_process(world, chunks, exchange):
    from paper_2011_03479_b200 import _capi
    _capi.load()  # build once in the parent, not in every rank
    import oracle as O
    O.Oracle()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), chunks, exchange, results), nprocs=world, join=True)
    assert dict(results) == {r: True for r in range(world)}


def test_block_cyclic_layout_is_a_partition():
    from paper_2011_03479_b200.sharded import block_layout, owner_of
    for n, world, chunks in [(1, 1, 1), (10, 2, 3), (203, 3, 2), (1 << 20, 8, 4), (1000, 8, 16)]:
        block_rows, rows = block_layout(n, world, chunks)
        assert rows >= n and rows == world * chunks * block_rows
        own = owner_of(np.arange(n), block_rows, world)
        assert own.min() >= 0 and own.max() < world
        # contiguity of each comm chunk: chunk c of all ranks is the row range [c*world*block_rows, (c+1)*...)
        for c in range(chunks):
            lo, hi = c * world * block_rows, min(n, (c + 1) * world * block_rows)
            if lo < hi:
                seg = own[lo:hi]
                assert (np.diff(seg) >= 0).all()  # rank 0 block, then rank 1 block, ...
