"""Vertex-sharded GEMPE rounds, one process per GPU.

Every rank holds the full X_t, CSR and edge filter; work ids (already randomly relabelled) are owned
block-cyclically -- block b of `block_rows` rows belongs to rank b % world, comm chunk b // world -- so the
updated rows of chunk c of all ranks form ONE contiguous region of X_{t+1}.  That makes the exchange an
in-place ``all_gather_into_tensor`` per chunk, issued as soon as the chunk's gather kernel is enqueued and
overlapped with the next chunk's kernel; the sampling passes of round t+1 do not read X and are enqueued
before the wait on round t's last all-gather.  Partner-side sample terms: each rank samples only the streams of
the anchors it owns, packs (partner, anchor) records by the partner's owner and the ranks swap the packed regions
with one equal-split all-to-all per round (8 bytes per sample; sampling work scales with 1/world).  With
`exchange=False` every rank instead enumerates all sample streams and keeps the partners it owns (no exchange,
replicated integer work).  The 2x512 tallies are summed with one all_reduce.

`peer_broadcast=True` removes the all-gather altogether: the ranks open each other's coordinate buffers (CUDA IPC,
peer memory over NVLink / NVSwitch) and the gather kernel stores every row it updates into all ranks' X_{t+1}
directly -- the update and its broadcast are one kernel, the transfer rides under the remaining rows' compute.
Between consecutive rounds the ranks pass a barrier (a one-element all_reduce, or the tally all_reduce).  With the
sample exchange on, the records travel the same way (the pack kernel stores them into the owners' receive areas) and
ONE barrier per round, between packing and bucketing, orders both transfers.

The collective logic is backend-agnostic (`ops` supplies the compute); tests drive it with gloo on CPU
tensors, the product with `CudaShardOps` over NCCL.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .engine import Context, Graph, optimize_sigma, histogram_objective

HIST = _capi.HIST_BINS


def block_layout(n: int, world: int, comm_chunks: int):
    """(block_rows, padded_rows) of the block-cyclic ownership map (same rule as gempe_create)."""
    blocks = world * comm_chunks
    block_rows = (max(n, 1) + blocks - 1) // blocks
    return block_rows, blocks * block_rows


def owner_of(v, block_rows: int, world: int):
    return (np.asarray(v) // block_rows) % world


class _DeviceArray:
    def __init__(self, ptr: int, shape, typestr="<f4"):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=typestr, data=(int(ptr), False), version=3)


class CudaShardOps:
    """Compute backend: the CUDA context of this rank, launching on torch's current stream."""

    def __init__(self, g: Graph, dim: int, seed: int, rank: int, world: int, comm_chunks: int, device: int, **kw):
        self.ctx = Context(g, dim, seed, rank=rank, world=world, comm_chunks=comm_chunks, device=device, **kw)
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=self.device)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.rows, self.ld = self.ctx.padded_rows, self.ctx.row_stride
        self._exchange = None
        self.direct_exchange = False  # records travel by peer stores from the pack kernel (connect_peers)
        if kw.get("exchange"):
            send, recv, send_cnt, recv_cnt, cap = self.ctx.exchange_layout()
            if recv != send:  # a single-rank context with exchange=1 is its own peer and buckets inside begin_round
                as_t = lambda ptr, shape: torch.as_tensor(_DeviceArray(ptr, shape, "<i4"), device=self.device)
                self._exchange = (as_t(send, (world, cap, 2)), as_t(recv, (world, cap, 2)),
                                  as_t(send_cnt, (world,)), as_t(recv_cnt, (world,)))

    def connect_peers(self, group=None):
        """Opens every other rank's coordinate buffers in this process (handles travel over the process group)."""
        world = dist.get_world_size(group)
        if world == 1:
            return
        me = dist.get_rank(group)
        mine = (self.ctx.coords_ipc_handles(), self.ctx.exchange_ipc_handle() if self._exchange is not None else None)
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        for r in range(world):
            if r != me:
                self.ctx.open_peer(handles[r][0])
        if self._exchange is not None and all(h[1] is not None for h in handles):
            # direct sample exchange: the pack kernel writes into the peers' receive areas, no all-to-all
            for r in range(world):
                if r != me:
                    self.ctx.open_peer_exchange(r, handles[r][1])
            self._exchange = None
            self.direct_exchange = True

    def exchange_tensors(self):
        """(send_records[world,cap,2], recv_records, send_counts[world], recv_counts) or None."""
        return self._exchange

    def bucket_received(self):
        self.ctx.bucket_received()

    def x_next(self) -> torch.Tensor:
        ptr = self.ctx.device_coords(1)
        return torch.as_tensor(_DeviceArray(ptr, (self.rows, self.ld)), device=self.device)

    def begin_round(self, mu, sigma, it):
        if mu is None:
            self.ctx.begin_round_auto(it)  # sigma lives on the device (sigma_update_kernel)
        else:
            self.ctx.begin_round(mu, sigma, it)

    def gather_chunk(self, c):
        self.ctx.gather_chunk(c)

    # device-resident sigma feedback: tallies are reduced across ranks on the device, every rank runs the same search
    def seed_sigma(self, mu, sigma):
        self.ctx.set_sigma(mu, sigma)

    def tallies_tensor(self) -> torch.Tensor:
        return torch.as_tensor(_DeviceArray(self.ctx.device_tallies(), (2 * HIST,), "<i8"), device=self.device)

    def sigma_update(self):
        self.ctx.sigma_update_async()

    def status_flags(self) -> torch.Tensor:
        """The round's status words on the device (int32[8], kernels.hpp StatusSlot), 32 bytes in front of the tallies."""
        return torch.as_tensor(_DeviceArray(self.ctx.device_tallies() - 32, (8,), "<i4"), device=self.device)

    def sigma_state(self):
        self.ctx.sync()  # raises on divergence / retry cap of the round
        return self.ctx.sigma_state()

    def end_round(self):
        self.ctx.end_round()

    def tallies(self) -> torch.Tensor:
        """int64[1024] on the compute device (edge bins then non-edge bins); synchronises the round."""
        he, hn = self.ctx.sync()
        return torch.from_numpy(np.concatenate([he, hn]).astype(np.int64)).to(self.device)


class ShardedEngine:
    """Drives rounds over a process group.  `ops` needs x_next(), begin_round, gather_chunk, end_round,
    tallies(), optionally exchange_tensors() + bucket_received(); `stream` (optional) is the CUDA stream the
    ops launch on."""

    def __init__(self, ops, n: int, m: int, world: int, rank: int, comm_chunks: int, group=None, stream=None,
                 force_collectives: bool = False, peer_broadcast: bool = False):
        self.ops, self.n, self.m, self.world, self.rank, self.chunks = ops, n, m, world, rank, comm_chunks
        self.group, self.stream = group, stream
        # True: the compute backend stores updated rows into every rank's X_{t+1} itself (peer memory); the driver
        # only separates consecutive rounds with a barrier
        self.peer_broadcast = peer_broadcast and world > 1
        self._flag = None
        # issue the collectives even for a single rank (exercises the NCCL plumbing on one GPU)
        self.collective = world > 1 or force_collectives
        self.block_rows, self.rows = block_layout(n, world, comm_chunks)
        self.mu, self.sigma, self.iter = 1.5, 1.0, 0
        self.pe_trace: List[float] = []
        self._pending = []
        self._seeded = False
        self.gather_events = None  # a list: round_async appends one CUDA event pair per gather launch (bench.py)

    def _wait_pending(self):
        for w in self._pending:
            w.wait()
        self._pending = []

    def round_async(self, mu: float, sigma: float, it: int):
        """Enqueues one round: sampling passes, then per comm chunk the gather kernel and the all-gather of
        that chunk's updated blocks.  Returns without waiting."""
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _Null()
        with ctx:
            self.ops.begin_round(mu, sigma, it)  # X-independent: overlaps the previous round's last exchange
            bufs = self.ops.exchange_tensors() if hasattr(self.ops, "exchange_tensors") else None
            if getattr(self.ops, "direct_exchange", False):
                # the pack kernel already stored the records at their owners: one barrier orders every rank's pack
                # (and its previous gather, whose peer stores filled X_t) before anybody buckets and gathers
                self._wait_pending()
                self._round_barrier(wait=True)
                self.ops.bucket_received()
            elif bufs is not None:
                # region d of every rank's send side lands in region <source rank> of rank d's receive side
                send, recv, send_cnt, recv_cnt = bufs
                dist.all_to_all_single(recv_cnt, send_cnt, group=self.group)
                dist.all_to_all_single(recv, send, group=self.group)
                self.ops.bucket_received()
            self._wait_pending()                 # X_t must be complete before the first gather reads it
            x_next = self.ops.x_next()
            span = self.world * self.block_rows
            for c in range(self.chunks):
                if self.gather_events is not None:  # bench: device time of this rank's gather launches
                    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    ev[0].record()
                    self.ops.gather_chunk(c)
                    ev[1].record()
                    self.gather_events.append(ev)
                else:
                    self.ops.gather_chunk(c)
                if self.collective and not self.peer_broadcast:
                    region = x_next[c * span:(c + 1) * span]
                    mine = region[self.rank * self.block_rows:(self.rank + 1) * self.block_rows]
                    self._pending.append(dist.all_gather_into_tensor(region, mine, group=self.group, async_op=True))
            self.ops.end_round()
            if self.peer_broadcast and not getattr(self.ops, "direct_exchange", False):
                self._round_barrier()  # with the direct exchange the barrier after the next pack does this job

    def _round_barrier(self, wait: bool = False):
        """No rank may start the next gather before every rank has finished this one (it reads what the peers wrote
        and overwrites what they were reading)."""
        if dist.get_backend(self.group) == "nccl":
            if self._flag is None:
                self._flag = torch.zeros(1, device="cuda")
            work = dist.all_reduce(self._flag, group=self.group, async_op=True)  # stream-ordered
            if wait:
                work.wait()
            else:
                self._pending.append(work)
        else:  # host-side backend (gloo): drain the stream, then meet
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)

    _FLAG_SLOTS = (0, 1, 4, 5)  # non-finite, retry cap, exchange overflow, empty tallies (not the draw counter)

    def _share_status(self):
        """A failure flag raised on one rank (divergence, retry cap, exchange overflow) is raised on all: every rank
        then throws the same error at its next status check instead of one rank leaving the others in a collective."""
        if not (self.collective and hasattr(self.ops, "status_flags")):
            return
        status = self.ops.status_flags()
        slots = torch.tensor(self._FLAG_SLOTS, device=status.device)
        flags = status[slots].clone()
        if dist.get_backend(self.group) != "nccl":
            flags = flags.cpu()
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=self.group)
        status[slots] = flags.to(status.device)

    def finish_round(self):
        """Waits for the exchange and returns the job-wide tallies (edge[512], nonedge[512])."""
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _Null()
        with ctx:
            self._wait_pending()
            self._share_status()
            t = self.ops.tallies()
            if self.collective:
                if t.is_cuda and dist.get_backend(self.group) != "nccl":
                    t = t.cpu()  # host-side backend
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        t = t.cpu().numpy().astype(np.uint64)
        return t[:HIST], t[HIST:]

    def run_single_iteration(self):
        """EmbeddingEngine::run_single_iteration across the group: every rank computes the same sigma from
        the reduced tallies (engine.cpp:293-314).  With a CUDA backend nothing but the scalar results leaves the
        device: the tallies are all-reduced in place and the sigma search runs on every rank's GPU."""
        if hasattr(self.ops, "sigma_update"):
            if not self._seeded:
                self.ops.seed_sigma(self.mu, self.sigma)
                self._seeded = True
            self.round_async(None, None, self.iter)
            ctx = torch.cuda.stream(self.stream) if self.stream is not None else _Null()
            with ctx:
                self._wait_pending()
                self._share_status()
                if self.collective:
                    dist.all_reduce(self.ops.tallies_tensor(), op=dist.ReduceOp.SUM, group=self.group)
                self.ops.sigma_update()
            self.sigma, pe, _ = self.ops.sigma_state()
            self.pe_trace.append(pe)
            self.iter += 1
            return pe, self.sigma
        self.round_async(self.mu, self.sigma, self.iter)
        he, hn = self.finish_round()
        pairs = self.n * (self.n - 1) // 2
        samples = int(hn.sum())
        weight = (pairs - self.m) / samples if samples else 1.0
        self.sigma = min(optimize_sigma(he, hn, weight, self.mu)[0], self.sigma * 1.5)
        pe = histogram_objective(he, hn, weight, self.mu, self.sigma) / pairs
        self.pe_trace.append(pe)
        self.iter += 1
        return pe, self.sigma


def replicas_agree(x: torch.Tensor, group=None) -> bool:
    """True when every rank holds bit-identical coordinates (all ranks keep the full X)."""
    h = x.contiguous().view(torch.int32).to(torch.int64)
    idx = torch.arange(h.numel(), device=h.device, dtype=torch.int64).view_as(h)
    digest = torch.stack([h.sum(), (h * (idx % 8191 + 1)).sum()])
    lo, hi = digest.clone(), digest.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return bool(torch.equal(lo, hi))


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def make_cuda_engine(g: Graph, dim: int, seed: int, *, comm_chunks: int = 4, group=None, device: Optional[int] = None,
                     force_collectives: bool = False, exchange: Optional[bool] = None, peer_broadcast: bool = False,
                     **ctx_kw) -> ShardedEngine:
    """One rank of a sharded engine over the default (NCCL) process group; world 1 without a group.
    `exchange` (default: on when collectives are in use) selects sampling of own anchors + all-to-all;
    `peer_broadcast` replaces the per-chunk all-gather by direct stores into the peers' buffers (one comm chunk)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    device = torch.cuda.current_device() if device is None else device
    chunks = comm_chunks if (world > 1 or force_collectives) else 1
    if peer_broadcast and world > 1:
        chunks = 1  # nothing to pipeline: the rows travel while the kernel runs
    if exchange is None:
        exchange = world > 1 or force_collectives
    if exchange:
        ctx_kw["exchange"] = 2 if (world == 1 and force_collectives) else 1  # 2: external exchange even for one rank
    ops = CudaShardOps(g, dim, seed, rank, world, chunks, device, **ctx_kw)
    if peer_broadcast and world > 1:
        # every rank must succeed (P2P-capable topology, IPC allowed) or none uses the path
        ok = torch.ones(1, device=ops.device)
        try:
            ops.connect_peers(group)
        except Exception:  # noqa: BLE001 - reported through the agreed flag
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() < 1:
            raise RuntimeError("peer_broadcast: a rank could not open its peers' coordinate buffers (CUDA IPC / P2P)")
    return ShardedEngine(ops, g.n, g.edge_count(), world, rank, chunks, group=group, stream=ops.stream,
                         force_collectives=force_collectives, peer_broadcast=peer_broadcast)
