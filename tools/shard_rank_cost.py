"""Per-rank device cost of one sharded round, measured on ONE GPU: rank 0 of a `world`-rank job is stepped alone
(no kernel waits on a peer).  For the exchange path the receive side is filled from the rank's own send regions,
which have the same expected fill as a peer's.  Reports sampling / bucketing / gather time per rank; the all-gather
and all-to-all volumes are printed so the NVLink time can be added (profiles/r01_shard_rank_cost.md).

  python tools/shard_rank_cost.py --config c4 [--worlds 1,2,4,8] [--chunks 4]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_03479_b200 as G  # noqa: E402
from paper_2011_03479_b200 import graphgen  # noqa: E402
from paper_2011_03479_b200.sharded import _DeviceArray  # noqa: E402


def timed(fn, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--chunk-entries", type=int, default=0)
    ap.add_argument("--peers", action="store_true",
                    help="also time the fused update + broadcast with world-1 stand-in peer buffers in LOCAL memory "
                         "(instruction and store-issue overhead only; NVLink is not involved on one GPU)")
    args = ap.parse_args()
    n, src, dst, dim, k, _, _, _ = graphgen.make_config(args.config, device="cuda:0")
    g = G.Graph(n, src, dst)
    mode = G.NEG_PER_VERTEX_K if k else G.NEG_PER_EDGE_2
    stream = torch.cuda.Stream()
    rows = []
    for world in [int(w) for w in args.worlds.split(",")]:
        for exchange, peers in ([(0, 0)] if world == 1 else [(0, 0), (1, 0)] + ([(1, 1)] if args.peers else [])):
            chunks = 1 if (world == 1 or peers) else args.chunks
            ctx = G.Context(g, dim, 1, neg_mode=mode, negatives=k, rank=0, world=world, comm_chunks=chunks,
                            exchange=exchange, chunk_entries=args.chunk_entries)
            ctx.set_stream(stream.cuda_stream)
            ctx.init_coords(G.INIT_NORMAL, 1, 0.01)
            dummies = []
            if peers:
                for _ in range(world - 1):
                    dummies.append((torch.empty(ctx.padded_rows * ctx.row_stride, device="cuda:0"),
                                    torch.empty(ctx.padded_rows * ctx.row_stride, device="cuda:0")))
                    ctx.add_peer_pointers(dummies[-1][0].data_ptr(), dummies[-1][1].data_ptr())
            views = None
            if exchange:
                send, recv, sc, rc, cap = ctx.exchange_layout()
                t = lambda p, shape: torch.as_tensor(_DeviceArray(p, shape, "<i4"), device="cuda:0")
                views = (t(send, (world, cap, 2)), t(recv, (world, cap, 2)), t(sc, (world,)), t(rc, (world,)))
            best = None
            with torch.cuda.stream(stream):
                for it in range(args.rounds):
                    ts = timed(lambda: ctx.begin_round(1.5, 1.0, it), stream)
                    tb = 0.0
                    if exchange:
                        # every peer's region for this rank looks like this rank's own region for itself
                        for s in range(world):
                            views[1][s].copy_(views[0][0])
                        views[3].fill_(int(views[2][0]))
                        tb = timed(ctx.bucket_received, stream)
                    tg = timed(lambda: [ctx.gather_chunk(c) for c in range(chunks)], stream)
                    ctx.end_round()
                    ctx.sync()
                    cur = (ts + tb + tg, ts, tb, tg)
                    if it >= 2 and (best is None or cur[0] < best[0]):
                        best = cur
            row = dict(config=args.config, world=world, exchange=exchange, peer_stores=peers, chunks=chunks, total_ms=round(best[0], 3),
                       sample_ms=round(best[1], 3), bucket_ms=round(best[2], 3), gather_ms=round(best[3], 3),
                       allgather_bytes_per_rank=int(ctx.padded_rows * ctx.row_stride * 4 * (world - 1) / world),
                       alltoall_bytes_per_rank=int(views[0].numel() * 4 * (world - 1) / world) if exchange else 0)
            print(json.dumps(row), flush=True)
            rows.append(row)
            if peers:
                ctx.clear_peers()
            ctx.close()
            del ctx, views, dummies


if __name__ == "__main__":
    main()
