"""Experiment: do the sampling passes of round t+1 hide beside the gather of round t?  Two contexts on one device (the
sampling passes need neither X nor sigma), each on its own stream: A runs whole rounds, B runs sampling passes only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_03479_b200 as P  # noqa: E402
from paper_2011_03479_b200 import graphgen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
R = 20
n, src, dst, dim, k, _, init, std = graphgen.make_config(cfg, device=torch.device("cuda", 0))
g = P.Graph(n, src, dst)
A = P.Context(g, dim, 1, neg_mode=P.NEG_PER_VERTEX_K, negatives=k)
B = P.Context(g, dim, 1, neg_mode=P.NEG_PER_VERTEX_K, negatives=k)
A.init_coords(P.INIT_UNIFORM_PM1 if init == "uniform_pm1" else P.INIT_NORMAL, 1, std)


def wall(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3 / R


def rounds_a():
    for it in range(R):
        A.iterate_async(1.5, 1.0, it)


def passes_b():
    for it in range(R):
        B.begin_round(1.5, 1.0, it)


def both():
    for it in range(R):
        A.iterate_async(1.5, 1.0, it)
        B.begin_round(1.5, 1.0, it + 1)


for name, fn in (("warm", both), ("A rounds alone", rounds_a), ("B sampling passes alone", passes_b), ("A and B together", both),
                 ("A rounds alone", rounds_a), ("A and B together", both)):
    print(f"{cfg} {name}: {wall(fn):.3f} ms per round")
    A.sync()
    A.elapsed_ms()
