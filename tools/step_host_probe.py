"""gempe_step_host on pinned against pageable host buffers (c4): what a caller with ordinary std::vector memory pays."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_03479_b200 as P
from paper_2011_03479_b200 import graphgen

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
n, src, dst, dim, k, _, init, std = graphgen.make_config(cfg, device=torch.device("cuda", 0))
ctx = P.Context(P.Graph(n, src, dst), dim, 1, neg_mode=P.NEG_PER_VERTEX_K, negatives=k)
ctx.init_coords(P.INIT_UNIFORM_PM1 if init == "uniform_pm1" else P.INIT_NORMAL, 1, std)
x0 = ctx.get_coords()
for name, make in (("pinned", lambda: torch.empty((n, dim), dtype=torch.float32, pin_memory=True).numpy()),
                   ("pageable", lambda: np.empty((n, dim), np.float32)),
                   ("page-locked through gempe_alloc_host", lambda: P.alloc_host((n, dim)))):
    a, b = make(), make()
    a[:] = x0
    b[:] = 0
    times = []
    for it in range(6):
        t = time.perf_counter()
        ctx.step_host(a, b, 1.5, 1.0, it)
        times.append(time.perf_counter() - t)
        a, b = b, a
    print(f"{cfg} {name}: " + " ".join(f"{t * 1e3:.1f}" for t in times) + " ms per step")
    if "gempe_alloc_host" in name:
        P.free_host(a)
        P.free_host(b)
