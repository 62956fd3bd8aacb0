import os, sys, time, subprocess, threading
sys.path.insert(0, "/root/repo")
import torch
import paper_2011_03479_b200 as P
from paper_2011_03479_b200 import graphgen
n, src, dst, dim, k, _, init, std = graphgen.make_config("c4", device=torch.device("cuda", 0))
ctx = P.Context(P.Graph(n, src, dst), dim, 1, neg_mode=P.NEG_PER_VERTEX_K, negatives=k)
ctx.init_coords(P.INIT_NORMAL, 1, std)
for warm in (0, 12):
    ctx.init_coords(P.INIT_NORMAL, 1, std)
    sigma = 1.0
    if warm:
        ctx.set_sigma(1.5, 1.0)
        for it in range(warm):
            sigma = ctx.iterate_auto(it)[0]
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active,temperature.gpu",
                          "--format=csv,noheader", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.5)
    for block in range(6):
        ctx.elapsed_ms()
        for it in range(100):
            ctx.iterate_async(1.5, sigma, 100 + it)
        ctx.sync()
        tot, samp, gath = ctx.elapsed_ms()
        print(f"warm {warm} block {block}: round {tot/100:.3f} sampling {samp/100:.3f} gather {gath/100:.3f}", flush=True)
    time.sleep(0.3)
    p.terminate()
    out = p.stdout.read().strip().splitlines()
    print("\n".join(out[::3]))
