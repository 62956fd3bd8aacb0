"""Small driver for ncu captures: builds a BASELINE configuration and runs a few rounds of the hot path.

    python tools/profile_round.py [--config c4] [--rounds 3] [--neg-mode per_vertex_k] [--precise]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_03479_b200 as P  # noqa: E402
from paper_2011_03479_b200 import graphgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--neg-mode", default="per_vertex_k")
ap.add_argument("--precise", action="store_true")
ap.add_argument("--chunk-entries", type=int, default=0)
ap.add_argument("--sigma", type=float, default=1.0)
ap.add_argument("--bucket-mode", type=int, default=0)
ap.add_argument("--dim", type=int, default=0, help="override the configuration's dimension")
ap.add_argument("--warm-iters", type=int, default=0, help="real iterations (device sigma feedback) before timing")
a = ap.parse_args()

import torch  # noqa: E402
if os.environ.get("GEMPE_L2_FETCH"):  # experiment: cudaLimitMaxL2FetchGranularity (0x05) on the primary context
    import ctypes
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    rt = ctypes.CDLL("libcudart.so.12")
    val = ctypes.c_size_t(0)
    rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(int(os.environ["GEMPE_L2_FETCH"])))
    rt.cudaDeviceGetLimit(ctypes.byref(val), 5)
    print("cudaLimitMaxL2FetchGranularity: set rc", rc, "now", val.value)
n, src, dst, dim, k, _, init, std = graphgen.make_config(a.config, device=torch.device('cuda', 0))
torch.cuda.empty_cache()
if a.dim:
    dim = a.dim
mode = P.NEG_PER_VERTEX_K if a.neg_mode == "per_vertex_k" else P.NEG_PER_EDGE_2
import time  # noqa: E402
_t0 = time.perf_counter()
ctx = P.Context(P.Graph(n, src, dst), dim, 1, neg_mode=mode, negatives=k if mode == P.NEG_PER_VERTEX_K else 0,
                precise_distance=a.precise, chunk_entries=a.chunk_entries, bucket_mode=a.bucket_mode)
print(f'context construction {time.perf_counter() - _t0:.2f} s (n={n}, m={len(src)})')
ctx.init_coords(P.INIT_UNIFORM_PM1 if init == "uniform_pm1" else P.INIT_NORMAL, 1, std)
sigma = a.sigma
if a.warm_iters:
    ctx.set_sigma(1.5, sigma)
    for it in range(a.warm_iters):
        sigma = ctx.iterate_auto(it)[0]
    print('sigma after warm iterations', sigma)
for it in range(2):
    ctx.iterate_async(1.5, sigma, it)
ctx.sync(); ctx.elapsed_ms()
for it in range(2, 2 + a.rounds):
    ctx.iterate_async(1.5, sigma, it)
he, hn = ctx.sync()
tot, samp, gath = ctx.elapsed_ms()
print('slot spills of the last round:', ctx.bucket_spills)
print(f"{a.config} bucket_mode {a.bucket_mode}: {a.rounds} rounds, {tot / a.rounds:.3f} ms/round (sampling passes {samp / a.rounds:.3f}, "
      f"gather {gath / a.rounds:.3f}); tallies {int(he.sum())} edges, {int(hn.sum())} samples")

if os.environ.get("GEMPE_LIVE_KERNEL_TIMES"):
    # live per-kernel durations (CUPTI through torch.profiler): warm, back to back, at the clocks of a running job --
    # unlike the ncu launch list, whose launches are serialised and start cold
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for it in range(10, 10 + a.rounds):
            ctx.iterate_async(1.5, sigma, it)
        ctx.sync()
    rows = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        r = rows.setdefault(e.name[:70], [0, 0.0])
        r[0] += 1
        r[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    print("live kernel times (us per round):")
    for name, (cnt, us) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
        print(f"  {us / a.rounds:12.1f}  x{cnt / a.rounds:5.1f}  {name}")
