#!/usr/bin/env python
"""Benchmark of the GEMPE round (BASELINE.json metric: edge+negative gradient terms per second per iteration,
and the fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

A "step" is one GEMPE iteration (sampling passes + gradient gather + update) over the synthetic graph of the
chosen BASELINE configuration (default c4: R-MAT scale 20, d=128, 20 negatives per vertex).  One JSON line is
printed by rank 0.  Besides the contract keys the N=1 line carries
  roofline        the gather kernel timed live (CUDA events); `frac` on ncu-measured DRAM bytes of THIS build
                  (profiles/traffic.json, keyed by a hash of the kernel sources -- null when the sources changed since),
                  `frac_algorithmic` on SURVEY 8(d)'s formula, both also for the whole step
  per_edge_2      the same graph with the REFERENCE's sampling scheme (2 negatives per edge): the like-for-like
                  partner of `--impl reference`
  largest_config  BASELINE config 5 (R-MAT scale 24, the largest single-GPU configuration), device-timed
  e2e, full_iteration, cuda_graph (small graphs), cpu_baseline.
`--impl reference` times the reference's own CPU engine (oracle/_ref, unmodified) on the host cores, on the FULL
edge list of the same graph snapshot.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pair_terms_per_second"
UNIT = "pair-terms/s"
KERNEL_SOURCES = ["kernels.cu", "kernels.hpp", "device_fns.cuh"]  # what the device code is compiled from


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--neg-mode", default="per_vertex_k", choices=["per_vertex_k", "per_edge_2"])
    p.add_argument("--comm-chunks", type=int, default=4)
    p.add_argument("--chunk-entries", type=int, default=0)
    p.add_argument("--bucket-mode", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-seconds", type=float, default=None,
                   help="CPU budget on rank 0 for the cpu_baseline leg of the GPU arm (default 30 s)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sub-records", action="store_true", help="skip per_edge_2 and largest_config")
    p.add_argument("--largest-cpu-baseline", action="store_true",
                   help="time the CPU reference on config 5 inside the largest_config record (adds ~3 minutes)")
    p.add_argument("--peer-broadcast", default="auto", choices=["auto", "off"],
                   help="N > 1: gather kernel stores updated rows into the peers' buffers (auto) or NCCL all-gather (off)")
    return p.parse_args()


def workload_name(cfg):
    return {"c1": "SBM n=3000 6 blocks d=2 k=5", "c2": "Barabasi-Albert n=1e5 m=8 d=2 k=10",
            "c3": "Dirichlet-SBM n=2e5 deg20 d=64 k=10", "c4": "R-MAT scale 20 ef16 d=128 k=20",
            "c5": "R-MAT scale 24 ef16 d=128 k=20"}[cfg]


def config_record(cfg, n, m, dim):
    """The SAME dictionary in both arms: what the workload is, nothing about how an arm runs it."""
    return {"workload": workload_name(cfg), "n": int(n), "m": int(m), "dim": int(dim),
            "graph": "full edge list of the seeded synthetic snapshot (graphgen.make_config)",
            "pair_term": "one processed edge or one accepted negative sample, both endpoints updated"}


def kernel_source_hash():
    h = hashlib.sha256()
    for name in KERNEL_SOURCES:
        with open(os.path.join(ROOT, "paper_2011_03479_b200", "csrc", name), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def measured_traffic(cfg, neg_mode="per_vertex_k"):
    """ncu DRAM bytes per gather launch for `cfg`, only when measured on the kernel sources of this checkout."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return None, "profiles/traffic.json missing"
    if t.get("kernel_source_hash") != kernel_source_hash():
        return None, "profiles/traffic.json was measured on other kernel sources (hash %s, now %s)" % (
            t.get("kernel_source_hash"), kernel_source_hash())
    rec = t.get(cfg if neg_mode == "per_vertex_k" else cfg + "_per_edge_2")
    return (rec, t.get("source", "ncu")) if rec else (None, "no ncu capture for this configuration")


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons (NVML when importable, else nvidia-smi) with a timestamp per sample."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.index, self.rows, self._halt = index, [], threading.Event()
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index(index))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.bits = [(pynvml.nvmlClocksThrottleReasonHwSlowdown, "hw_slowdown"),
                         (pynvml.nvmlClocksThrottleReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                         (pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                         (pynvml.nvmlClocksThrottleReasonSwPowerCap, "sw_power_cap")]
        except Exception:
            self.nvml = None

    @staticmethod
    def _physical_index(index: int) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v for v in vis.split(",") if v.strip()]
        return int(ids[index]) if ids and index < len(ids) and ids[index].strip().isdigit() else index

    def run(self):
        while not self._halt.is_set():
            try:
                if self.nvml:
                    mhz = self.nvml.nvmlDeviceGetClockInfo(self.handle, self.nvml.NVML_CLOCK_SM)
                    mask = self.nvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
                    self.rows.append((time.perf_counter(), int(mhz), int(self.max_mhz),
                                      [name for bit, name in self.bits if mask & bit]))
                else:
                    out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i",
                                          str(self.index)], capture_output=True, text=True, timeout=5).stdout.strip()
                    c = [v.strip() for v in out.split(",")]
                    if len(c) >= 6 and c[0].isdigit():
                        self.rows.append((time.perf_counter(), int(c[0]), int(c[1]) if c[1].isdigit() else 0,
                                          [n for n, v in zip(self.NAMES, c[2:6]) if v.lower().startswith("active")]))
            except Exception:
                pass
            self._halt.wait(0.002 if self.nvml else 0.2)

    def finish(self, t0=None, t1=None):
        """Summary over the whole sampling window; `samples_in_timed_region` counts those inside [t0, t1]."""
        self._halt.set()
        self.join(timeout=6)
        sm = sorted(r[1] for r in self.rows)
        inside = [r for r in self.rows if t0 is not None and t0 <= r[0] <= t1]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max((r[2] for r in self.rows), default=None),
                "reasons": sorted({n for r in self.rows for n in r[3]}), "samples": len(self.rows),
                "samples_in_timed_region": len(inside),
                "window": "the timed steps and the same steps continued untimed until >= 0.5 s of load was sampled",
                "source": "nvml" if self.nvml else "nvidia-smi"}


def host_memory_available():
    try:
        return int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) * 1024
    except Exception:
        return 32 << 30


def cpu_reference_arm(n, src, dst, dim, steps, warmup, budget_s=None):
    """EmbeddingEngine::run_single_iteration of the UNMODIFIED reference (oracle/_ref) on the host cores, on the FULL
    edge list (the reference's own 2-draws-per-edge sampling: pair-terms = 3 m per round).  `budget_s` (the GPU arm's
    cpu_baseline leg) bounds the number of timed rounds, never the graph."""
    import oracle as O
    ref = O.Ref()
    cores = os.cpu_count() or 1
    lanes = 16 if dim <= 8 else 1
    # accumulator bank = workers * lanes * n * (d+1) * 4 bytes (engine.cpp:77-86), hash table up to 2 GiB
    avail = host_memory_available()
    table = min(1 << 31, 1 << max(6, int(np.ceil(np.log2(64.0 * max(1, len(src)))))))
    per_worker = lanes * n * (dim + 1) * 4
    workers = int(min(cores, (0.6 * avail - table - 16 * len(src)) // max(1, per_worker)))
    m = int(len(src))
    if workers < 1:
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "host_cores": cores,
                "sample": "DNF (memory): one accumulator replica is %.1f GB + a %.1f GB edge table, %.1f GB available"
                          % (per_worker / 1e9, table / 1e9, avail / 1e9)}
    t0 = time.perf_counter()
    eng = O.RefEngine(ref, n, src, dst, dim, 1, lane_width=lanes, workers=workers)
    eng.set_capture(False)
    t_build = time.perf_counter() - t0
    times = []

    def one():
        t = time.perf_counter()
        eng.iterate(capture=False)
        times.append(time.perf_counter() - t)

    one()  # first round: also the probe for the budget
    if budget_s is not None:
        # the reference's first three rounds are ~12 % slower than the ones after them (c4: 2.75 s, then 2.45 s): three
        # warm-up rounds when the budget holds them plus three timed ones, else one
        afford = int((budget_s - t_build - times[0]) // max(times[0], 1e-9))
        warmup = 3 if afford >= 5 else 1
        steps = int(max(1, min(steps, afford - (warmup - 1))))
    if steps * times[0] > 1500.0:  # the driver's limit is 1800 s: never fewer than 3 timed rounds, never the whole hour
        steps = max(3, int(1500.0 // times[0]))
    for _ in range(max(0, warmup - 1)):
        one()
    timed = []
    for _ in range(steps):
        one()
        timed.append(times[-1])
    sec = float(np.median(timed))
    return {"value": 3.0 * m / sec, "unit": UNIT, "cores": workers, "kind": "reference",
            "sample": f"full edge list ({m} edges, {n} vertices), reference sampling (2 draws/edge, 3m = {3 * m} pair-terms "
                      f"per round), lane_width={lanes}, workers={workers}, {len(timed)} timed rounds after {max(1, warmup)} "
                      f"warm-up, median {sec:.3f} s/round (engine construction {t_build:.1f} s, not timed)",
            "host_cores": cores, "sample_ms_per_round": sec * 1e3, "timed_rounds": len(timed), "construction_s": t_build,
            "round_seconds": [round(t, 4) for t in times]}  # every round in order, warm-up included


def embed_call_record(P, n, src, dst, dim, iterations):
    """The reference's public entry point, `embed(g, dim, cfg, seed)` (engine.hpp:170-171), as a user calls it: HOST edge
    arrays in, `iterations` whole iterations (the reference's 2-per-edge sampling, sigma feedback, PE trace, best-PE
    snapshot), HOST embedding out.  Upload, relabel, CSR / hash-set construction, the run and the download are all inside
    the timed region.  A convergence window longer than the run keeps it from stopping early."""
    src_h = np.ascontiguousarray(src.cpu().numpy() if hasattr(src, "cpu") else src, dtype=np.uint32)
    dst_h = np.ascontiguousarray(dst.cpu().numpy() if hasattr(dst, "cpu") else dst, dtype=np.uint32)
    cfg = P.IterationConfig(max_iters=iterations, convergence_window=iterations + 1)
    out = []
    for _ in range(4):  # the first call pays lazy CUDA module loading and is dropped; the median of the other three is reported
        t0 = time.perf_counter()
        res = P.embed(P.Graph(n, src_h, dst_h), dim, cfg, 1)
        out.append((time.perf_counter() - t0, res.iterations))
        if not np.isfinite(res.embedding).all():
            raise RuntimeError("embed() returned non-finite coordinates")
        del res
    calls = sorted(t for t, _ in out[1:])
    sec, iters = calls[len(calls) // 2], out[-1][1]
    m = int(len(src_h))
    return {"iterations": int(iters), "seconds": sec, "seconds_all_calls": [t for t, _ in out],
            "value": 3.0 * m * iters / sec, "unit": UNIT, "h2d_bytes": int(2 * 4 * m), "d2h_bytes": int(4 * n * dim),
            "what": "embed(g, dim, cfg, seed) with host edge arrays in and the host embedding out: construction + "
                    f"{iters} iterations (2 negatives per edge, 3m pair-terms each) + download, wall clock of the call"}


# ---------------------------------------------------------------------------------------------- one GPU, one context

def time_steps(torch, ctx, stream, mu, sigma, first_iter, steps):
    """K rounds back to back on `stream`, device-timed.  Returns (ms, wall t0, wall t1)."""
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ev0.record(stream)
    for s in range(steps):
        ctx.iterate_async(mu, sigma, first_iter + s)
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1), w0, time.perf_counter()


def roofline_record(ctx, cfg, neg_mode, gather_ms, step_ms, peaks):
    """HBM roofline of the gather kernel (and of the whole step) from times measured in this run."""
    _, draws = ctx.sample(1 << 20)  # p-bar: LCG draws per accepted sample (any round index)
    p_bar = draws / max(1, ctx.sample_slots)
    b_alg = ctx.algorithmic_bytes + int((p_bar - 1.0) * ctx.sample_slots)
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic, traffic_source = measured_traffic(cfg, neg_mode)
    gs, ss = gather_ms * 1e-3, step_ms * 1e-3
    alg = b_alg / gs / 1e9
    rec = {"bound": "hbm", "peak": peak, "unit": "GB/s", "kernel": "gather_batched_kernel", "kernel_ms": gather_ms,
           "algorithmic_bytes": int(b_alg), "achieved_algorithmic": alg, "frac_algorithmic": alg / peak,
           "step_frac_algorithmic": b_alg / ss / 1e9 / peak, "draws_per_sample": p_bar,
           "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if peaks else "fallback 6650 GB/s",
           "traffic_source": traffic_source}
    if traffic:
        dram = float(traffic["gather_dram_bytes"])
        rec.update({"traffic": int(dram), "achieved": dram / gs / 1e9, "frac": dram / gs / 1e9 / peak,
                    "frac_basis": "ncu dram__bytes_read + dram__bytes_write of one gather launch of this build / live kernel time",
                    "l2_hit_rate_pct": traffic.get("gather_l2_hit_pct"),
                    "step_traffic": int(traffic.get("step_dram_bytes", 0)) or None,
                    "step_frac": (float(traffic["step_dram_bytes"]) / ss / 1e9 / peak) if traffic.get("step_dram_bytes") else None})
    else:  # no DRAM byte count for this build: the algorithmic figure stands in and says so
        rec.update({"traffic": None, "achieved": alg, "frac": alg / peak,
                    "frac_basis": "ALGORITHMIC bytes (counts L2-served hub rows as HBM traffic: can exceed 1)"})
    return rec


def single_context_record(torch, P, g, cfg, dim, k, init, std, neg_mode, steps, warmup, stream_owner=None, e2e_steps=0,
                          sampler_index=None, bucket_mode=0, chunk_entries=0, peaks=None):
    """Builds a context for (graph, sampling scheme), warms it up with real iterations (device sigma search) and times
    `steps` rounds.  Returns (record, ctx, mu, sigma, next_iter)."""
    mode = P.NEG_PER_VERTEX_K if neg_mode == "per_vertex_k" else P.NEG_PER_EDGE_2
    t0 = time.perf_counter()
    ctx = P.Context(g, dim, 1, neg_mode=mode, negatives=k if mode == P.NEG_PER_VERTEX_K else 0, bucket_mode=bucket_mode,
                    chunk_entries=chunk_entries)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.init_coords(P.INIT_UNIFORM_PM1 if init == "uniform_pm1" else P.INIT_NORMAL, 1, std)
    mu, sigma = 1.5, 1.0
    ctx.set_sigma(mu, sigma)
    it = 0
    for _ in range(max(warmup, 3)):
        sigma = ctx.iterate_auto(it)[0]
        it += 1
    ctx.elapsed_ms()
    sampler = ClockSampler(sampler_index) if sampler_index is not None else None
    launches0 = ctx.kernel_launches
    if sampler:
        sampler.start()
    ms, w0, w1 = time_steps(torch, ctx, stream, mu, sigma, it, steps)
    launches = ctx.kernel_launches - launches0
    tot, samp_ms, gath_ms = ctx.elapsed_ms()
    it += steps
    clocks = None
    if sampler:  # the timed region is ~0.1 s: keep the same load running (untimed) until the sampler has seen >= 0.5 s
        t_end = time.perf_counter() + max(0.0, 0.5 - (w1 - w0))
        while time.perf_counter() < t_end:
            for s in range(4):
                ctx.iterate_async(mu, sigma, it + s)
            torch.cuda.synchronize()
        ctx.elapsed_ms()
        clocks = sampler.finish(w0, w1)
    ctx.sync()  # status check of the last timed round (raises on divergence / retry cap)
    step_ms = ms / steps
    rec = {"value": ctx.pair_terms / (step_ms * 1e-3), "unit": UNIT, "ms_per_step": step_ms, "steps": steps,
           "pair_terms_per_iteration": int(ctx.pair_terms), "sigma": sigma, "gpu_launches": int(launches),
           "sampling": "k=%d negatives per vertex (S = n k)" % k if mode == P.NEG_PER_VERTEX_K
                       else "2 negatives per edge (S = 2 m), the reference's scheme (engine.cpp:227-249)",
           "sampling_passes_ms": samp_ms / steps, "context_construction_s": build_s,
           "roofline": roofline_record(ctx, cfg, neg_mode, gath_ms / steps, step_ms, peaks or {})}
    if clocks:
        rec["clocks"] = clocks
    if e2e_steps:
        rec["e2e"] = e2e_record(torch, ctx, g.n, dim, mu, sigma, it + 100, e2e_steps)
    return rec, ctx, stream, mu, sigma, it


def e2e_record(torch, ctx, n, dim, mu, sigma, first_iter, steps):
    """The round through the C-ABI with HOST buffers: X_t in (pinned), round, X_{t+1} + tallies out."""
    bufs = [torch.empty((n, dim), dtype=torch.float32, pin_memory=True).numpy() for _ in range(2)]
    ctx.get_coords(bufs[0])
    t = []
    for s in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.step_host(bufs[s % 2], bufs[(s + 1) % 2], mu, sigma, first_iter + s)
        t.append(time.perf_counter() - t0)
    sec = float(np.median(t[1:]))
    return {"value": ctx.pair_terms / sec, "unit": UNIT, "h2d_bytes_per_step": int(n * dim * 4),
            "d2h_bytes_per_step": int(n * dim * 4 + 2 * 512 * 8), "ms_per_step": sec * 1e3,
            "call": "gempe_step_host: X_t in, round, X_{t+1} + tallies out (pinned host buffers, copies overlapped)"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2011_03479_b200 import graphgen

    def gen_device():
        """torch CUDA device for the R-MAT generator when a GPU is present (same graph as the numpy path)."""
        try:
            import torch
            return torch.device("cuda", local_rank) if torch.cuda.is_available() else None
        except Exception:
            return None

    if args.impl == "reference":
        if rank != 0:
            return
        n, src, dst, dim, k, _, _, _ = graphgen.make_config(args.config, device=gen_device())
        base = cpu_reference_arm(n, src, dst, dim, steps=args.steps, warmup=max(1, args.warmup))
        line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": base.get("sample_ms_per_round"),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": config_record(args.config, n, len(src), dim),
                "sampling": "2 negatives per edge (S = 2 m), the reference's only scheme (engine.cpp:227-249)",
                "pair_terms_per_iteration": 3 * int(len(src)), "cpu_baseline": base,
                "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    import paper_2011_03479_b200 as P
    from paper_2011_03479_b200 import sharded

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass

    # test hook: GEMPE_BENCH_TEST_BACKEND=gloo runs the N > 1 control flow with every rank time-sliced on cuda:0 (no
    # kernel waits on another rank; sample exchange off because gloo has no CUDA all-to-all) -- never a bench number
    test_backend = os.environ.get("GEMPE_BENCH_TEST_BACKEND")
    if test_backend:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        # leave NCCL's communicator-setup lines ("... nranks N ...") in the log of a multi-GPU run; on stderr, so that
        # stdout stays the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if test_backend:
            dist.init_process_group(test_backend)
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    n, src, dst, dim, k, _, init, std = graphgen.make_config(args.config, device=gen_device())
    torch.cuda.empty_cache()
    g = P.Graph(n, src, dst)
    warmup = max(args.warmup, 3)
    base_line = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": warmup,
                 "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                 "config": config_record(args.config, n, len(src), dim)}

    if world == 1:
        rec, ctx, stream, mu, sigma, it = single_context_record(
            torch, P, g, args.config, dim, k, init, std, args.neg_mode, args.steps, warmup, e2e_steps=max(1, args.e2e_steps),
            sampler_index=local_rank, bucket_mode=args.bucket_mode, chunk_entries=args.chunk_entries, peaks=peaks)
        line = dict(base_line)
        line.update({"value": rec["value"], "ms_per_step": rec["ms_per_step"], "sampling": rec["sampling"],
                     "pair_terms_per_iteration": rec["pair_terms_per_iteration"], "sigma": rec["sigma"],
                     "l2": "inputs larger than L2 (X %.0f MB + lists)" % (n * dim * 4 / 1e6) if n * dim * 4 > 126e6
                           else "working set fits L2 (reported as is)",
                     "parallelism": "1 GPU", "clocks": rec["clocks"], "gpu_launches": rec["gpu_launches"],
                     "roofline": rec["roofline"], "sampling_passes_ms": rec["sampling_passes_ms"], "e2e": rec["e2e"]})

        # whole iterations with the device-resident sigma feedback (round + sigma search + PE estimate, no host sync)
        ctx.set_sigma(mu, sigma)
        for s in range(3):
            ctx.iterate_auto_async(it + 200 + s)
        torch.cuda.synchronize()
        fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fe0.record(stream)
        for s in range(args.steps):
            ctx.iterate_auto_async(it + 203 + s)
        fe1.record(stream)
        torch.cuda.synchronize()
        ctx.sync()
        full_ms = fe0.elapsed_time(fe1) / args.steps
        line["full_iteration"] = {"ms_per_step": full_ms, "value": ctx.pair_terms / (full_ms * 1e-3), "unit": UNIT,
                                  "what": "round + device sigma search + PE estimate (run_single_iteration), no host sync"}
        ctx.elapsed_ms()

        # small graphs: the same rounds as one CUDA graph of 50, gaps between the ~5 kernels removed
        if rec["ms_per_step"] < 1.0:
            reps = 50
            ctx.graph_capture(mu, sigma, it + 300, reps)
            ctx.graph_launch()
            torch.cuda.synchronize()
            ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ge0.record(stream)
            ctx.graph_launch()
            ge1.record(stream)
            torch.cuda.synchronize()
            ctx.sync()
            g_ms = ge0.elapsed_time(ge1) / reps
            line["cuda_graph"] = {"rounds_per_graph": reps, "ms_per_step": g_ms, "value": ctx.pair_terms / (g_ms * 1e-3),
                                  "unit": UNIT, "what": "50 rounds captured into one CUDA graph, one launch"}
            ctx.elapsed_ms()
            # ... and WHOLE iterations (round + sigma search + PE trace / best-PE / convergence bookkeeping on the device)
            # replayed the same way: what gempe_engine_run queues per host round trip
            ctx.run_begin(mu, sigma, it + 400, window=1 << 20, tol=0.0, max_rounds=4 * reps)
            ctx.run_enqueue(reps, reps, True)
            ctx.run_poll()
            ge0.record(stream)
            ctx.run_enqueue(reps, 2 * reps, True)
            ge1.record(stream)
            torch.cuda.synchronize()
            st = ctx.run_poll()
            assert st["rounds_done"] == 2 * reps
            r_ms = ge0.elapsed_time(ge1) / reps
            line["full_iteration_graph"] = {"rounds_per_graph": reps, "ms_per_step": r_ms,
                                            "value": ctx.pair_terms / (r_ms * 1e-3), "unit": UNIT,
                                            "what": "50 whole iterations (sigma feedback, PE trace, best-PE snapshot, convergence "
                                                    "window on the device) as one CUDA graph launch"}
        ctx.close()
        del ctx

        if not args.no_sub_records and args.neg_mode == "per_vertex_k":
            # the same graph with the reference's own sampling scheme: like-for-like with `--impl reference`
            sub, sctx, *_ = single_context_record(torch, P, g, args.config, dim, k, init, std, "per_edge_2", args.steps,
                                                  warmup, e2e_steps=max(1, args.e2e_steps), peaks=peaks)
            sctx.close()
            del sctx
            line["per_edge_2"] = sub
        if not args.no_sub_records:
            try:
                line["embed_call"] = embed_call_record(P, n, src, dst, dim, 20)
            except Exception as e:  # noqa: BLE001
                line["embed_call"] = {"unavailable": str(e)[:300]}
        if not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_reference_arm(n, src, dst, dim, steps=3, warmup=1,
                                                         budget_s=args.cpu_seconds or 30.0)
            except Exception as e:  # the reference build is test infrastructure; its absence is reported, not fatal
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
        cb, call = line.get("cpu_baseline") or {}, line.get("embed_call") or {}
        if call.get("seconds") and cb.get("value") and cb.get("construction_s") is not None:
            # the same call on the reference, from ITS construction time and median round measured above on this host
            call["reference_seconds"] = cb["construction_s"] + call["iterations"] * cb["sample_ms_per_round"] * 1e-3
            call["reference_basis"] = "engine construction + iterations x median round of the cpu_baseline leg of this run"
        if not args.no_sub_records and args.config == "c4" and torch.cuda.mem_get_info()[1] > 150e9:
            # BASELINE config 5, the largest configuration that fits one GPU (~30 GB): device-timed here so that the
            # number is produced by the same run as the headline
            try:
                del g
                n5, s5, d5, dim5, k5, _, init5, std5 = graphgen.make_config("c5", device=gen_device())
                torch.cuda.empty_cache()
                g5 = P.Graph(n5, s5, d5)
                big, bctx, *_ = single_context_record(torch, P, g5, "c5", dim5, k5, init5, std5, "per_vertex_k",
                                                      min(args.steps, 5), 3, sampler_index=local_rank, peaks=peaks)
                bctx.close()
                big["config"] = config_record("c5", n5, len(s5), dim5)
                if args.largest_cpu_baseline:  # one round of the reference on c5 is about a minute after a minute of construction
                    big["cpu_baseline"] = cpu_reference_arm(n5, s5, d5, dim5, steps=1, warmup=1)
                else:
                    big["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                           "sample": "not timed in the default run: one round of the reference on this graph is ~60 s "
                                                     "after ~66 s of engine construction (13 workers x 8.7 GB of accumulators fit this "
                                                     "host).  `bench.py --impl reference --config c5` times it on the full graph: "
                                                     "12.98 M pair-terms/s on this pool's 16-core host (profiles/r02_reference_c5.json); "
                                                     "`--largest-cpu-baseline` runs it inside this record"}
                line["largest_config"] = big
            except Exception as e:  # noqa: BLE001
                line["largest_config"] = {"unavailable": str(e)[:300]}
        print(json.dumps(line))
        return

    # ------------------------------------------------------------------------------------------------ N > 1
    neg_mode = P.NEG_PER_VERTEX_K if args.neg_mode == "per_vertex_k" else P.NEG_PER_EDGE_2

    def build_engine(peer_broadcast):
        e = sharded.make_cuda_engine(g, dim, 1, comm_chunks=args.comm_chunks, device=local_rank, neg_mode=neg_mode,
                                     negatives=k if neg_mode == P.NEG_PER_VERTEX_K else 0,
                                     chunk_entries=args.chunk_entries, bucket_mode=args.bucket_mode,
                                     peer_broadcast=peer_broadcast,
                                     exchange=False if (test_backend and not peer_broadcast) else None)
        e.ops.ctx.init_coords(P.INIT_UNIFORM_PM1 if init == "uniform_pm1" else P.INIT_NORMAL, 1, std)
        return e

    # fused update + broadcast into the peers' buffers when every rank can open them AND the replicas agree after two
    # trial rounds; otherwise the NCCL all-gather per comm chunk
    exchange_path = "nccl all-gather per chunk"
    eng = None
    if args.peer_broadcast != "off":
        try:
            eng = build_engine(True)
            for _ in range(2):
                eng.run_single_iteration()
            torch.cuda.synchronize()
            dist.barrier()
            if sharded.replicas_agree(eng.ops.x_next(), None) and sharded.replicas_agree(
                    torch.as_tensor(sharded._DeviceArray(eng.ops.ctx.device_coords(0), (eng.ops.rows, eng.ops.ld)),
                                    device=eng.ops.device), None):
                exchange_path = "peer stores from the gather kernel (CUDA IPC)"
            else:
                raise RuntimeError("replicas differ")
        except Exception as e:  # noqa: BLE001
            if rank == 0:
                print(f"[bench] peer broadcast unavailable ({e}); using the all-gather path", file=sys.stderr)
            eng = None
    if eng is None:
        eng = build_engine(False)
    ctx = eng.ops.ctx
    stream = eng.ops.stream

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        eng.run_single_iteration()
    mu, sigma = eng.mu, eng.sigma

    sampler = ClockSampler(local_rank)
    launches0 = ctx.kernel_launches
    ctx.elapsed_ms()
    barrier()
    sampler.start()
    w0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    eng.gather_events = []
    for s in range(args.steps):
        eng.round_async(mu, sigma, eng.iter + s)
    with torch.cuda.stream(stream):
        eng._wait_pending()
    ev1.record(stream)
    barrier()
    w1 = time.perf_counter()
    ms = ev0.elapsed_time(ev1)
    gather_ms = sum(a.elapsed_time(b) for a, b in eng.gather_events) / args.steps  # this rank's gather launches per round
    eng.gather_events = None
    launches = ctx.kernel_launches - launches0
    ctx.sync()
    t = torch.tensor([ms, gather_ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, gather_ms = float(t[0].item()), float(t[1].item())
    # the timed region is short: the same rounds continue untimed (the same number on every rank) until the clock sampler
    # has seen ~0.5 s of this load
    extra = max(0, int(500.0 / max(ms / args.steps, 1e-3)) - args.steps)
    for s in range(extra):
        eng.round_async(mu, sigma, eng.iter + 10000 + s)
    with torch.cuda.stream(stream):
        eng._wait_pending()
    barrier()
    clocks = sampler.finish(w0, w1)
    ctx.sync()
    pair_terms = ctx.pair_terms  # m + S, job-wide per iteration
    ms_per_step = ms / args.steps
    line = dict(base_line)
    samples_path = ("own anchors + peer stores from the pack kernel" if eng.ops.direct_exchange else
                    ("own anchors + all-to-all" if eng.ops.exchange_tensors() is not None else "replicated enumeration"))
    line.update({"value": pair_terms / (ms_per_step * 1e-3), "ms_per_step": ms_per_step,
                 "sampling": "k=%d negatives per vertex (S = n k)" % k if neg_mode == P.NEG_PER_VERTEX_K else "2 negatives per edge",
                 "pair_terms_per_iteration": int(pair_terms), "sigma": sigma,
                 "parallelism": f"vertex-sharded x{world}, samples: {samples_path}, coordinates: {exchange_path}",
                 "clocks": clocks, "gpu_launches": int(launches)})

    # HBM roofline of the dominant kernel per rank: a rank gathers for the vertices it owns, 1/world of the job's
    # algorithmic bytes (section 8d formula), in `chunks` launches per round; the slowest rank's time; no DRAM byte count
    # (ncu runs on one GPU only), so the algorithmic figure stands in and says so

    peak = float(peaks.get("hbm_gbs", 6650.0))
    b_rank = ctx.algorithmic_bytes / world
    alg = b_rank / (gather_ms * 1e-3) / 1e9
    line["roofline"] = {"bound": "hbm", "peak": peak, "unit": "GB/s", "kernel": "gather_batched_kernel (per rank)",
                        "kernel_ms": gather_ms, "launches_per_round": eng.chunks, "algorithmic_bytes": int(b_rank),
                        "achieved": alg, "frac": alg / peak, "traffic": None,
                        "frac_basis": "ALGORITHMIC bytes of one rank's share (counts L2-served hub rows as HBM traffic: can exceed 1) "
                                      "/ slowest rank's live gather time per round",
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if peaks else "fallback 6650 GB/s",
                        "step_frac": ctx.algorithmic_bytes / world / (ms_per_step * 1e-3) / 1e9 / peak}

    # end to end at N GPUs with HOST buffers: every rank uploads X_t (each needs all of it; N PCIe links in
    # parallel), the round runs, every rank returns the rows it owns (together X_{t+1}) and the job-wide tallies
    x_host = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
    ctx.get_coords(x_host.numpy())
    block, rows_pad, ld = eng.block_rows, eng.ops.rows, eng.ops.ld
    own = [(min(n, (ch * world + rank) * block), min(n, (ch * world + rank + 1) * block)) for ch in range(eng.chunks)]
    out_host = torch.empty((sum(hi - lo for lo, hi in own), dim), dtype=torch.float32, pin_memory=True)
    t_e2e = []
    for s in range(max(1, args.e2e_steps) + 1):
        barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            ctx.set_coords(x_host.numpy())
            eng.round_async(mu, sigma, eng.iter + args.steps + s)
            eng.finish_round()
            x_dev = torch.as_tensor(sharded._DeviceArray(ctx.device_coords(0), (rows_pad, ld)), device=eng.ops.device)
            at = 0
            for lo, hi in own:
                out_host[at:at + hi - lo].copy_(x_dev[lo:hi, :dim], non_blocking=True)
                at += hi - lo
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        t_e2e.append(float(dt.item()))
    e2e_s = float(np.median(t_e2e[1:]))
    if rank == 0:
        line["e2e"] = {"value": pair_terms / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(world * n * dim * 4),
                       "d2h_bytes_per_step": int(n * dim * 4 + 2 * 512 * 8), "ms_per_step": e2e_s * 1e3,
                       "call": "per rank: X_t in (pinned host), sharded round, owned rows of X_{t+1} + tallies out"}
        print(json.dumps(line))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
