#!/usr/bin/env python
"""Benchmark of the GEMPE round (BASELINE.json metric: edge+negative gradient terms per second per iteration,
and the fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

A "step" is one GEMPE iteration (sampling passes + gradient gather + update) over the synthetic graph of the
chosen BASELINE configuration (default c4: R-MAT scale 20, d=128, 20 negatives per vertex).  One JSON line is
printed by rank 0.  `--impl reference` times the reference's own CPU engine (oracle/_ref) on host cores.
"""
from __future__ import annotations

import argparse
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
                   help="CPU budget on rank 0 (default: 20 s for the cpu_baseline leg, 30 s for --impl reference)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--peer-broadcast", default="auto", choices=["auto", "off"],
                   help="N > 1: gather kernel stores updated rows into the peers' buffers (auto) or NCCL all-gather (off)")
    return p.parse_args()


def workload_name(cfg):
    return {"c1": "SBM n=3000 6 blocks d=2 k=5", "c2": "Barabasi-Albert n=1e5 m=8 d=2 k=10",
            "c3": "Dirichlet-SBM n=2e5 deg20 d=64 k=10", "c4": "R-MAT scale 20 ef16 d=128 k=20",
            "c5": "R-MAT scale 24 ef16 d=128 k=20"}[cfg]


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons while the timed region runs: NVML every 5 ms when pynvml is importable
    (the timed region is ~0.1 s), else `nvidia-smi` every 0.2 s."""
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
                    self.rows.append([str(mhz), str(self.max_mhz)] +
                                     ["active" if mask & bit else "not active" for bit, _ in self.bits])
                else:
                    out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i",
                                          str(self.index)], capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._halt.wait(0.005 if self.nvml else 0.2)

    def finish(self):
        self._halt.set()
        self.join(timeout=6)
        sm = sorted(int(r[0]) for r in self.rows if r[0].isdigit())
        mx = [int(r[1]) for r in self.rows if r[1].isdigit()]
        reasons = sorted({n for r in self.rows for n, v in zip(self.NAMES, r[2:6]) if v.lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def cpu_reference_arm(n, src, dst, dim, budget_s, steps=None, warmup=1):
    """Times EmbeddingEngine::run_single_iteration of the UNMODIFIED reference (oracle/_ref) on the host cores.
    Bounded sample: the leading edges of the workload's edge list on the full vertex set (the reference's
    own 2-draws-per-edge sampling, so pair-terms = 3 m'), sized from a probe round to fit the budget."""
    import oracle as O
    ref = O.Ref()
    cores = os.cpu_count() or 1
    # accumulator bank = workers * lanes * n * (d+1) * 4 bytes (engine.cpp:77-86): keep it under ~40% of RAM
    try:
        avail = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) * 1024
    except Exception:
        avail = 32 << 30
    lanes = 16 if dim <= 8 else 1
    workers = max(1, min(cores, int(0.4 * avail / max(1, lanes * n * (dim + 1) * 4))))
    m_probe = min(len(src), 200_000)

    def rate(m_use, rounds, warm):
        eng = O.RefEngine(ref, n, src[:m_use], dst[:m_use], dim, 1, lane_width=lanes, workers=workers)
        eng.set_capture(False)
        for _ in range(warm):
            eng.iterate(capture=False)
        times = []
        for _ in range(rounds):
            t0 = time.perf_counter()
            eng.iterate(capture=False)
            times.append(time.perf_counter() - t0)
        return 3.0 * m_use / float(np.median(times)), float(np.median(times))

    r_probe, _ = rate(m_probe, 1, 1)
    rounds = steps if steps else 3
    m_use = int(min(len(src), max(m_probe, r_probe / 3.0 * budget_s / (rounds + warmup + 1))))
    value, sec = rate(m_use, rounds, warmup)
    return {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
            "sample": f"first {m_use} of {len(src)} edges on all {n} vertices, reference sampling (2 draws/edge, "
                      f"3m pair-terms), lane_width={lanes}, {rounds} timed rounds, median {sec:.3f} s/round",
            "host_cores": cores, "sample_ms_per_round": sec * 1e3}


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
        base = cpu_reference_arm(n, src, dst, dim, args.cpu_seconds or 30.0, steps=args.steps, warmup=args.warmup)
        line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": base["sample_ms_per_round"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": {"workload": workload_name(args.config), "n": n, "m": int(len(src))},
                "cpu_baseline": base,
                "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    import paper_2011_03479_b200 as P
    from paper_2011_03479_b200 import sharded

    # test hook: GEMPE_BENCH_TEST_BACKEND=gloo runs the N > 1 control flow with every rank time-sliced on cuda:0 (no
    # kernel waits on another rank; sample exchange off because gloo has no CUDA all-to-all) -- never a bench number
    test_backend = os.environ.get("GEMPE_BENCH_TEST_BACKEND")
    if test_backend:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if test_backend:
            dist.init_process_group(test_backend)
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    n, src, dst, dim, k, _, init, std = graphgen.make_config(args.config, device=gen_device())
    torch.cuda.empty_cache()
    g = P.Graph(n, src, dst)
    neg_mode = P.NEG_PER_VERTEX_K if args.neg_mode == "per_vertex_k" else P.NEG_PER_EDGE_2
    def build_engine(peer_broadcast):
        e = sharded.make_cuda_engine(g, dim, 1, comm_chunks=args.comm_chunks, device=local_rank, neg_mode=neg_mode,
                                     negatives=k if neg_mode == P.NEG_PER_VERTEX_K else 0,
                                     chunk_entries=args.chunk_entries, bucket_mode=args.bucket_mode,
                                     peer_broadcast=peer_broadcast,
                                     exchange=False if (test_backend and not peer_broadcast) else None)
        e.ops.ctx.init_coords(P.INIT_UNIFORM_PM1 if init == "uniform_pm1" else P.INIT_NORMAL, 1, std)
        return e

    # N > 1: fused update + broadcast into the peers' buffers when every rank can open them AND the replicas agree
    # after two trial rounds; otherwise the NCCL all-gather per comm chunk
    exchange_path = "none"
    if world > 1:
        exchange_path = "nccl all-gather per chunk"
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
        if exchange_path.startswith("nccl"):
            eng = build_engine(False)
    else:
        eng = build_engine(False)
    ctx = eng.ops.ctx
    stream = eng.ops.stream

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: real iterations with the host sigma search (the state the timed rounds start from)
    for _ in range(max(args.warmup, 3)):
        eng.run_single_iteration()
    mu, sigma = eng.mu, eng.sigma

    sampler = ClockSampler(local_rank)
    launches0 = ctx.kernel_launches
    ctx.elapsed_ms()  # reset the context's event log
    barrier()
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in range(args.steps):
        if world > 1:
            eng.round_async(mu, sigma, eng.iter + s)
        else:
            ctx.iterate_async(mu, sigma, eng.iter + s)
    if world > 1:
        with torch.cuda.stream(stream):
            eng._wait_pending()
    ev1.record(stream)
    barrier()
    clocks = sampler.finish()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.kernel_launches - launches0
    he, hn = ctx.sync()  # status check of the last timed round (raises on divergence / retry cap)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pair_terms = ctx.pair_terms  # m + S, job-wide per iteration
    ms_per_step = ms / args.steps
    value = pair_terms / (ms_per_step * 1e-3)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "n": n, "m": int(len(src)), "dim": dim,
                       "negatives": "k=%d per vertex" % k if neg_mode == P.NEG_PER_VERTEX_K else "2 per edge",
                       "pair_terms_per_iteration": int(pair_terms), "sigma": sigma,
                       "l2": "inputs larger than L2 (X %.0f MB + lists)" % (n * dim * 4 / 1e6) if n * dim * 4 > 126e6
                             else "working set fits L2 (reported as is)",
                       "parallelism": f"vertex-sharded x{world}, samples: "
                                      f"{'own anchors + peer stores from the pack kernel' if eng.ops.direct_exchange else ('own anchors + all-to-all' if eng.ops.exchange_tensors() is not None else 'replicated enumeration')}"
                                      f", coordinates: {exchange_path}"
                                      if world > 1 else "1 GPU"},
            "clocks": clocks, "gpu_launches": int(launches)}

    if rank == 0 and world == 1:
        # roofline of the dominant kernel (gather+update), timed live with CUDA events on its own stream
        tot, samp_ms, gath_ms = ctx.elapsed_ms()
        draws = None
        _, draws = ctx.sample(eng.iter)  # p-bar: LCG draws per accepted sample
        p_bar = draws / max(1, ctx.sample_slots)
        b_alg = ctx.algorithmic_bytes + int((p_bar - 1.0) * ctx.sample_slots)
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        peak = float(peaks.get("hbm_gbs", 6650.0))
        gather_s = gath_ms / args.steps * 1e-3
        achieved = b_alg / gather_s / 1e9
        traffic = None
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config)
        except Exception:
            pass
        line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                            "traffic": traffic, "kernel": "gather_kernel", "algorithmic_bytes": int(b_alg),
                            "kernel_ms": gath_ms / args.steps, "sampling_passes_ms": samp_ms / args.steps,
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s",
                            "draws_per_sample": p_bar,
                            # the same launch on ncu's DRAM byte count (hub rows re-read from L2 are not HBM traffic)
                            "achieved_dram": (traffic / gather_s / 1e9) if traffic else None,
                            "frac_dram": (traffic / gather_s / 1e9 / peak) if traffic else None}

        # whole iterations with the device-resident sigma feedback (round + sigma search + PE estimate, no host sync)
        ctx.set_sigma(mu, sigma)
        for s in range(3):
            ctx.iterate_auto_async(eng.iter + s)
        torch.cuda.synchronize()
        fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fe0.record(stream)
        for s in range(args.steps):
            ctx.iterate_auto_async(eng.iter + 3 + s)
        fe1.record(stream)
        torch.cuda.synchronize()
        ctx.sync()
        full_ms = fe0.elapsed_time(fe1) / args.steps
        line["full_iteration"] = {"ms_per_step": full_ms, "value": pair_terms / (full_ms * 1e-3), "unit": UNIT,
                                  "what": "round + device sigma search + PE estimate (run_single_iteration), no host sync"}
        ctx.elapsed_ms()

        # small graphs: the same rounds as one CUDA graph of 50, gaps between the ~5 kernels removed
        if ms_per_step < 1.0:
            reps = 50
            ctx.graph_capture(mu, sigma, eng.iter + 100, reps)
            ctx.graph_launch()
            torch.cuda.synchronize()
            if reps % 2:
                ctx.graph_capture(mu, sigma, eng.iter + 100, reps)
            ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ge0.record(stream)
            ctx.graph_launch()
            ge1.record(stream)
            torch.cuda.synchronize()
            ctx.sync()
            g_ms = ge0.elapsed_time(ge1) / reps
            line["cuda_graph"] = {"rounds_per_graph": reps, "ms_per_step": g_ms, "value": pair_terms / (g_ms * 1e-3),
                                  "unit": UNIT, "what": "50 rounds captured into one CUDA graph, one launch"}
            ctx.elapsed_ms()

        # end to end through the C-ABI with HOST buffers: X_t in (pinned), round, X_{t+1} + tallies out
        x_host = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
        x_np = x_host.numpy()
        ctx.get_coords(x_np)
        steps_e2e = max(1, args.e2e_steps)
        t_e2e = []
        x_out_host = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
        bufs = [x_np, x_out_host.numpy()]
        for s in range(steps_e2e + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.step_host(bufs[s % 2], bufs[(s + 1) % 2], mu, sigma, eng.iter + s)
            t_e2e.append(time.perf_counter() - t0)
        e2e_s = float(np.median(t_e2e[1:]))
        line["e2e"] = {"value": pair_terms / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(n * dim * 4),
                       "d2h_bytes_per_step": int(n * dim * 4 + 2 * 512 * 8), "ms_per_step": e2e_s * 1e3,
                       "call": "gempe_step_host: X_t in, round, X_{t+1} + tallies out (pinned host buffers, copies overlapped)"}
        if not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_reference_arm(n, src, dst, dim, args.cpu_seconds or 20.0)
            except Exception as e:  # the reference build is test infrastructure; its absence is reported, not fatal
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
    if world > 1:
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
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
