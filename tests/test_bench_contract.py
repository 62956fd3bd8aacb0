"""bench.py's JSON contract: the reference arm runs on the host alone (checked without a GPU); the GPU arm at N = 1 and the
N = 2 control flow are `-m gpu` tests."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgempe_ref.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1", "--cpu-seconds", "2"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "pair_terms_per_second" and d["unit"] == "pair-terms/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["config"]["workload"] and d["n_gpus"] == 1 and d["ms_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_leaves_other_ranks_idle():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT,
                         env={**os.environ, "RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1", "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0 and out.stdout.strip() == ""


def _one_line(out):
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


CONTRACT_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                 "vs_baseline", "dtype", "data", "config", "clocks", "gpu_launches", "roofline", "e2e")


@pytest.mark.gpu
def test_gpu_arm_prints_one_contract_line():
    """The default arm on a small BASELINE configuration (c2): every key of the contract, live roofline, CPU baseline."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c2", "--steps", "5", "--warmup", "3",
                          "--cpu-seconds", "2", "--no-sub-records"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    d = _one_line(out)
    for key in CONTRACT_KEYS + ("cpu_baseline",):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"] and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and r["achieved"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] < d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_gpu_arm_control_flow_with_two_ranks():
    """torchrun with two ranks, both time-sliced on cuda:0 over gloo (GEMPE_BENCH_TEST_BACKEND: no kernel waits on another
    rank) -- not a bench number, a check that the N > 1 path (engine build, peer stores, barriers, max over ranks, e2e
    leg, one JSON line from rank 0) runs."""
    env = {**os.environ, "GEMPE_BENCH_TEST_BACKEND": "gloo"}
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "c2"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    d = _one_line(out)
    for key in CONTRACT_KEYS:
        assert key in d, key
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["roofline"]["kernel_ms"] > 0 and d["e2e"]["value"] > 0
    assert "vertex-sharded x2" in d["parallelism"]
