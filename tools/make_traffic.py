"""Turns ncu launch lists of the round into profiles/traffic.json (read by bench.py's roofline record).

    python tools/make_traffic.py c4=gpurun_out/r02_c4_round_metrics.csv c5=gpurun_out/r02_c5_round_metrics.csv \
        c4_per_edge_2=gpurun_out/r02_c4_pe2_round_metrics.csv

Each CSV is the `--csv --log-file` output of

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
        --clock-control none python tools/profile_round.py --config cN --rounds 2 --warm-iters 3

(all launches of the process).  Only the launches from the first sampling kernel on are rounds; per configuration the
file keeps the DRAM bytes of ONE gather launch (median over the profiled rounds), its L2 hit rate, the bytes of one
whole round and the per-kernel table.  The file is stamped with a hash of the kernel sources, and bench.py ignores it
when the sources have changed since -- a traffic figure always belongs to the build it was measured on.
"""
import collections
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import kernel_source_hash  # noqa: E402

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
        "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "second": 1e3, "%": 1.0, "": 1.0}


def launches(path):
    rows = [r for r in csv.reader(open(path, newline="")) if len(r) > 10]
    hdr = next(r for r in rows if "Metric Name" in r)
    col = {name: hdr.index(name) for name in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    out = collections.OrderedDict()
    for r in rows:
        if r is hdr or not r[col["ID"]].isdigit():
            continue
        rec = out.setdefault(int(r[col["ID"]]), {"name": r[col["Kernel Name"]]})
        value = float(r[col["Metric Value"]].replace(",", "")) * UNIT.get(r[col["Metric Unit"]], 1.0)
        rec[r[col["Metric Name"]]] = value
    return list(out.values())


def short(name):
    name = name.split("(")[0]
    return name.split("::")[-1].split("<")[0].strip()


def summarise(path):
    ls = launches(path)
    first = next(i for i, l in enumerate(ls) if short(l["name"]).startswith("sample"))
    ls = ls[first:]
    gathers = [l for l in ls if short(l["name"]).startswith("gather")]
    rounds = len(gathers)
    dram = lambda l: l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    per_kernel = collections.OrderedDict()
    for l in ls:
        k = per_kernel.setdefault(short(l["name"]), {"launches_per_round": 0.0, "ms": 0.0, "dram_bytes": 0.0})
        k["launches_per_round"] += 1.0 / rounds
        k["ms"] += l.get("gpu__time_duration.sum", 0.0) / rounds
        k["dram_bytes"] += dram(l) / rounds
    return {"gather_dram_bytes": statistics.median(dram(l) for l in gathers),
            "gather_dram_read_bytes": statistics.median(l.get("dram__bytes_read.sum", 0.0) for l in gathers),
            "gather_l2_hit_pct": statistics.median(l.get("lts__t_sector_hit_rate.pct", 0.0) for l in gathers),
            "gather_ms_under_ncu": statistics.median(l.get("gpu__time_duration.sum", 0.0) for l in gathers),
            "step_dram_bytes": sum(dram(l) for l in ls) / rounds, "rounds_profiled": rounds,
            "per_kernel": per_kernel}


if __name__ == "__main__":
    out = {"_comment": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (tools/make_traffic.py); bench.py reads "
                       "gather_dram_bytes / step_dram_bytes into roofline.traffic when kernel_source_hash matches",
           "kernel_source_hash": kernel_source_hash(), "source": "ncu --metrics dram__bytes_{read,write}.sum, all launches of "
                                                                "tools/profile_round.py (--clock-control none)"}
    path = os.path.join(ROOT, "profiles", "traffic.json")
    for arg in sys.argv[1:]:
        key, csv_path = arg.split("=", 1)
        out[key] = summarise(csv_path)
        print(key, json.dumps({k: v for k, v in out[key].items() if k != "per_kernel"}))
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path)
