"""Summarises an Nsight Compute report (read on the CPU box) into profiles/<name>.md.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r01_x.md ["free-text note"]
"""
import collections
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
lines = [f"# ncu summary: {rep}", "", note, ""]
for k, vals in enumerate(rows[2:]):
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else f"launch {k}"
    lines.append(f"## launch {k}: `{name[:110]}`")
    lines.append("")
    lines.append("| metric | value | unit |")
    lines.append("|---|---|---|")
    for key in KEYS:
        if key in hdr:
            i = hdr.index(key)
            lines.append(f"| {key} | {vals[i]} | {units[i]} |")
    lines.append("")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
srows = [r for r in csv.reader(io.StringIO(src)) if len(r) > 6 and r[0].startswith("0x")]
if srows:
    tot_s = sum(int(r[2]) for r in srows) or 1
    tot_i = sum(int(r[5]) for r in srows) or 1
    lines += ["## SASS hot spots (first launch): stall samples / executed count", "", "```"]
    for r in sorted(srows, key=lambda r: -int(r[2]))[:20]:
        lines.append(f"{100 * int(r[2]) / tot_s:5.1f}%  {int(r[5]):>12}  {r[1].strip()[:100]}")
    lines += ["```", "", "## opcode mix (share of executed warp instructions, share of stall samples)", "", "```"]
    mix, smp = collections.Counter(), collections.Counter()
    for r in srows:
        parts = r[1].strip().split()
        op = (parts[1] if parts[0].startswith("@") else parts[0]).split(".")[0]
        mix[op] += int(r[5])
        smp[op] += int(r[2])
    for op, c in mix.most_common(20):
        lines.append(f"{op:<10} {100 * c / tot_i:5.1f}%  {100 * smp[op] / tot_s:5.1f}%")
    lines += ["```", ""]
open(out, "w").write("\n".join(lines))
print("wrote", out)
