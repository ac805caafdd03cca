#!/usr/bin/env python3
"""Summarise an ncu --set full report of one kernel into profiles/ (text + json).

usage: python profiles/summarize.py <report.ncu-rep> <out-prefix> [kernels.cu]
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else "paper_2507_11941_b200/csrc/kernels.cu"


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
summary = {k: d.get(k) for k in keys if k in d}
for k in list(summary):
    if u.get(k):
        summary[k] = f"{summary[k]} {u[k]}"
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(k) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(v for v in stalls.values() if v) or 1
stalls = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0)) if v}
rb, wb = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = None
if rb is not None and wb is not None:
    traffic = rb * scale.get(u.get("dram__bytes_read.sum", "byte"), 1) + wb * scale.get(u.get("dram__bytes_write.sum", "byte"), 1)
summary["traffic_bytes"] = traffic
summary["stall_pct_of_samples"] = stalls
with open(out + ".json", "w") as f:
    json.dump(summary, f, indent=1)
lines = [f"{k}: {v}" for k, v in summary.items() if k != "stall_pct_of_samples"]
lines.append("stalls (% of pc samples): " + ", ".join(f"{k} {v}" for k, v in list(stalls.items())[:8]))
with open(out + ".txt", "w") as f:
    f.write("\n".join(lines) + "\n\nhottest source lines:\n")
    cs = ncu("--page", "source", "--csv", "--print-source=cuda,sass")
    tmp = out + ".source.csv.tmp"
    open(tmp, "w").write(cs)
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), tmp, "25"], capture_output=True, text=True)
    f.write(r.stdout or r.stderr)
    os.remove(tmp)
print(open(out + ".txt").read())
