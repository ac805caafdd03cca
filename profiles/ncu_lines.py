#!/usr/bin/env python3
"""Summarise an ncu `--page source --csv --print-source=cuda,sass` dump by CUDA
source line: samples (stall), instructions executed, top stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = []
tot_s = tot_i = 0
for r in rows[3:]:
    if r and r[0] and len(r) == len(hdr):
        try:
            s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
            ins = int(r[idx["Instructions Executed"]] or 0)
        except ValueError:
            continue
        st = sorted(((int(r[idx[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
        lines.append((s, ins, r[0], r[1][:70], st))
        tot_s += s
        tot_i += ins
lines.sort(reverse=True)
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, ins, no, src, st in lines[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/max(tot_s,1):5.1f}% {100*ins/max(tot_i,1):5.1f}%i L{no:>4} {src:70s} {st}")
