#!/usr/bin/env python3
"""Summarise an ncu `--page source --csv --print-source=cuda,sass` dump by CUDA
source line (all files of the dump): stall samples, instructions executed, top
stall reasons.  usage: ncu_lines.py dump.csv [top_n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
lines, tot_s, tot_i = [], 0, 0
fname, hdr, idx, stalls = "?", None, {}, []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(hdr)}
        stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        ins = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    st = sorted(((int(r[idx[k]] or 0), k[6:]) for k in stalls if (r[idx[k]] or "0").isdigit()), reverse=True)[:3]
    lines.append((s, ins, f"{fname}:{r[0]}", r[1][:70], st))
    tot_s += s
    tot_i += ins
lines.sort(reverse=True)
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, ins, no, src, st in lines[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/max(tot_s,1):5.1f}% {100*ins/max(tot_i,1):5.1f}%i {no:>16} {src:70s} {st}")
