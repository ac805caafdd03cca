#!/usr/bin/env python3
"""Bucket ncu per-line instruction counts of kernels.cu by function / k_pieces step."""
import csv
import re
import sys

src = open(sys.argv[2]).read().split("\n")
tiles = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
funcs = []
for i, l in enumerate(src, 1):
    m = re.search(r"(?:__global__|__device__).*?\b(\w+)\s*\(", l)
    if m and not l.strip().startswith("//"):
        funcs.append((i, m.group(1)))
kp = [i for i, l in enumerate(src, 1) if "k_pieces(EncodeArgs a, DevTable T)" in l][0]
steps = [(kp, "k_pieces:setup")]
for i, l in enumerate(src, 1):
    if i > kp:
        m = re.match(r"\s*// \((\w+)\)", l)
        if m:
            steps.append((i, "k_pieces:" + m.group(1)))
        if "load_window(S.w" in l:
            steps.append((i, "k_pieces:window"))
        if re.match(r"^(// k_|__global__|template)", l) and i > kp + 5:
            steps.append((i, None))
            break
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
idx = {h: i for i, h in enumerate(hdr)}
agg = {}
samp = {}
tot = 0
tots = 0
for r in rows[3:]:
    if not (r and r[0] and len(r) == len(hdr) and r[0].isdigit()):
        continue
    ln = int(r[0])
    ins = int(r[idx["Instructions Executed"]] or 0)
    sm = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    tot += ins
    tots += sm
    name = None
    for i, n in steps:
        if i <= ln:
            name = n
    if name is None or ln < kp:
        name = "?"
        for i, n in funcs:
            if i <= ln:
                name = n
    agg[name] = agg.get(name, 0) + ins
    samp[name] = samp.get(name, 0) + sm
print(f"{'region':24s} {'instr/unit':>10s} {'instr%':>6s} {'samples%':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -samp.get(x[0], 0)):
    print(f"{k:24s} {v / tiles:10.0f} {100 * v / max(tot, 1):5.1f}% {100 * samp.get(k, 0) / max(tots, 1):7.1f}%")
print(f"{'total':24s} {tot / tiles:10.0f}")
