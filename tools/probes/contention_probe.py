#!/usr/bin/env python3
"""Device-resident encode of one wave-sized batch (cfg2 rows), timed with CUDA
events: alone, with a concurrent pinned H2D copy, and with a concurrent D2H
copy. Separates per-wave fixed cost from PCIe-copy contention."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import text as synth

t = bb.load_merge_table_files(os.path.join(ROOT, "tests/golden/gpt2.bbpt"), None, "binary")
gen = synth.TextGen(synth.word_list(t))
enc = bb.Encoder(device=0)
enc.prepare(t)
s = torch.cuda.Stream()
side = torch.cuda.Stream()
big_h = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
big_d = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for rows in (4096, 32768, 87381, 1 << 20):
    data, off, _ = synth.config_rows(gen, 2, scale=rows / (1 << 20), seed=7)
    n = off.size - 1
    total = int(off[-1])
    d_data = torch.from_numpy(data).cuda()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_ids = torch.empty(total, dtype=torch.int32, device="cuda")
    d_oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")

    def step():
        enc.encode_device(t, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), d_oo.data_ptr(),
                          stream=s.cuda_stream, sync=False)
    for mode in ("alone", "h2d", "d2h"):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        if mode == "h2d":
            with torch.cuda.stream(side):
                big_d.copy_(big_h, non_blocking=True)
        elif mode == "d2h":
            with torch.cuda.stream(side):
                big_h.copy_(big_d, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 5
        e0.record(s)
        for _ in range(K):
            step()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        kt, kc = enc.kernel_times(reset=True)
        res[f"{total >> 10}KiB/{mode}"] = {"ms": round(ms, 4), "kernels": {k: round(v / max(kc, 1), 4) for k, v in kt.items()}}
        print(f"{total >> 10} KiB {mode}: {ms:.4f} ms", {k: round(v / max(kc, 1), 4) for k, v in kt.items()}, flush=True)
