#!/usr/bin/env python3
"""Device-resident encode of a wave-sized batch, eager vs captured into a CUDA
graph, alone and under a concurrent pinned D2H copy (BBPE_NO_KERNEL_TIMING=1)."""
import os, sys
import numpy as np
os.environ["BBPE_NO_KERNEL_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import text as synth

t = bb.load_merge_table_files(os.path.join(ROOT, "tests/golden/gpt2.bbpt"), None, "binary")
gen = synth.TextGen(synth.word_list(t))
enc = bb.Encoder(device=0)
enc.prepare(t)
s, side = torch.cuda.Stream(), torch.cuda.Stream()
big_h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
big_d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for rows in (4096, 87381):
    data, off, _ = synth.config_rows(gen, 2, scale=rows / (1 << 20), seed=7)
    n, total = off.size - 1, int(off[-1])
    d_data = torch.from_numpy(data).cuda()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_ids = torch.empty(total, dtype=torch.int32, device="cuda")
    d_oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")

    def step():
        enc.encode_device(t, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), d_oo.data_ptr(),
                          stream=s.cuda_stream, sync=False)
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    want = d_ids.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    torch.cuda.synchronize()
    for mode in ("alone", "d2h"):
        for kind in ("eager", "graph"):
            torch.cuda.synchronize()
            d_ids.zero_()
            if mode == "d2h":
                with torch.cuda.stream(side):
                    big_h.copy_(big_d, non_blocking=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 5
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(K):
                    step() if kind == "eager" else g.replay()
                e1.record(s)
            torch.cuda.synchronize()
            ok = bool(torch.equal(d_ids, want))
            print(f"{total >> 10} KiB {mode} {kind}: {e0.elapsed_time(e1) / K:.4f} ms ok={ok}", flush=True)
