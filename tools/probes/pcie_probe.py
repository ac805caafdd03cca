#!/usr/bin/env python3
"""PCIe probe: pinned H2D, D2H and concurrent (bidirectional) copy bandwidth on
cuda:0, CUDA events, best of 5. Bounds the e2e (host-buffer) encode."""
import json
import torch

def bw(n):
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                     ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))]:
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[name] = n / best / 1e6
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e0.record()
        with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1 = torch.cuda.Event(enable_timing=True); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res["bidir_each"] = n / best / 1e6
    return res

out = {str(n >> 20) + "MiB": bw(n) for n in (32 << 20, 256 << 20)}
print(json.dumps({"pcie_GBps": out}))
