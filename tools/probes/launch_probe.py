#!/usr/bin/env python3
"""Per-launch cost of tiny dependent kernels on one stream, alone and while a
large pinned H2D / D2H copy runs on another stream; eager vs CUDA graph."""
import torch
s, side = torch.cuda.Stream(), torch.cuda.Stream()
x = torch.zeros(1024, device="cuda")
big_h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
big_d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
N = 200

def work():
    for _ in range(N):
        x.add_(1)

g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    work()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        work()
for mode in ("alone", "h2d", "d2h"):
    for kind in ("eager", "graph"):
        torch.cuda.synchronize()
        if mode == "h2d":
            with torch.cuda.stream(side):
                big_d.copy_(big_h, non_blocking=True)
        elif mode == "d2h":
            with torch.cuda.stream(side):
                big_h.copy_(big_d, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            if kind == "eager":
                work()
            else:
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        print(f"{mode:5s} {kind:5s}: {1000 * e0.elapsed_time(e1) / N:.2f} us/launch", flush=True)
