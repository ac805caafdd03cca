#!/usr/bin/env python3
"""PCIe bound of the e2e pipeline: the same H2D (bytes + offsets) and D2H
(ids + offsets) volumes as cfg2, in 16 MiB waves, H2D and D2H on two streams
(D2H of wave k after H2D of wave k), no kernels."""
import sys
import time
import torch
# argv[1]: output bytes per output id (4 = u32 ids, 2 = u16 transport)
IN, OUT, W = 276824072, 275898992 * int(sys.argv[1] if len(sys.argv) > 1 else 4) // 4, 16 << 20
h_in = torch.empty(IN, dtype=torch.uint8).pin_memory()
h_out = torch.empty(OUT, dtype=torch.uint8).pin_memory()
d_in = torch.empty(IN, dtype=torch.uint8, device="cuda")
d_out = torch.empty(OUT, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(w):
    n = (IN + w - 1) // w
    ev = [torch.cuda.Event() for _ in range(n)]
    for k in range(n):
        a, b = k * w, min(IN, (k + 1) * w)
        with torch.cuda.stream(s1):
            d_in[a:b].copy_(h_in[a:b], non_blocking=True)
            ev[k].record(s1)
    for k in range(n):
        a, b = k * w * OUT // IN, min(OUT, (k + 1) * w * OUT // IN)
        with torch.cuda.stream(s2):
            s2.wait_event(ev[k])
            h_out[a:b].copy_(d_out[a:b], non_blocking=True)
    torch.cuda.synchronize()
for w in (4 << 20, 16 << 20, 64 << 20):
    run(w)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); run(w); ts.append(time.perf_counter() - t0)
    print(f"wave {w >> 20} MiB: {1e3 * sorted(ts)[2]:.3f} ms (H2D {IN / 1e6:.0f} MB + D2H {OUT / 1e6:.0f} MB)", flush=True)
