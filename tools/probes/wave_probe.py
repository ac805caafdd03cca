"""Device-resident cfg2 encoded as W row waves (W in argv) instead of one call:
does an L2-sized staging working set cut the step? Times the whole sequence of
encode_device calls with CUDA events.  python tools/probes/wave_probe.py 1 2 4 8"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import tables as WT, text as WX

t = bb.load_merge_table_files(WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
data, off, _ = WX.config_rows(WX.make_gen("zipf", WT.gpt2_table()[0]), 2, seed=2000)
n, total = off.size - 1, int(off[-1])
enc = bb.Encoder(0)
d = torch.from_numpy(data).cuda()
o = torch.from_numpy(off.view(np.int64)).cuda()
ids = torch.empty(total, dtype=torch.int32, device="cuda")
oo = torch.empty(n + 1 + 64, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for W in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
    cuts = [n * k // W for k in range(W + 1)]
    waves = []
    for k in range(W):
        r0, r1 = cuts[k], cuts[k + 1]
        b0 = int(off[r0])
        waves.append((r0, r1, b0, int(off[r1]) - b0, (o[r0:r1 + 1] - b0).contiguous()))
    def step():
        obase = 0
        for r0, r1, b0, tb, wo in waves:
            enc.encode_device(t, d.data_ptr() + b0, wo.data_ptr(), r1 - r0, tb, ids.data_ptr() + 4 * obase,
                              oo.data_ptr() + 8 * (r0 + k), sync=False,
                               stream=torch.cuda.current_stream().cuda_stream)
            obase += tb // 2  # ids region per wave (rough: < bytes / 2 tokens)
    k = 0
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    enc.kernel_times(reset=True)
    step()
    torch.cuda.synchronize()
    kt, calls = enc.kernel_times(reset=True)
    print(W, "waves: ms/step median", round(sorted(ms)[len(ms) // 2], 3), {k: round(v, 3) for k, v in kt.items() if v > 0.01})
