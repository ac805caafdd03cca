#!/usr/bin/env python3
"""e2e (host-buffer) encode of cfg2 with the pipelined host API: wall time per
call for several wave sizes; with BBPE_TIMELINE=1 the library prints the
per-wave copy/kernel timeline to stderr."""
import os, sys, time, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import text as synth

t = bb.load_merge_table_files(os.path.join(ROOT, "tests/golden/gpt2.bbpt"), None, "binary")
gen = synth.TextGen(synth.word_list(t))
data, offsets, desc = synth.config_rows(gen, 2, scale=1.0, seed=2000)
n = offsets.size - 1
total = int(offsets[-1])
enc = bb.Encoder(device=0)
enc.prepare(t)
hd = torch.from_numpy(data).pin_memory().numpy()
ho = torch.from_numpy(offsets.view(np.int64)).pin_memory().numpy().view(np.uint64)
hi = torch.empty(total, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
hoo = torch.empty(n + 1, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
waves = [int(x) for x in sys.argv[1:]] or [0]
res = {}
for wb in waves:
    enc.set_config(wave_bytes=wb)
    for _ in range(2):
        enc.encode_packed(t, hd, ho, hi, hoo)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        _, _, st = enc.encode_packed(t, hd, ho, hi, hoo)
        ts.append((time.perf_counter() - t0) * 1e3)
    res[wb] = (float(np.median(ts)), st.get("waves"))
    print(json.dumps({"wave_bytes": wb, "ms_median": float(np.median(ts)), "ms_min": min(ts), "waves": st.get("waves")}), flush=True)
