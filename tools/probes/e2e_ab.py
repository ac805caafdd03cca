"""e2e A/B of two library builds (same C-ABI subset): median bbpe_encode time
on cfg2 from pinned host buffers.  python tools/probes/e2e_ab.py lib1.so [lib2.so ...]"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from workloads import tables as WT, text as WX  # noqa: E402


class Config(C.Structure):
    _fields_ = [("block_size", C.c_uint32), ("max_passes", C.c_int64), ("engine", C.c_int32),
                ("wave_bytes", C.c_uint64), ("piece_memo", C.c_int32), ("no_dedup", C.c_int32),
                ("pattern", C.c_int32)]


data, off, _ = WX.config_rows(WX.TextGen(WX.word_list(WT.gpt2_table()[0])), 2)
n, total = off.size - 1, int(off[-1])
for path in sys.argv[1:]:
    L = C.CDLL(os.path.abspath(path))
    t, ctx = C.c_void_p(), C.c_void_p()
    assert L.bbpe_table_load_files(WT.GPT2_VOCAB.encode(), WT.GPT2_MERGES.encode(), 0, C.byref(t)) == 0
    cfg = Config(256, 0, 0, 0, 1, 0, 0)
    assert L.bbpe_ctx_create(0, C.byref(cfg), C.byref(ctx)) == 0
    bufs = []
    for nb in (total, (n + 1) * 8, total * 4, (n + 1) * 8):
        p = C.c_void_p()
        assert L.bbpe_host_alloc(C.c_size_t(nb), C.byref(p)) == 0
        bufs.append(p)
    C.memmove(bufs[0], data.ctypes.data, total)
    C.memmove(bufs[1], off.ctypes.data, (n + 1) * 8)
    enc = L.bbpe_encode
    enc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint64,
                    C.c_void_p, C.c_void_p]
    times = []
    for k in range(40):
        t0 = time.perf_counter()
        assert enc(ctx, t, bufs[0], bufs[1], n, bufs[2], total, bufs[3], None) == 0
        if k >= 10:
            times.append(time.perf_counter() - t0)
    print(os.path.basename(path), "e2e median ms", round(float(np.median(times)) * 1e3, 3),
          "min", round(min(times) * 1e3, 3), flush=True)
