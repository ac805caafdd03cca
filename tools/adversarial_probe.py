"""Full-size adversarial batches (256 MiB each, SURVEY §8d sidecar set):
random bytes, 64 KiB runs of one byte, 4 KiB digit rows, 1 KiB rows of
random CJK. Every row is checked against the compiled reference
(bench.parity_check: oracle/_ref heap_bpe on every row + the block engine on
a sample); prints the wall time per synchronous encode and the per-kernel split.

  python tools/adversarial_probe.py [case ...] [--engine pieces|block]
"""
import os, sys, json, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2507_11941_b200 as bb
from oracle.oracle import Reference
from workloads import tables as WT

engine = "block" if "--engine=block" in sys.argv else "pieces"
want = [a for a in sys.argv[1:] if not a.startswith("--")]
t = bb.load_merge_table_files(WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
ref = Reference.load_files(WT.GPT2_VOCAB, WT.GPT2_MERGES)
rng = np.random.default_rng(7)
N = 256 << 20


def cjk(n):
    cp = rng.integers(0x4E00, 0xA000, n // 3 + 1)
    b = np.stack([0xE0 | (cp >> 12), 0x80 | ((cp >> 6) & 0x3F), 0x80 | (cp & 0x3F)], 1).astype(np.uint8).reshape(-1)
    return b[:n]


cases = {
    "random_bytes_256B_rows": (lambda: rng.integers(0, 256, N, dtype=np.uint8), 256),
    "runs_a_64KiB_rows": (lambda: np.full(N, ord("a"), np.uint8), 65536),
    "runs_dot_64KiB_rows": (lambda: np.full(N, ord("."), np.uint8), 65536),
    "digits_4KiB_rows": (lambda: rng.integers(ord("0"), ord("9") + 1, N, dtype=np.uint8), 4096),
    "cjk_1KiB_rows": (lambda: cjk(N), 1023),
}
enc = bb.Encoder(0, engine=engine)
for name, (mk, L) in cases.items():
    if want and name not in want:
        continue
    data = mk()
    n = N // L
    off = np.arange(0, n + 1, dtype=np.uint64) * np.uint64(L)
    data = data[: int(off[-1])]
    tot = int(off[-1])
    dd = torch.from_numpy(data).cuda(); do = torch.from_numpy(off.view(np.int64)).cuda()
    di = torch.empty(tot, dtype=torch.int32, device="cuda"); doo = torch.empty(off.size, dtype=torch.int64, device="cuda")
    for _ in range(2):
        enc.encode_device(t, dd.data_ptr(), do.data_ptr(), n, tot, di.data_ptr(), doo.data_ptr())
    enc.kernel_times(reset=True)
    enc.piece_stats(reset=True)
    # (the encoder's own stream: wall time around synchronous calls)
    torch.cuda.synchronize(); w0 = time.perf_counter()
    for _ in range(3):
        enc.encode_device(t, dd.data_ptr(), do.data_ptr(), n, tot, di.data_ptr(), doo.data_ptr(), sync=True)
    wall_ms = (time.perf_counter() - w0) * 1000 / 3
    kt, kc = enc.kernel_times(reset=True)
    ps = enc.piece_stats(reset=True)
    oo = doo.cpu().numpy().view(np.uint64)
    ids = di[: int(oo[-1])].cpu().numpy().view(np.uint32)
    par = bench.parity_check(ref, data, off, ids, oo, 30.0)
    print(json.dumps({"case": name, "engine": engine, "rows": n, "tokens": int(oo[-1]),
                      "wall_ms": round(wall_ms, 3),
                      "kernel_ms": {k: round(v / kc, 3) for k, v in kt.items() if v},
                      "long_pieces": ps["long_pieces"] // 3, "long_byte_fraction": ps["long_byte_fraction"],
                      "parity": {k: par[k] for k in ("rows_checked", "mismatches", "oracle")}}), flush=True)
    assert par["mismatches"] == 0, par
    del dd, do, di, doo
    torch.cuda.empty_cache()
