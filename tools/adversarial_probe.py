"""Full-size adversarial batches (256 MiB each): random bytes, 64 KiB runs of
one byte, digit runs. Checks: decode(encode(x)) == x, ids of sampled rows vs
the reference (oracle/_ref encode_batch), and the device time."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_11941_b200 as bb
from oracle.oracle import Reference
t = bb.load_merge_table_files("tests/golden/gpt2.bbpt", None, "binary")
ref = Reference.from_arrays(*t.export())
rng = np.random.default_rng(7)
N = 256 << 20
cases = {
    "random_bytes_256B_rows": (rng.integers(0, 256, N, dtype=np.uint8), 256),
    "runs_a_64KiB_rows": (np.full(N, ord("a"), np.uint8), 65536),
    "digits_4KiB_rows": (rng.integers(ord("0"), ord("9") + 1, N, dtype=np.uint8), 4096),
}
enc = bb.Encoder(0)
for name, (data, L) in cases.items():
    off = np.arange(0, N + 1, L, dtype=np.uint64)
    ids, oo, st = enc.encode_packed(t, data, off)
    d, bo = enc.decode_packed(t, ids, oo)
    assert np.array_equal(np.asarray(d), data), name
    for r in rng.integers(0, off.size - 1, 3):
        s = slice(int(off[r]), int(off[r + 1]))
        w, wo = ref.encode_batch(data[s], np.array([0, L], np.uint64), workers=8)
        assert ids[int(oo[r]):int(oo[r + 1])].tolist() == w.tolist(), (name, int(r))
    dd = torch.from_numpy(data).cuda(); do = torch.from_numpy(off.view(np.int64)).cuda()
    di = torch.empty(N, dtype=torch.int32, device="cuda"); doo = torch.empty(off.size, dtype=torch.int64, device="cuda")
    for _ in range(2):
        enc.encode_device(t, dd.data_ptr(), do.data_ptr(), off.size - 1, N, di.data_ptr(), doo.data_ptr())
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        enc.encode_device(t, dd.data_ptr(), do.data_ptr(), off.size - 1, N, di.data_ptr(), doo.data_ptr())
    e1.record(); torch.cuda.synchronize()
    print(name, "tokens", int(oo[-1]), "device ms", round(e0.elapsed_time(e1) / 3, 2), "ok", flush=True)
