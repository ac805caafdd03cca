#!/usr/bin/env python3
"""Batch-encode benchmark (BASELINE.json metric) -- one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5]
                  [--text zipf|corpus|mixed] [--table wordlevel|trained]
                  [--engine pieces|block] [--impl ours|reference]

Default workload: BASELINE.json configs[1] (cfg2), the config the metric is
quoted on at 1/2/4/8 GPUs: 2^20 synthetic 256-byte rows per GPU, GPT-2 table
(50,000 merges), weak scaling (every rank encodes its own 2^20 rows, seed
per rank; no collective on the data path). --config 5 is ONE 16 GB corpus
cut into contiguous cost-balanced shards by the encoder's partitioner
(bbpe_partition), one per rank: strong scaling. With --gpus N > 1 and no
torchrun environment the script relaunches itself under torchrun; a rank
count different from --gpus is an error.

value     device-resident throughput (tokens/s over all ranks): bytes + offsets
          already in HBM, CUDA events around K steps on the encode stream,
          max over ranks; inputs larger than L2 (else L2 flushed between steps).
e2e       the same metric through the public host API (bbpe_encode) from pinned
          host memory: H2D of bytes + offsets, encode, D2H of ids + offsets,
          every step (pipelined waves); median call time, max over ranks.
parity    after the timed region, the step's whole CSR output against the
          compiled reference (oracle/_ref): encode_batch (block engine, the
          drop-in target) on every row when that fits the time budget, else
          heap_bpe on every row (equal to block on these rank-consistent
          tables; any row where heap differs is re-checked with the block
          engine) plus encode_batch on a deterministic row sample.
roofline  the dominant kernel (largest CUDA-event time): algorithmic bytes per
          launch (input bytes + 4 x tokens + 16 x rows) / its
          average duration, against MEASURED_PEAKS.json; `step_frac` is the
          same bytes over the whole step. traffic = DRAM bytes of that kernel
          per launch from the committed ncu capture, when there is one.
workloads (default line, one GPU) other DESIGN §5 workloads measured the same
          way, each with its own parity: the paper's block-engine configuration
          on this line's rows, cfg2-shaped mixed text, and cfg4 with the §8d
          trained 200k-merge table (--no-workload-legs skips them).
cpu_baseline  the unmodified reference encode_batch (oracle/_ref, block engine,
          PhasePool over all host cores) on a bounded sample of the same rows
          (+ its heap_bpe engine).
--impl reference  the reference's own CPU encoder on the same workload: table
          loaded by the reference's load_merge_table_files, rows from
          workloads/ (no import of the B200 package), rank 0 only.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import tables as WT  # noqa: E402  (no product import)
from workloads import text as WX  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
METRIC = "batch-encode tokens/sec and input GB/s at 1/2/4/8 B200 vs CPU ref (host cores)"
L2_BYTES = 126 << 20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every
    2 ms, nvidia-smi every 200 ms without it."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = "nvml"
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None
            self.source = "nvidia-smi"

    def _sample_smi(self):
        f = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + f, "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        v = [x.strip() for x in out.split(",")]
        mask = sum(bit for bit, x in zip(self.REASONS.values(), v[2:6]) if x == "Active")
        return float(v[0]), float(v[1]), mask

    def _sample(self):
        try:
            if self._nv:
                nv, h = self._nv, self._h
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), self._max,
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            else:
                self.samples.append(self._sample_smi())
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.002 if self._nv else 0.2)

    def __enter__(self):
        # A short timed region (cfg2: ~15 ms) is mostly Python enqueueing that
        # holds the GIL: a shorter switch interval lets the sampler run.
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(0.0002)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for s in self.samples for n, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


# ---------------------------------------------------------------------------
# Workload (shared by both arms; nothing here imports the B200 package)


class Workload:
    """Table files + rows of one rank for the chosen config / text class."""

    def __init__(self, args, rank: int, world: int):
        self.args = args
        self.tmp = tempfile.mkdtemp(prefix="bbpe_bench_")
        tokens, merges = WT.gpt2_table()
        self.table_desc = "gpt2 (50,000 merges; tests/golden/gpt2/vocab.json + merges.txt)"
        self.files = (WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
        if args.config == 4:
            if args.table == "trained":
                from workloads.train import trained_table
                tokens, merges, how = trained_table(tokens, merges, args.merges)
                self.table_desc = f"gpt2 continued to {len(merges):,} merges: {how}"
            else:
                tokens, merges = WT.extend_wordlevel(tokens, merges, args.merges)
                self.table_desc = (f"gpt2 extended to {len(merges):,} merges (workloads.tables.extend_wordlevel, "
                                   "word-internal merges, seed 4)")
            path = WT.write_canonical(os.path.join(self.tmp, "cfg4.json"), tokens, merges)
            self.files = (path, None, "json")
        self.tokens = tokens
        self.merges = merges
        corpus = open(os.path.join(GOLDEN, "corpus.txt"), "rb").read() if args.text == "corpus" else None
        # the trained table's text is the GPT-2 Zipf text it was trained on (other seed)
        words_from = WT.gpt2_table()[0] if (args.config == 4 and args.table == "trained") else tokens
        self.gen = WX.make_gen(args.text, words_from, corpus)
        self.rank, self.world = rank, world

    def rows(self, bounds=None):
        a = self.args
        if a.config == 5:  # ONE corpus, this rank's shard (strong scaling)
            data, off, desc, rr, _ = WX.cfg5_shard(self.gen, a.scale, self.world, self.rank, bounds=bounds)
            self.scaling = "strong"
            self.desc = (f"cfg5: one {16 * a.scale:g} GB corpus, logU[128 B, 64 KiB] rows, contiguous "
                         f"cost-balanced shards over {self.world} GPU(s)")
            self.shard = desc
            return data, off
        data, off, desc = WX.config_rows(self.gen, a.config, scale=a.scale, seed=a.config * 1000 + self.rank)
        self.scaling = "weak"
        self.desc = f"cfg{a.config}: {desc} per GPU"
        self.shard = None
        return data, off

    def corpus_offsets(self):
        rng = np.random.default_rng(1000 + 5)
        L = WX.cfg5_lengths(self.args.scale, rng)
        off = np.zeros(L.size + 1, np.uint64)
        np.cumsum(L.astype(np.uint64), out=off[1:])
        return off

    def config(self):
        return {"workload": self.desc, "table": self.table_desc, "text": TEXT_DESC[self.args.text],
                "l2": L2_NOTE}


TEXT_DESC = {
    "zipf": "zipf: words drawn Zipf(1.1) from the table's ' [a-z]{2,}' tokens, 3% numbers, punctuation (SURVEY §8d)",
    "corpus": "corpus: the reference bench's tests/testdata/corpus.txt cut as ingest_corpus does",
    "mixed": "mixed: random-letter words, long numbers, hex, code identifiers/punctuation, CJK and Cyrillic",
}
L2_NOTE = "inputs larger than L2 (126 MB), else L2 flushed between steps"


# ---------------------------------------------------------------------------
# Distributed plumbing


def profile_tag(args):
    """Name of a workload in profiles/ (r2_<kernel>_<tag>.json ncu summaries)."""
    tag = f"cfg{args.config}_{args.text}"
    if args.config == 4 and args.table == "trained":
        tag += "_trained"
    if args.engine == "block":
        tag += "_block"
    return tag


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """--gpus N > 1 outside torchrun: relaunch as N ranks (one per GPU)."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but {world} rank(s) were launched")
    if world > 1:
        import torch
        import torch.distributed as dist
        if SHARED_GPU:  # test mode: every rank on GPU 0, gloo for the barriers and the max over ranks
            local = 0
            dist.init_process_group("gloo")
            return rank, world, local
        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} GPU(s) visible")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return rank, world, local


# BBPE_BENCH_SHARED_GPU=1: run the N-rank path with every rank on device 0
# (checks the sharding, aggregation and reporting of --gpus N on a one-GPU
# box; the numbers are not a scaling measurement and the line says so).
SHARED_GPU = os.environ.get("BBPE_BENCH_SHARED_GPU") == "1"


def allreduce(world, value, op="max"):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device="cpu" if SHARED_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# Reference side (oracle/_ref: the unmodified reference headers, compiled)


def reference_table(w: Workload):
    from oracle.oracle import Reference
    vocab, merges, fmt = w.files
    return Reference.load_files(vocab, merges, canonical=(fmt == "json"))


def calibrate(fn, offsets, seconds, n0=2048):
    """Largest row prefix that fn encodes in about `seconds`."""
    n_all = offsets.size - 1
    n = min(n_all, n0)
    fn(offsets[: n + 1])
    t0 = time.perf_counter()
    fn(offsets[: n + 1])
    dt = time.perf_counter() - t0
    return int(min(n_all, max(n, n * seconds / max(dt, 1e-3))))


def reference_arm(args):
    """The reference's own CPU encoder (encode_batch, block engine, PhasePool
    over all host cores) on a bounded sample of our arm's workload."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    w = Workload(args, 0, args.gpus)
    ref = reference_table(w)
    data, offsets = w.rows()
    cores = os.cpu_count() or 1
    enc = lambda off: ref.encode_batch(data, off, workers=cores)  # noqa: E731
    n = calibrate(enc, offsets, args.ref_seconds)
    sub = offsets[: n + 1]
    for _ in range(args.warmup):
        enc(sub)
    times, toks = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, oo = enc(sub)
        times.append(time.perf_counter() - t0)
        toks = int(oo[-1])
    t = float(np.median(times))
    v = toks / t
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": w.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": w.config(),
        "input_GBps": int(sub[-1]) / t / 1e9,
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "sample": f"first {n} of {offsets.size - 1} rows of rank 0's workload "
                                   f"({int(sub[-1])} B), median of {args.steps}; reference encode_batch "
                                   f"(block engine, PhasePool({cores}))"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "loaded": "oracle/_ref/libbbpe_ref.so only (table via the reference's load_merge_table_files)",
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(w: Workload, ref, data, offsets, seconds):
    cores = os.cpu_count() or 1
    n_all = offsets.size - 1
    enc = lambda off: ref.encode_batch(data, off, workers=cores)  # noqa: E731
    n = calibrate(enc, offsets, seconds)
    t0 = time.perf_counter()
    _, oo = enc(offsets[: n + 1])
    dt = time.perf_counter() - t0
    out = {"value": int(oo[-1]) / dt, "unit": "tokens/s", "cores": cores, "kind": "reference",
           "sample": f"first {n} of {n_all} rows ({int(offsets[n])} B), reference encode_batch "
                     f"(block engine, PhasePool({cores}))",
           "input_GBps": int(offsets[n]) / dt / 1e9}
    heap = lambda off: ref.encode_heap(data, off, workers=cores)  # noqa: E731
    m = calibrate(heap, offsets, seconds / 2, 4096)
    t0 = time.perf_counter()
    _, ho = heap(offsets[: m + 1])
    dt = time.perf_counter() - t0
    out["heap_engine"] = {"value": int(ho[-1]) / dt, "unit": "tokens/s", "cores": cores,
                          "sample": f"first {m} of {n_all} rows ({int(offsets[m])} B), reference heap_bpe "
                                    f"over PhasePool::run_items({cores})",
                          "input_GBps": int(offsets[m]) / dt / 1e9}
    return out


def csr_diff(ids_a, off_a, ids_b, off_b):
    """Indices of rows whose token lists differ (vectorised on the fast path)."""
    n = off_a.size - 1
    if off_a.size == off_b.size and np.array_equal(off_a, off_b) and np.array_equal(ids_a, ids_b):
        return []
    la, lb = np.diff(off_a.astype(np.int64)), np.diff(off_b.astype(np.int64))
    cand = np.nonzero(la != lb)[0].tolist()
    same = np.nonzero(la == lb)[0]
    # rows of equal length: compare their ids; positions where ids differ map to rows
    if same.size:
        rowid_a = np.repeat(np.arange(n), la)
        ok_len = np.repeat(la == lb, la)
        pos_a = np.nonzero(ok_len)[0]
        r_of = rowid_a[pos_a]
        pos_b = pos_a - off_a[r_of].astype(np.int64) + off_b[r_of].astype(np.int64)
        diff = ids_a[pos_a] != ids_b[pos_b]
        cand += np.unique(r_of[diff]).tolist()
    return sorted(set(cand))


def parity_check(ref, data, offsets, ids, oo, budget_s):
    """The step's whole CSR output vs the compiled reference (module doc)."""
    cores = os.cpu_count() or 1
    n = offsets.size - 1
    t0 = time.perf_counter()
    # Time estimate of the block engine on everything: a short calibration.
    m = min(n, 512)
    tc = time.perf_counter()
    ref.encode_batch(data, offsets[: m + 1], workers=cores)
    est = (time.perf_counter() - tc) * (float(offsets[-1]) / max(float(offsets[m]), 1.0))
    if est <= budget_s:
        wi, wo = ref.encode_batch(data, offsets, workers=cores)
        bad = csr_diff(ids, oo, wi, wo)
        out = {"rows_checked": n, "mismatches": len(bad), "tokens_checked": int(wo[-1]),
               "bytes_checked": int(offsets[-1]),
               "oracle": f"oracle/_ref encode_batch (block engine, the drop-in target) on every row, "
                         f"PhasePool({cores})"}
    else:
        hi, ho = ref.encode_heap(data, offsets, workers=cores)
        sus = csr_diff(ids, oo, hi, ho)
        # Rows where heap differs from the GPU: the block engine decides.
        bad = []
        for r in sus:
            sub_d = data[int(offsets[r]):int(offsets[r + 1])]
            bi, bo = ref.encode_batch(sub_d, np.array([0, sub_d.size], np.uint64), workers=1)
            if not np.array_equal(bi, ids[int(oo[r]):int(oo[r + 1])]):
                bad.append(r)
        # Block engine on a deterministic sample (every k-th row) within the budget.
        k = max(1, int(np.ceil(est / max(budget_s / 2, 1.0))))
        rows = np.arange(0, n, k)
        lens = np.diff(offsets.astype(np.int64))[rows]
        so = np.zeros(rows.size + 1, np.uint64)
        np.cumsum(lens.astype(np.uint64), out=so[1:])
        sd = np.concatenate([data[int(offsets[r]):int(offsets[r + 1])] for r in rows]) if rows.size else data[:0]
        bi, bo = ref.encode_batch(sd, so, workers=cores)
        gi = np.concatenate([ids[int(oo[r]):int(oo[r + 1])] for r in rows]) if rows.size else ids[:0]
        go = np.zeros(rows.size + 1, np.uint64)
        np.cumsum(np.diff(oo.astype(np.int64))[rows].astype(np.uint64), out=go[1:])
        bad_s = [int(rows[i]) for i in csr_diff(gi, go, bi, bo)]
        bad = sorted(set(bad) | set(bad_s))
        out = {"rows_checked": n, "mismatches": len(bad), "tokens_checked": int(ho[-1]),
               "bytes_checked": int(offsets[-1]),
               "oracle": f"oracle/_ref heap_bpe over PhasePool::run_items({cores}) on every row "
                         f"({len(sus)} row(s) where heap differed re-checked with the block engine), "
                         f"plus encode_batch (block engine) on every {k}-th row ({rows.size} rows)",
               "block_rows_checked": int(rows.size)}
    if bad:
        out["first_mismatch_rows"] = bad[:5]
    out["seconds"] = time.perf_counter() - t0
    return out


# ---------------------------------------------------------------------------
# Our arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--text", default="zipf", choices=["zipf", "corpus", "mixed"])
    ap.add_argument("--table", default="wordlevel", choices=["wordlevel", "trained"], help="cfg4 table")
    ap.add_argument("--merges", type=int, default=200000, help="cfg4 table size")
    ap.add_argument("--scale", type=float, default=1.0, help="row-count scale (cfg5: corpus size / 16 GB)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", default="pieces", choices=["pieces", "block"])
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--parity", default="full", choices=["full", "none"])
    ap.add_argument("--parity-budget", type=float, default=60.0, help="seconds of block-engine work for parity")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the §8f legs (decode, padding, JSONL, ...)")
    ap.add_argument("--no-workload-legs", action="store_true",
                    help="skip the other-workload legs of the default line (trained cfg4, block engine, mixed text)")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    maybe_spawn(args)
    if args.impl == "reference":
        # CPU only, rank 0 alone (the other ranks exit 0 at once).
        reference_arm(args)
        return
    rank, world, local = dist_init(args)

    import torch
    import paper_2507_11941_b200 as bb

    torch.cuda.set_device(local)
    w = Workload(args, rank, world)
    vocab, merges, fmt = w.files
    table = bb.load_merge_table_files(vocab, merges, fmt)
    bounds = None
    if args.config == 5:
        bounds = bb.partition(w.corpus_offsets(), world).astype(np.int64)
    data, offsets = w.rows(bounds)
    n = offsets.size - 1
    total = int(offsets[-1])
    enc = bb.Encoder(device=local, engine=args.engine)
    enc.prepare(table)

    # ---- device-resident timing ----
    d_data = torch.from_numpy(data).cuda()
    d_off = torch.from_numpy(offsets.view(np.int64)).cuda()
    d_ids = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    d_oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    stream = torch.cuda.Stream()
    flush = None
    if total < 2 * L2_BYTES:  # small inputs: flush L2 between steps (outside the kernels' events)
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    def step():
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(1)
        enc.encode_device(table, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(),
                          d_oo.data_ptr(), stream=stream.cuda_stream, sync=False)

    def timed(k):
        enc.sync()
        enc.kernel_times(reset=True)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fl_ms = 0.0
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(k):
                step()
            e1.record(stream)
        enc.sync()
        torch.cuda.synchronize()
        if flush is not None:  # the flush is not encode time: measure it alone and subtract
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                f0.record(stream)
                for _ in range(k):
                    flush.fill_(1)
                f1.record(stream)
            torch.cuda.synchronize()
            fl_ms = f0.elapsed_time(f1)
        return (e0.elapsed_time(e1) - fl_ms) / k

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    enc.sync()
    launches0 = enc.kernel_launches()
    stats0 = enc.piece_stats(reset=True) if hasattr(enc, "piece_stats") else None
    with ClockSampler(local) as clocks:
        ms_local = timed(args.steps)
    barrier(world)
    launches = enc.kernel_launches() - launches0
    ktimes, kcalls = enc.kernel_times(reset=True)
    pstats = enc.piece_stats(reset=True) if stats0 is not None else None
    ntok = int(d_oo[-1].item())
    ms = allreduce(world, ms_local, "max")
    tokens_all = int(allreduce(world, ntok, "sum"))
    bytes_all = int(allreduce(world, total, "sum"))
    rows_all = int(allreduce(world, n, "sum"))
    value = tokens_all / (ms / 1e3)

    ids_h = d_ids[:ntok].cpu().numpy().view(np.uint32)
    oo_h = d_oo.cpu().numpy().view(np.uint64)

    # ---- end to end through the host API (pinned host buffers), right after
    # the device timing and before the CPU-heavy legs ----
    e2e = None
    if not args.no_e2e:
        h_data = torch.from_numpy(data).pin_memory()
        h_off = torch.from_numpy(offsets.view(np.int64)).pin_memory()
        h_ids = torch.empty(max(total, 1), dtype=torch.int32).pin_memory()
        h_oo = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        hd, ho = h_data.numpy(), h_off.numpy().view(np.uint64)
        hi, hoo = h_ids.numpy().view(np.uint32), h_oo.numpy().view(np.uint64)
        tw, k = time.perf_counter(), 0
        while k < max(5, args.warmup) or time.perf_counter() - tw < 0.5:
            enc.encode_packed(table, hd, ho, hi, hoo)
            k += 1
        barrier(world)
        times = []
        for _ in range(max(10, args.steps)):
            t0 = time.perf_counter()
            enc.encode_packed(table, hd, ho, hi, hoo)
            times.append(time.perf_counter() - t0)
        assert np.array_equal(hoo, oo_h) and np.array_equal(hi[:ntok], ids_h), "e2e output differs from device"
        e_ms = allreduce(world, float(np.median(times)) * 1e3, "max")
        e2e = {"value": tokens_all / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(allreduce(world, total + (n + 1) * 8, "sum")),
               "d2h_bytes_per_step": int(allreduce(world, ntok * 4 + (n + 1) * 8, "sum")),
               "input_GBps": bytes_all / (e_ms / 1e3) / 1e9,
               "timing": "median wall time of bbpe_encode (pinned host in, pinned host out), max over ranks"}
        del h_data, h_off, h_ids, h_oo

    # ---- parity: the step's whole output vs the compiled reference ----
    parity = None
    ref = None
    try:
        ref = reference_table(w)
    except Exception as ex:  # oracle/_ref missing on this box
        parity = {"rows_checked": 0, "mismatches": None, "oracle": f"unavailable: {ex}"}
    if ref is not None and args.parity == "full":
        parity = parity_check(ref, data, offsets, ids_h, oo_h, args.parity_budget)
        tot = {k: int(allreduce(world, parity[k], "sum")) for k in ("rows_checked", "mismatches", "bytes_checked")}
        parity.update(tot)

    # ---- merge passes only (piece memo and dedupe off) ----
    extras = args.engine == "pieces" and not args.no_extras and args.config == 2
    merge_only = None
    if args.engine == "pieces" and not args.no_extras:
        enc.set_config(piece_memo=False, dedup=False)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                step()
        mo_ms = allreduce(world, timed(args.steps), "max")
        kt, kc = enc.kernel_times(reset=True)
        assert int(d_oo[-1].item()) == ntok
        merge_only = {"value": tokens_all / (mo_ms / 1e3), "unit": "tokens/s", "ms_per_step": mo_ms,
                      "kernel_ms": {k: v / max(kc, 1) for k, v in kt.items()}}
        enc.set_config(piece_memo=True, dedup=True)

    decode = epilogue = jsonl = pattern = specials_line = None
    workloads = None
    if extras and world == 1 and not args.no_workload_legs:
        workloads = workload_legs(args, bb, torch, stream, table, d_data, d_off, ids_h, oo_h, n, total)
    if extras:
        decode, epilogue, jsonl, pattern, specials_line = extra_legs(args, bb, enc, table, torch, stream, step,
                                                                     d_data, d_off, d_ids, d_oo, n, total, ntok)

    # ---- roofline of the dominant kernel ----
    k_ms = {k: v / max(kcalls, 1) for k, v in ktimes.items()}
    dom = max(k_ms, key=k_ms.get)
    per_step = max(kcalls, 1) / max(args.steps, 1)  # >1 when a device batch runs as 2 GiB chunks
    alg_bytes = (total + 4 * ntok + 16 * n) / per_step
    peak, peak_src = peaks()
    achieved = alg_bytes / (k_ms[dom] / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"r2_{dom}_{profile_tag(args)}.json")
    if os.path.exists(prof) and args.scale == 1.0:
        with open(prof) as f:
            pj = json.load(f)
        if pj.get("engine", "pieces") == args.engine:
            traffic = pj.get("traffic_bytes")

    cpu = None
    if rank == 0 and ref is not None and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, ref, data, offsets, args.ref_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": w.scaling,
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": dict(w.config(), l2=(f"inputs ({total / 2**20:.0f} MiB per GPU) larger than L2 (126 MB): "
                                           "no flush" if flush is None else
                                           f"inputs ({total / 2**20:.1f} MiB) smaller than 2x L2: a 252 MB buffer "
                                           "written before every step, its time measured alone and subtracted")),
            "engine": args.engine,
            "parallelism": (f"rows sharded, {world} independent GPU(s), no collective on the data path" if not SHARED_GPU
                            else f"TEST MODE: {world} ranks sharing GPU 0 (BBPE_BENCH_SHARED_GPU), not a scaling number"),
            "input_GBps": bytes_all / (ms / 1e3) / 1e9,
            "tokens_per_step": tokens_all, "rows_per_step": rows_all, "bytes_per_step": bytes_all,
            "gpu_launches": launches,
            "kernel_ms": k_ms,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes,
                         "step_frac": (total + 4 * ntok + 16 * n) / (ms_local / 1e3) / 1e9 / peak},
            "parity": parity,
            "pieces": pstats,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "merge_only": merge_only,
            "decode": decode, "epilogue": epilogue, "jsonl": jsonl, "pattern_mode": pattern,
            "specials_mode": specials_line,
            "workloads": workloads,
            "clocks": clocks.summary(),
        }
        if w.shard:
            line["shard_rank0"] = w.shard
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def device_leg(bb, torch, table, data, offsets, engine, steps, warmup=2):
    """Device-resident encode of one batch: (ms per step, tokens, ids, offsets,
    per-kernel ms, piece stats), CUDA events on the encode stream."""
    n, total = offsets.size - 1, int(offsets[-1])
    enc = bb.Encoder(device=torch.cuda.current_device(), engine=engine)
    enc.prepare(table)
    dd = torch.from_numpy(data).cuda()
    do = torch.from_numpy(offsets.view(np.int64)).cuda()
    di = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    doo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()

    def run():
        enc.encode_device(table, dd.data_ptr(), do.data_ptr(), n, total, di.data_ptr(), doo.data_ptr(),
                          stream=st.cuda_stream, sync=False)
    for _ in range(warmup):
        run()
    enc.sync()
    enc.kernel_times(reset=True)
    enc.piece_stats(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(steps):
            run()
        e1.record(st)
    enc.sync()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    kt, kc = enc.kernel_times(reset=True)
    ps = enc.piece_stats(reset=True)
    ntok = int(doo[-1].item())
    ids = di[:ntok].cpu().numpy().view(np.uint32)
    oo = doo.cpu().numpy().view(np.uint64)
    return ms, ntok, ids, oo, {k: v / max(kc, 1) for k, v in kt.items()}, ps


def workload_legs(args, bb, torch, stream, table, d_data, d_off, ids_h, oo_h, n, total):
    """Other workloads of DESIGN §5, measured in the default line so the driver
    sees them (device-resident, CUDA events, every row checked):
      * block_engine_cfg2: the paper's configuration (BBPE_ENGINE_BLOCK, every
        row one piece) on this line's cfg2 rows; checked equal to the pieces
        engine's output, which `parity` checked against the reference;
      * mixed_text_cfg2: cfg2 shape, text the piece memo has not seen;
      * trained_cfg4: cfg4 with SURVEY §8d's trained 200k-merge table (merges
        cross words: every row is one long piece)."""
    from oracle.oracle import Reference
    out = {}
    peak, _ = peaks()

    def line(name, desc, ms, ntok, rows, nbytes, km, ps, par):
        dom = max(km, key=km.get)
        out[name] = {"workload": desc, "ms_per_step": ms, "tokens_per_s": ntok / (ms / 1e3),
                     "input_GBps": nbytes / (ms / 1e3) / 1e9, "dominant_kernel": dom,
                     "roofline_frac": (nbytes + 4 * ntok + 16 * rows) / (km[dom] / 1e3) / 1e9 / peak,
                     "kernel_ms": km, "pieces": ps, "parity": par}

    data = d_data.cpu().numpy()
    offs = d_off.cpu().numpy().view(np.uint64)
    ms, ntok, ids, oo, km, ps = device_leg(bb, torch, table, data, offs, "block", max(3, args.steps // 4))
    same = bool(np.array_equal(oo, oo_h) and np.array_equal(ids, ids_h))
    line("block_engine_cfg2", "cfg2 rows, --engine block (BBPE_ENGINE_BLOCK: every row one piece)", ms, ntok, n,
         total, km, ps, {"rows_checked": n, "mismatches": 0 if same else None,
                         "oracle": "equal to the pieces engine's output on every row (checked by `parity`)"})
    assert same, "block engine differs from the pieces engine"

    gen = WX.make_gen("mixed", None)
    md, mo, _ = WX.config_rows(gen, 2, seed=2002)
    ms, ntok, ids, oo, km, ps = device_leg(bb, torch, table, md, mo, "pieces", max(3, args.steps // 2))
    ref = Reference.load_files(WT.GPT2_VOCAB, WT.GPT2_MERGES)
    line("mixed_text_cfg2", f"{mo.size - 1} x 256 B, {TEXT_DESC['mixed']}", ms, ntok, mo.size - 1, int(mo[-1]), km, ps,
         parity_check(ref, md, mo, ids, oo, 30.0))

    from workloads.train import trained_table
    tokens, merges, how = trained_table(*WT.gpt2_table(), 200000)
    tdir = tempfile.mkdtemp(prefix="bbpe_trained_")
    path = WT.write_canonical(os.path.join(tdir, "cfg4_trained.json"), tokens, merges)
    ttable = bb.load_merge_table_files(path, None, "json")
    td, to, desc = WX.config_rows(WX.TextGen(WX.word_list(WT.gpt2_table()[0])), 4)
    ms, ntok, ids, oo, km, ps = device_leg(bb, torch, ttable, td, to, "pieces", 3)
    tref = Reference.load_files(path, None, canonical=True)
    line("trained_cfg4", f"cfg4: {desc}, table: {how}", ms, ntok, to.size - 1, int(to[-1]), km, ps,
         parity_check(tref, td, to, ids, oo, 20.0))
    return out


def extra_legs(args, bb, enc, table, torch, stream, step, d_data, d_off, d_ids, d_oo, n, total, ntok):
    """The §8f device paths on the step's output (cfg2): decode (round trip
    checked), padded BatchEncoding, JSON lines, gpt2 pattern mode, specials."""
    import ctypes as C
    from paper_2507_11941_b200._lib import LIB

    def wall(fn, k):
        fn()
        times = []
        for _ in range(k):
            t0 = time.perf_counter()
            fn()
            times.append(time.perf_counter() - t0)
        return float(np.median(times)) * 1e3

    d_back = torch.empty(max(total, 1), dtype=torch.uint8, device="cuda")
    d_boff = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    dec_args = (table, d_ids.data_ptr(), d_oo.data_ptr(), n, ntok, d_back.data_ptr(), total, d_boff.data_ptr())
    enc.decode_device(*dec_args)
    assert torch.equal(d_back[:total], d_data), "device decode did not invert the encode"
    d_ms = wall(lambda: enc.decode_device(*dec_args), max(3, args.steps // 2))
    decode = {"ms_per_step": d_ms, "output_GBps": total / (d_ms / 1e3) / 1e9, "tokens_per_s": ntok / (d_ms / 1e3),
              "timing": "wall clock of the synchronous call", "round_trip": "bit-exact"}
    del d_back, d_boff

    wd = C.c_uint64()
    assert LIB.bbpe_batch_widest_device(enc.handle, C.c_void_p(d_oo.data_ptr()), n, 0, 0, C.byref(wd)) == 0
    L = int(wd.value)
    p_ids = torch.empty(max(n * L, 1), dtype=torch.int32, device="cuda")
    p_mask = torch.empty(max(n * L, 1), dtype=torch.uint8, device="cuda")
    p_len = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    tr = C.c_uint64()

    def pad():
        assert LIB.bbpe_pad_device(enc.handle, C.c_void_p(d_ids.data_ptr()), C.c_void_p(d_oo.data_ptr()), n, 0,
                                   0xFFFFFFFF, 0xFFFFFFFF, L, C.c_void_p(p_ids.data_ptr()),
                                   C.c_void_p(p_len.data_ptr()), C.c_void_p(p_mask.data_ptr()), C.byref(tr)) == 0
    pad()
    assert int(p_len.sum().item()) == ntok
    p_ms = wall(pad, max(3, args.steps // 2))
    epilogue = {"ms_per_step": p_ms, "max_len": L, "output_GBps": n * L * 5 / (p_ms / 1e3) / 1e9,
                "timing": "wall clock of the synchronous call (widest row not included)"}
    del p_ids, p_mask, p_len

    cap = enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), n, ntok, 0, 0)
    j_out = torch.empty(max(cap, 1), dtype=torch.uint8, device="cuda")
    j_ms = wall(lambda: enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), n, ntok, j_out.data_ptr(), cap),
                max(3, args.steps // 2))
    jsonl = {"ms_per_step": j_ms, "text_bytes": cap, "output_GBps": cap / (j_ms / 1e3) / 1e9,
             "timing": "wall clock of the synchronous call"}
    del j_out

    enc.set_config(pattern="gpt2")
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    enc.sync()
    enc.kernel_times(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
    enc.sync()
    torch.cuda.synchronize()
    pt_ms = e0.elapsed_time(e1) / args.steps
    kt, kc = enc.kernel_times(reset=True)
    pattern = {"value": int(d_oo[-1].item()) / (pt_ms / 1e3), "unit": "tokens/s", "ms_per_step": pt_ms,
               "kernel_ms": {k: v / max(kc, 1) for k, v in kt.items()},
               "note": "k_tile_first includes the gpt2 splitter (k_pretok_rows + k_pretok_spans)"}
    enc.set_config(pattern=None)

    specials_line = None
    if total == 256 * n and n:
        sp = bb.SpecialTokenSet()
        sp.add("<|endoftext|>", 50256)
        d_sp = d_data.clone().view(n, 256)
        d_sp[:, -13:] = torch.tensor(list(b"<|endoftext|>"), dtype=torch.uint8, device="cuda")
        enc.set_specials(sp)
        cap = total + 2 * n
        d_sp_ids = torch.empty(cap, dtype=torch.int32, device="cuda")

        def sp_step():
            return enc.encode_batch_device(table, d_sp.data_ptr(), d_off.data_ptr(), n, total, d_sp_ids.data_ptr(),
                                           cap, d_oo.data_ptr(), bos_id=50256)
        for _ in range(args.warmup):
            sp_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            n_sp = sp_step()
        e1.record()
        torch.cuda.synchronize()
        sp_ms = e0.elapsed_time(e1) / args.steps
        specials_line = {"value": n_sp / (sp_ms / 1e3), "unit": "tokens/s", "ms_per_step": sp_ms,
                         "workload": "cfg2 rows ending in <|endoftext|> (a special), BOS added",
                         "timing": "CUDA events around synchronous calls (split, encode, stitch)"}
        enc.set_specials(None)
        del d_sp, d_sp_ids
    # leave d_oo holding the plain encode's offsets again
    step()
    enc.sync()
    return decode, epilogue, jsonl, pattern, specials_line


if __name__ == "__main__":
    main()
