#!/usr/bin/env python3
"""Batch-encode benchmark (BASELINE.json metric) -- one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Workload (BASELINE.json configs[1], the high-batch config): 2^20 synthetic
256-byte ASCII rows per GPU, GPT-2 table (50,000 merges). A step encodes the
whole batch to CSR token ids + row offsets. Weak scaling: every rank encodes
its own 2^20-row batch (different seed); rows are independent so there is no
collective on the data path; ranks only barrier and max-reduce their timings.

value     device-resident throughput (tokens/s over all ranks): bytes + offsets
          already in HBM, CUDA events around K steps on the encode stream,
          max over ranks. Inputs (256 MiB) exceed the 126 MB L2.
e2e       same metric through the public host API (bbpe_encode) from pinned
          host memory: H2D of the bytes+offsets, encode, D2H of ids+offsets,
          every step (pipelined waves).
roofline  k_pieces (the dominant kernel): algorithmic bytes per launch =
          input bytes + 4 x tokens + 16 x rows / its average
          CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs; traffic =
          DRAM bytes of one launch from profiles/r1_k_pieces_cfg<N>.json.
cpu_baseline  the unmodified reference encode_batch (oracle/_ref, block engine,
          PhasePool over all host cores) on a bounded sample of the same rows;
          heap_engine: the reference's heap_bpe over PhasePool::run_items.
decode / epilogue / jsonl  the §8f device paths on the step's output: decode
          back to bytes (round trip checked), padded BatchEncoding, JSON-lines.
merge_only  memo and dedupe off: every piece through the merge passes.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
METRIC = "batch-encode tokens/sec and input GB/s at 1/2/4/8 B200 vs CPU ref (host cores)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every
    2 ms (the timed region is tens of ms), nvidia-smi every 200 ms without it."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = "nvml"
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))  # ~50 ms: once
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

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nv:
                    nv, h = self._nv, self._h
                    self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), self._max,
                                         int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
                else:
                    self.samples.append(self._sample_smi())
            except Exception:
                pass
            self._stop.wait(0.002 if self._nv else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for s in self.samples for n, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


def load_table(cfg):
    """GPT-2 (50,000 merges) for configs 1, 2, 3, 5; config 4 extends it to
    200,000 consistent word-level merges (paper_2507_11941_b200.synth.extend_table)."""
    from paper_2507_11941_b200 import load_merge_table_files, synth
    gpt2 = load_merge_table_files(os.path.join(GOLDEN, "gpt2.bbpt"), None, "binary")
    if cfg == 4:
        t, _ = synth.extend_table(gpt2, 200000)
        return t, "gpt2 extended to 200,000 merges (synth.extend_table, seed 4)"
    return gpt2, "gpt2 (50,000 merges)"


def make_rows(table, cfg, rank, scale):
    from paper_2507_11941_b200 import synth
    gen = synth.TextGen(synth.word_list(table))
    return synth.config_rows(gen, cfg, scale=scale, seed=cfg * 1000 + rank)


def dist_init(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return rank, world, local


def barrier_max(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reference_arm(args, rank, world):
    """Times the reference's own CPU implementation (oracle/_ref encode_batch,
    block engine, PhasePool(nproc)) on a bounded sample of our arm's workload."""
    if rank != 0:
        return
    from oracle.oracle import Reference
    table, table_desc = load_table(args.config)
    data, offsets, desc = make_rows(table, args.config, 0, args.scale)
    ids_, off_, blob_, m4_ = table.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    cores = os.cpu_count() or 1
    n_all = offsets.size - 1
    # Sample size: ~args.ref_seconds of CPU work per step (calibrated).
    n = min(n_all, 2048)
    t0 = time.perf_counter()
    ref.encode_batch(data, offsets[: n + 1], workers=cores)
    dt = time.perf_counter() - t0
    n = int(min(n_all, max(n, n * args.ref_seconds / max(dt, 1e-3))))
    sub_off = offsets[: n + 1]
    for _ in range(args.warmup):
        ref.encode_batch(data, sub_off, workers=cores)
    times, toks = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ids, oo = ref.encode_batch(data, sub_off, workers=cores)
        times.append(time.perf_counter() - t0)
        toks = int(oo[-1])
    t = float(np.median(times))
    v = toks / t
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"cfg{args.config}: {desc}", "table": table_desc,
                   "sample_rows": n, "sample_bytes": int(sub_off[-1])},
        "input_GBps": int(sub_off[-1]) / t / 1e9,
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "sample": f"first {n} of {n_all} rows ({int(sub_off[-1])} B), median of {args.steps}"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(table, data, offsets, seconds):
    from oracle.oracle import Reference
    cores = os.cpu_count() or 1
    ids_, off_, blob_, m4_ = table.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    n_all = offsets.size - 1
    n = min(n_all, 2048)
    ref.encode_batch(data, offsets[: n + 1], workers=cores)  # warm
    t0 = time.perf_counter()
    ref.encode_batch(data, offsets[: n + 1], workers=cores)
    dt = time.perf_counter() - t0
    n = int(min(n_all, max(n, n * seconds / max(dt, 1e-3))))
    t0 = time.perf_counter()
    ids, oo = ref.encode_batch(data, offsets[: n + 1], workers=cores)
    dt = time.perf_counter() - t0
    out = {"value": int(oo[-1]) / dt, "unit": "tokens/s", "cores": cores, "kind": "reference",
           "sample": f"first {n} of {n_all} rows ({int(offsets[n])} B), reference encode_batch "
                     f"(block engine, PhasePool({cores}))",
           "input_GBps": int(offsets[n]) / dt / 1e9}
    # The reference's fastest CPU engine too: heap_bpe per row
    # over PhasePool::run_items -- equal results on these rank-consistent tables.
    m = min(n_all, 4096)
    ref.encode_heap(data, offsets[: m + 1], workers=cores)
    t0 = time.perf_counter()
    ref.encode_heap(data, offsets[: m + 1], workers=cores)
    dt = time.perf_counter() - t0
    m = int(min(n_all, max(m, m * seconds / 2 / max(dt, 1e-3))))
    t0 = time.perf_counter()
    _, ho = ref.encode_heap(data, offsets[: m + 1], workers=cores)
    dt = time.perf_counter() - t0
    out["heap_engine"] = {"value": int(ho[-1]) / dt, "unit": "tokens/s", "cores": cores,
                          "sample": f"first {m} of {n_all} rows ({int(offsets[m])} B), reference heap_bpe "
                                    f"over PhasePool::run_items({cores})",
                          "input_GBps": int(offsets[m]) / dt / 1e9}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=None,
                    help="row-count scale (default 1; config 5 defaults to 1/8 = 2 GB per GPU)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", default="pieces", choices=["pieces", "block"])
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-merge-only", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else max(args.warmup, 1)
    if args.scale is None:
        args.scale = 1 / 8 if args.config == 5 else 1.0  # cfg5: 16 GB over 8 GPUs = 2 GB per GPU

    if args.impl == "reference":
        # CPU only, rank 0 alone: no process group (the other ranks exit 0 at once).
        reference_arm(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world, local = dist_init(args.gpus)

    import torch
    import paper_2507_11941_b200 as bb

    torch.cuda.set_device(local)
    table, table_desc = load_table(args.config)
    data, offsets, desc = make_rows(table, args.config, rank, args.scale)
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

    def step():
        enc.encode_device(table, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(),
                          d_oo.data_ptr(), stream=stream.cuda_stream, sync=False)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    enc.sync()
    enc.kernel_times(reset=True)
    launches0 = enc.kernel_launches()
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
        enc.sync()
        torch.cuda.synchronize()
    barrier(world)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    launches = enc.kernel_launches() - launches0
    ktimes, kcalls = enc.kernel_times(reset=True)
    ntok = int(d_oo[-1].item())
    ms = barrier_max(world, ms_local)
    tokens_all = ntok * world
    bytes_all = total * world
    value = tokens_all / (ms / 1e3)

    # ---- the same, merge passes only (piece memo off), for reference ----
    merge_only = None
    if args.engine == "pieces" and not args.no_merge_only:
        enc.set_config(piece_memo=False, dedup=False)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                step()
        enc.sync()
        enc.kernel_times(reset=True)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
        enc.sync()
        torch.cuda.synchronize()
        mo_ms = barrier_max(world, e0.elapsed_time(e1) / args.steps)
        kt, kc = enc.kernel_times(reset=True)
        assert int(d_oo[-1].item()) == ntok
        merge_only = {"value": tokens_all / (mo_ms / 1e3), "unit": "tokens/s", "ms_per_step": mo_ms,
                      "kernel_ms": {k: v / max(kc, 1) for k, v in kt.items()}}
        enc.set_config(piece_memo=True, dedup=True)

    # ---- device decode of the step's output, round-trip checked ----
    decode = None
    if args.engine == "pieces":
        d_back = torch.empty(max(total, 1), dtype=torch.uint8, device="cuda")
        d_boff = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        dec_args = (table, d_ids.data_ptr(), d_oo.data_ptr(), n, ntok, d_back.data_ptr(), total, d_boff.data_ptr())
        enc.decode_device(*dec_args)
        assert torch.equal(d_back[:total], d_data), "device decode did not invert the encode"
        times = []
        for _ in range(max(3, args.steps // 2)):
            t0 = time.perf_counter()
            enc.decode_device(*dec_args)
            times.append(time.perf_counter() - t0)
        d_ms = float(np.median(times)) * 1e3
        decode = {"ms_per_step": d_ms, "output_GBps": total / (d_ms / 1e3) / 1e9,
                  "tokens_per_s": ntok / (d_ms / 1e3), "timing": "wall clock of the synchronous call",
                  "round_trip": "bit-exact"}

    # ---- device padded BatchEncoding of the step's output ----
    epilogue = None
    if args.engine == "pieces":
        import ctypes as C
        from paper_2507_11941_b200._lib import LIB
        w = C.c_uint64()
        assert LIB.bbpe_batch_widest_device(enc.handle, C.c_void_p(d_oo.data_ptr()), n, 0, 0, C.byref(w)) == 0
        L = int(w.value)
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
        times = []
        for _ in range(max(3, args.steps // 2)):
            t0 = time.perf_counter()
            pad()
            times.append(time.perf_counter() - t0)
        p_ms = float(np.median(times)) * 1e3
        epilogue = {"ms_per_step": p_ms, "max_len": L, "output_GBps": n * L * 5 / (p_ms / 1e3) / 1e9,
                    "timing": "wall clock of the synchronous call (widest row not included)"}

    # ---- JSON-lines text of the step's output on the device ----
    jsonl = None
    if args.engine == "pieces":
        cap = enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), n, ntok, 0, 0)
        j_out = torch.empty(max(cap, 1), dtype=torch.uint8, device="cuda")
        times = []
        for _ in range(max(3, args.steps // 2)):
            t0 = time.perf_counter()
            assert enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), n, ntok, j_out.data_ptr(), cap) == cap
            times.append(time.perf_counter() - t0)
        j_ms = float(np.median(times)) * 1e3
        jsonl = {"ms_per_step": j_ms, "text_bytes": cap, "output_GBps": cap / (j_ms / 1e3) / 1e9,
                 "timing": "wall clock of the synchronous call"}
        del j_out

    # ---- gpt2 split pattern mode (encode_reference pattern mode) ----
    pattern = None
    if args.engine == "pieces":
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

    # ---- special tokens + BOS on the device (bbpe_encode_batch_device) ----
    specials_line = None
    if args.engine == "pieces" and args.config == 2 and n and total == 256 * n:
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

    # ---- roofline of the dominant kernel ----
    k_ms = {k: v / max(kcalls, 1) for k, v in ktimes.items()}
    dom = max(k_ms, key=k_ms.get)
    # Per launch: a device batch above 2 GiB runs as several chunk launches.
    per_step = max(kcalls, 1) / max(args.steps, 1)
    alg_bytes = (total + 4 * ntok + 16 * n) / per_step
    peak, peak_src = peaks()
    achieved = alg_bytes / (k_ms["k_pieces"] / 1e3) / 1e9
    # DRAM traffic of the same kernel on the same command, from the committed
    # ncu --set full capture (profiles/<round>_k_pieces_cfg<N>.json), if any.
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"r1_k_pieces_cfg{args.config}.json")
    if os.path.exists(prof) and args.scale == 1.0 and args.engine == "pieces":
        with open(prof) as f:
            traffic = json.load(f).get("traffic_bytes")

    # ---- end to end through the host API (pinned host buffers) ----
    e2e = None
    if not args.no_e2e:
        h_data = torch.from_numpy(data).pin_memory()
        h_off = torch.from_numpy(offsets.view(np.int64)).pin_memory()
        h_ids = torch.empty(max(total, 1), dtype=torch.int32).pin_memory()
        h_oo = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        hd, ho = h_data.numpy(), h_off.numpy().view(np.uint64)
        hi, hoo = h_ids.numpy().view(np.uint32), h_oo.numpy().view(np.uint64)
        # Warm-up by time as well as count: after the device-only legs the PCIe
        # link needs sustained traffic before copies run at full rate.
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
        e_ms = barrier_max(world, float(np.median(times)) * 1e3)
        e2e = {"value": tokens_all / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": total + (n + 1) * 8, "d2h_bytes_per_step": ntok * 4 + (n + 1) * 8,
               "input_GBps": bytes_all / (e_ms / 1e3) / 1e9}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(table, data, offsets, 10.0)
        except Exception as ex:  # reference not built on this box
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"cfg{args.config}: {desc} per GPU (Zipf words of the table)",
                       "table": table_desc, "engine": args.engine,
                       "parallelism": f"rows sharded, {world} independent GPU(s), no collective",
                       "l2": "inputs (%d MiB) larger than L2" % (total >> 20)},
            "input_GBps": bytes_all / (ms / 1e3) / 1e9,
            "tokens_per_step": tokens_all,
            "gpu_launches": launches,
            "kernel_ms": k_ms,
            "roofline": {"bound": "hbm", "kernel": "k_pieces", "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                         "dominant_kernel": dom},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "merge_only": merge_only,
            "decode": decode,
            "epilogue": epilogue,
            "jsonl": jsonl,
            "pattern_mode": pattern,
            "specials_mode": specials_line,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
