"""Multi-process plumbing of bench.py's N-GPU mode, on CPU with gloo
(world_size 2, 127.0.0.1): per-rank deterministic shards, no data-path
collective, max-over-ranks timing, whole-job token totals."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Args:
    def __init__(self, **kw):
        self.__dict__.update(dict(config=2, text="zipf", table="wordlevel", merges=200000, scale=1 / 4096), **kw)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import paper_2507_11941_b200 as bb
    w = bench.Workload(_Args(), rank, world)
    data, off = w.rows()
    # Each rank's shard is its own (weak scaling): seeds differ per rank.
    digest = int(np.frombuffer(data.tobytes()[:4096], np.uint8).astype(np.int64).sum())
    # cfg5 (strong scaling): ONE corpus, contiguous shards from the encoder's partitioner.
    w5 = bench.Workload(_Args(config=5, scale=1 / 20000), rank, world)
    corpus = w5.corpus_offsets()
    bounds = bb.partition(corpus, world).astype(np.int64)
    d5, o5 = w5.rows(bounds)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # what bench.allreduce does (nccl on GPU)
    n = torch.tensor([off.size - 1, o5.size - 1, int(o5[-1])], dtype=torch.int64)
    dist.all_reduce(n)
    q.put((rank, digest, float(t.item()), n.tolist(), int(corpus.size - 1), int(corpus[-1]), w5.scaling))
    dist.destroy_process_group()


def test_two_rank_gloo_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] != res[1][1]                 # distinct shards
    assert res[0][2] == res[1][2] == 2.0          # max over ranks
    assert res[0][3][0] == 2 * 256                # whole-job row count (weak scaling)
    rows5, bytes5 = res[0][4], res[0][5]
    assert res[0][3][1:] == [rows5, bytes5]       # cfg5 shards partition the one corpus
    assert res[0][6] == "strong"


def test_bench_rank_count_must_match(monkeypatch):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    monkeypatch.setenv("WORLD_SIZE", "1")
    with pytest.raises(SystemExit, match="--gpus 2 but 1 rank"):
        bench.dist_init(_Args(gpus=2))


def test_partition_shards_cover_rows():
    import paper_2507_11941_b200 as bb
    off = np.arange(0, 1001, dtype=np.uint64) * np.uint64(7)
    b = bb.partition(off, 8)
    assert b[0] == 0 and b[-1] == 1000
    sizes = np.diff(b.astype(np.int64))
    assert sizes.max() - sizes.min() <= 1


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2507_11941_b200 as bb
    # rank r holds rows of lengths r+1, r+2, ... (rank 1's shard has an empty row)
    rng = np.random.default_rng(rank)
    lens = [0, 3, 5] if rank == 1 else [2, 4]
    ids = torch.tensor(rng.integers(0, 50000, sum(lens)), dtype=torch.int32)
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64)
    got = bb.gather_csr(ids, off, dst=0)
    q.put((rank, None if got is None else (got[0].tolist(), got[1].tolist()), ids.tolist(), off.tolist()))
    dist.destroy_process_group()


def test_gather_csr_two_ranks_gloo():
    """The optional gather-to-one-GPU epilogue (bb.gather_csr): rank order,
    rebased offsets, empty rows kept; nothing on the non-destination rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, got, ids0, off0), (_, none, ids1, off1) = res
    assert none is None
    assert got[0] == ids0 + ids1
    assert got[1] == off0 + [o + len(ids0) for o in off1[1:]]
