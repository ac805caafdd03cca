"""Shared fixtures. GPU tests are marked @pytest.mark.gpu and need a CUDA device."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2507_11941_b200", "libbbpe_b200.so")
    orc = os.path.join(ROOT, "oracle", "libbpe_oracle.so")
    if not os.path.exists(lib) or not os.path.exists(orc):
        import __graft_entry__
        __graft_entry__.build()


_ensure_built()


def has_gpu():
    try:
        import paper_2507_11941_b200._lib as L
        import ctypes
        n = ctypes.c_int(0)
        return L.LIB.bbpe_device_count(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpt2():
    from paper_2507_11941_b200 import load_merge_table_files
    return load_merge_table_files(os.path.join(GOLDEN, "gpt2.bbpt"), None, "binary")


@pytest.fixture(scope="session")
def toy_tables():
    with open(os.path.join(GOLDEN, "toy_tables.json")) as f:
        return json.load(f)


def table_from_json(t):
    from paper_2507_11941_b200 import MergeTable
    return MergeTable.build([(i, bytes(b)) for i, b in t["tokens"]], [tuple(m) for m in t["merges"]])


def extend_table(table, total_merges):
    """(MergeTable, arrays) of `table` extended by word-level merges
    (workloads.tables.extend_wordlevel) to `total_merges` merges."""
    from paper_2507_11941_b200 import MergeTable
    from workloads.tables import arrays, extend_wordlevel
    ids, off, blob, m4 = table.export()
    raw = blob.tobytes()
    toks = {int(i): raw[int(off[k]):int(off[k + 1])] for k, i in enumerate(ids)}
    t, m = extend_wordlevel(toks, [tuple(int(x) for x in r) for r in m4], total_merges)
    arrs = arrays(t, m)
    return MergeTable.from_arrays(*arrs), arrs


def arrays_from_json(t):
    toks = sorted((i, bytes(b)) for i, b in t["tokens"])
    ids = np.array([x[0] for x in toks], np.uint32)
    off = np.zeros(len(toks) + 1, np.uint64)
    np.cumsum([len(x[1]) for x in toks], out=off[1:])
    blob = np.frombuffer(b"".join(x[1] for x in toks), np.uint8)
    return ids, off, blob, np.array(t["merges"], np.uint32).reshape(-1, 4)


def load_vectors(name):
    z = np.load(os.path.join(GOLDEN, f"vectors_{name}.npz"))
    return {k: z[k] for k in z.files}


VECTOR_SETS = ["gpt2_random", "gpt2_text", "gpt2_adversarial", "toy8_exhaustive", "inconsistent",
               "random0", "random1", "random2", "random3", "doubling"]


@pytest.fixture(scope="session")
def oracle_for():
    """name -> CRestatement for the named table (gpt2 or a toy table)."""
    from oracle.oracle import CRestatement
    cache = {}
    with open(os.path.join(GOLDEN, "toy_tables.json")) as f:
        toys = json.load(f)

    def get(name):
        if name not in cache:
            if name == "gpt2":
                from paper_2507_11941_b200 import load_merge_table_files
                t = load_merge_table_files(os.path.join(GOLDEN, "gpt2.bbpt"), None, "binary")
                _, _, _, m4 = t.export()
                cache[name] = CRestatement(m4, [t.byte_token(b) for b in range(256)])
            else:
                ids, off, blob, m4 = arrays_from_json(toys[name])
                bt = [0xFFFFFFFF] * 256
                for k, i in enumerate(ids):
                    if off[k + 1] - off[k] == 1:
                        bt[blob[off[k]]] = int(i)
                cache[name] = CRestatement(m4, bt)
        return cache[name]
    return get
