"""The C-ABI library loads and exports every symbol include/bbpe_b200.h
declares; host-only entry points behave (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2507_11941_b200 as bb
from paper_2507_11941_b200 import _lib
from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bbpe_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bbpe_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = C.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_abi_version():
    assert _lib.LIB.bbpe_abi_version() == 2


def test_library_is_built_for_sm100a():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_partition_balances_cost():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 5000, 10000).astype(np.uint64)
    off = np.zeros(lens.size + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    for parts in (1, 2, 4, 8):
        b = bb.partition(off, parts)
        assert b[0] == 0 and b[-1] == lens.size and np.all(np.diff(b.astype(np.int64)) >= 0)
        cost = [(off[b[i + 1]] - off[b[i]]) + 64 * (b[i + 1] - b[i]) for i in range(parts)]
        total = sum(int(c) for c in cost)
        assert max(cost) <= total / parts + 5000 + 64


def test_bad_block_size_is_usage_error():
    with pytest.raises(bb.UsageError):
        bb.BlockConfig(48).validate()
    cfg = _lib.Config(48, 0, 0, 0, 1)
    h = C.c_void_p()
    assert _lib.LIB.bbpe_ctx_create(0, C.byref(cfg), C.byref(h)) == 1
    assert b"block_size" in _lib.LIB.bbpe_last_error()
    assert bb.coarsening_factor(2048, bb.BlockConfig(256)) == 8
    assert bb.coarsening_factor(1025, bb.BlockConfig(1024)) == 2


def test_header_is_plain_c99(tmp_path):
    """include/bbpe_b200.h is the FFI boundary for any language: it compiles as
    pedantic C99, links against libbbpe_b200.so and runs (no GPU call)."""
    import subprocess
    from conftest import ROOT
    src = tmp_path / "c_abi.c"
    src.write_text('#include "bbpe_b200.h"\n'
                   "int main(void) { bbpe_config c = {256, 0, BBPE_ENGINE_PIECES, 0, 1, 0, 0}; (void)c;\n"
                   "  return bbpe_abi_version() > 0 ? 0 : 1; }\n")
    lib = os.path.join(ROOT, "paper_2507_11941_b200")
    exe = tmp_path / "c_abi"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I" + os.path.join(ROOT, "include"),
                        str(src), "-L" + lib, "-lbbpe_b200", "-Wl,-rpath," + lib, "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0
