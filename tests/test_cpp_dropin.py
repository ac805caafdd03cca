"""The C++ drop-in header (include/blockbpe_b200/blockbpe.hpp) compiles and
links against libbbpe_b200.so (CPU); its reference-mirroring checks run on the
GPU (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

EXE = os.path.join(ROOT, "build", "test_dropin")


def build_exe():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L" + os.path.join(ROOT, "paper_2507_11941_b200"),
           "-lbbpe_b200", "-Wl,-rpath," + os.path.join(ROOT, "paper_2507_11941_b200"), "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_dropin_header_compiles_and_links():
    build_exe()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    build_exe()
    r = subprocess.run([EXE, GOLDEN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
