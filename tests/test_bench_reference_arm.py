"""bench.py --impl reference runs the reference's own CPU encoder without
loading anything from the B200 package (the driver's reference arm must not
map libbbpe_b200.so): checked on cfg1 on CPU."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle.oracle import Reference


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
def test_reference_arm_does_not_import_the_package():
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--config', '1', '--steps', '1', '--warmup', '1',"
            " '--ref-seconds', '0.2']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n"
            "bad = [m for m in sys.modules if m.startswith('paper_2507_11941_b200')]\n"
            "assert not bad, bad\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libbbpe_b200' not in maps and 'libbbpe_ref' in maps\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "tokens/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
