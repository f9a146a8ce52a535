"""The opt-in LU variants are bitwise equal to the default row-block LU (k_lu_solve).

Each variant is switched on by an environment variable read once per process, so the check
runs tools/lu_rank2_check.py, which steps cfg1, cfg2, cfg2 n_q = 31 and n_q = 64 for 3
fixed-iteration steps in a fresh process per variant and compares the states bitwise.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("switch", ["NLROM_LU_LA", "NLROM_LU_RANK2"])
def test_lu_variant_bitwise(switch):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "lu_rank2_check.py"), switch],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    lines = [l for l in out.splitlines() if l.strip()]
    assert len(lines) == 4, out
    assert all(l.endswith("bitwise") for l in lines), out
