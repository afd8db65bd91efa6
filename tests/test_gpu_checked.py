"""Every kernel mode on small lattices under the checked build (tools/_checked.so, -DESCG_CHECKED:
device asserts on shared-memory window rows/columns, deferred-tile queue and ring-mailbox slots and
snapshot rows), each run bit-exact against the oracle.  compute-sanitizer is closed on the GPU pool,
so this (with the bit-exact parity suite) is the bounds/race evidence."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "_checked.so")


def test_all_kernels_under_device_bounds_asserts():
    if not os.path.exists(LIB):
        pytest.skip("tools/_checked.so not built (__graft_entry__.build builds it)")
    env = dict(os.environ, ESCG_LIB=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), "all"], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("bit-exact") == 9 and "MISMATCH" not in r.stdout
