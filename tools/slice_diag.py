"""Per-warp phase timeline of the bit-sliced kernel from a diagnostic build (clock64 stamps).

    python tools/slice_diag.py <lib.so built with ESCG_DIAG_SLICE> [L]
Events per (warp, phase): 0 phase start, 1 draws done (first item), 2 exchanges done, 3 bulk done
(before barrier A), 4 after barrier A, 5 replay pass done, 6 after barrier B, 7 first replay done.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
os.environ["ESCG_LIB"] = os.path.abspath(sys.argv[1])
import paper_2508_16639_b200 as e  # noqa: E402
from paper_2508_16639_b200 import _lib  # noqa: E402

L = int(sys.argv[2]) if len(sys.argv) > 2 else 3200
os.environ["ESCG_DRAW_FORMAT"] = "sliced"
lib = _lib.lib()
fn = lib.escg_diag_slice
fn.argtypes = [C.c_void_p, C.c_int]
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
    eng.init_lattice()
    eng.advance(20)
    fn(None, 1)
    eng.advance(2)
    buf = np.zeros(4 * 16 * 8 * 8, np.int64)
    fn(buf.ctypes.data, 0)
    print(eng.describe())
d = buf.reshape(4, 16, 8, 8)
for cta in range(2):
    t0 = d[cta, 0, 0, 0]
    print("CTA", cta)
    for ph in range(8):
        rows = []
        for w in range(8):
            v = d[cta, w, ph]
            rows.append("w%d: %s" % (w, " ".join("%6d" % ((x - t0) if x else -1) for x in v[:8])))
        print(" phase", ph)
        print("   " + "\n   ".join(rows))
