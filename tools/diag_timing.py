"""Per-section timing of the block kernel from %globaltimer stamps (diagnostic build)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_16639_b200 as e  # noqa: E402
from paper_2508_16639_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
    eng.init_lattice()
    eng.advance(50)
    d = eng.describe()
    buf = np.zeros(4096 * 16, np.uint64)
    lib = _lib.lib()
    lib.escg_diag_timing.argtypes = [C.c_void_p, C.c_int]
    lib.escg_diag_timing(buf.ctypes.data, buf.size)
    ms, n = eng.last_timing()
    print(d, "ms/launch %.2f us" % (ms / n * 1e3))
    ctas = d["ctas"]
    t = buf.reshape(4096, 16)[:ctas].astype(np.int64)
    t0 = t[:, 0].min()
    names = ["start", "load_issued", "load_done", "ph0", "ph1", "ph2", "ph3", "-", "counted", "end"]
    for s in [0, 1, 2, 3, 4, 5, 6, 8, 9]:
        rel = (t[:, s] - t0) / 1e3
        print("%-12s min %7.2f  median %7.2f  max %7.2f us" % (names[s], rel.min(), np.median(rel), rel.max()))
    wb = np.zeros(8 * 32 * 16, np.uint64)
    lib.escg_diag_warps.argtypes = [C.c_void_p, C.c_int]
    lib.escg_diag_warps(wb.ctypes.data, wb.size)
    w = wb.reshape(8, 32, 16).astype(np.int64)
    for c in range(2):
        base = t[c, 2]  # load_done of that CTA
        print("CTA %d per-phase warp finish times (us after load): " % c)
        prev = base
        for q in range(4 * d["kmcs"]):
            col = w[c, :, q]
            if col.max() == 0:
                break
            rel = (col - prev) / 1e3
            print("  phase %d: warp work min %.2f median %.2f max %.2f us" % (q, rel.min(), np.median(rel), rel.max()))
            prev = col.max()
