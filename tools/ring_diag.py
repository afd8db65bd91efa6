"""Phase timeline of the ring kernel (csrc/ring.cu) from a diagnostic build (ESCG_DIAG_RING).

    python tools/ring_diag.py <lib.so built with -DESCG_DIAG_RING> [L]
Stamps (launch phases 800..831, every CTA < 160, every warp), clock64: 0 slab start, 1 draws done,
2 import done, 3 bit-parallel attempts done, 4 undecided-tile replay done, 5 words stored,
6 publish/snapshot done, 7 after the phase barrier; plus import poll rounds.  Prints medians
(cycles) per segment for the boundary warps (0: top, 1: bottom) and the interior warps, and the
phase period (cycles, CTA-local).
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
lib = _lib.lib()
fn = lib.escg_diag_ring
fn.argtypes = [C.c_void_p, C.c_int]
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="ring") as eng:
    eng.init_lattice()
    eng.advance(20)
    fn(None, 1)
    eng.advance(300)
    ms, _ = eng.last_timing()
    buf = np.zeros(160 * 32 * 8 * 8 + 160 * 32 + 160 * 32 * 4, np.int64)
    fn(buf.ctypes.data, 0)
    d_ = eng.describe()
print(d_, "advance(300): %.3f ms = %.2f us/MCS" % (ms, ms * 1e3 / 300))
polls = buf[160 * 32 * 8 * 8:160 * 32 * 8 * 8 + 160 * 32].view(np.int32).reshape(160, 32, 2)
gt = buf[160 * 32 * 8 * 8 + 160 * 32:].reshape(160, 32, 4)
d = buf[:160 * 32 * 8 * 8].reshape(160, 32, 8, 8)
nb = d_["ctas"]
d = d[:nb]
polls = polls[:nb]
per = np.diff(d[:, :, 0, 7].astype(np.float64), axis=1)
print("phase period (cycles): median %.0f  p10 %.0f  p90 %.0f  max %.0f" % (np.median(per), np.percentile(per, 10),
                                                                            np.percentile(per, 90), per.max()))
pv = polls[polls > 0]
print("import poll rounds: mean %.2f  p90 %.0f  max %d  (%d imports with data)" % (pv.mean(), np.percentile(pv, 90),
                                                                                  pv.max(), pv.size))
names = ["draws", "import", "attempts", "replay", "store", "publish", "barrier"]
for label, ws in (("warp0 (top)", [0]), ("warp1 (bottom)", [1]), ("interior", [2, 3, 4, 5])):
    segs, start = [], []
    for w in ws:
        x = d[:, 1:, w, :].astype(np.float64)
        prev = d[:, :-1, w, 7].astype(np.float64)
        ok = (x[..., 0] > 0) & (prev > 0)
        segs.append(np.diff(x, axis=-1)[ok])
        start.append((x[..., 0] - prev)[ok])
    s = np.concatenate(segs)
    st = np.concatenate(start)
    if len(s) == 0:
        continue
    print("%-15s start %6.0f | " % (label, np.median(st)) +
          " | ".join("%s %6.0f" % (n, np.median(s[:, i])) for i, n in enumerate(names)) +
          " | sum %6.0f (p90 %6.0f)" % (np.median(s.sum(1)), np.percentile(s.sum(1), 90)))

gt = gt[:nb].astype(np.float64)
# top import of band c at phase q waits for band c-1's bottom publish of phase q
lat_top = gt[:, :, 2] - np.roll(gt[:, :, 1], 1, axis=0)
lat_bot = gt[:, :, 3] - np.roll(gt[:, :, 0], -1, axis=0)
ok = (gt[:, :, 2] > 0) & (np.roll(gt[:, :, 1], 1, axis=0) > 0)
lt = np.concatenate([lat_top[ok], lat_bot[ok]])
print("publish -> import done (ns): median %.0f  p10 %.0f  p90 %.0f" % (np.median(lt), np.percentile(lt, 10), np.percentile(lt, 90)))
for w, nm in ((6, "producer top"), (7, "producer bottom")):
    x = d[:, :, w, :].astype(np.float64)
    ok = x[..., 0] > 0
    print("%-15s draws %6.0f | import %6.0f | phase period %6.0f" % (nm, np.median((x[..., 1] - x[..., 0])[ok]),
          np.median((x[..., 2] - x[..., 1])[ok]), np.median(np.diff(x[..., 0], axis=1)[ok[:, 1:] & ok[:, :-1]])))
