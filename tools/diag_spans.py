"""Per-launch timeline of the block kernel from %globaltimer stamps (diagnostic build, ESCG_DIAG_TIMING):
first CTA start, first CTA past griddepcontrol.wait, last CTA end — launch period vs kernel span."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_16639_b200 as e  # noqa: E402
from paper_2508_16639_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
lib = _lib.lib()
lib.escg_diag_spans.argtypes = [C.c_void_p, C.c_int]
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
    eng.init_lattice()
    eng.advance(10)
    lib.escg_diag_spans(None, 1)
    eng.advance(n)
    ms, launches = eng.last_timing()
    buf = np.zeros(256 * 3, np.uint64)
    lib.escg_diag_spans(buf.ctypes.data, 0)
k = eng.describe()["kmcs"] if False else None
s = buf.reshape(256, 3).astype(np.float64)
valid = s[(s[:, 0] < 1.8e19) & (s[:, 2] > 0)]
valid = valid[np.argsort(valid[:, 1])]
span = (valid[:, 2] - valid[:, 1]) / 1e3
wait = (valid[:, 1] - valid[:, 0]) / 1e3
period = np.diff(valid[:, 1]) / 1e3
handoff = (valid[1:, 1] - valid[:-1, 2]) / 1e3
print("launches %d  event ms/launch %.2f us" % (len(valid), ms / launches * 1e3))
print("span (first past wait -> last end): median %.2f us" % np.median(span))
print("period (wait-to-wait):             median %.2f us" % np.median(period))
print("handoff (prev last end -> next first past wait): median %.2f us" % np.median(handoff))
print("early start before wait: median %.2f us" % np.median(wait))

# isolated launches: one 2-MCS advance at a time, synchronised in between
spans = []
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
    eng.init_lattice()
    eng.advance(10)
    for i in range(6):
        lib.escg_diag_spans(None, 1)
        eng.advance(2)
        lib.escg_diag_spans(buf.ctypes.data, 0)
        s = buf.reshape(256, 3).astype(np.float64)
        v = s[(s[:, 0] < 1.8e19) & (s[:, 2] > 0)]
        spans.append(float((v[:, 2] - v[:, 1]).max() / 1e3))
print("isolated launch span: %s us" % " ".join("%.1f" % x for x in spans))
