"""Small runs of every kernel, each checked bit for bit against the oracle — under a checked build
(ESCG_CHECKED: device asserts on window rows/columns, queue and mailbox slots, snapshot rows) since
compute-sanitizer is closed on this pool:

    ESCG_LIB=tools/_checked.so python tools/sanitize_cases.py all
cases: tile, block, block_seam, block_reflect, slice, slice_qcap, slice_lpi2, ring, ring_stop, all
Each case runs a few MCS on a small lattice through the C ABI and checks the result against the oracle
(so a sanitizer-perturbed schedule would also show as a mismatch)."""
import os
import sys

import numpy as np

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2508_16639_b200 as e  # noqa: E402
from pyoracle import Oracle  # noqa: E402

O = Oracle()


def run(L, H, M, kernel, mcs=3, env=None, S=3, flux=True, seed=11):
    for k, v in (env or {}).items():
        os.environ[k] = v
    model = e.make_circulant(3, [1]) if S == 3 else e.make_rpsls()
    p = e.SimParams(length=L, height=H, species=S, mobility=M, empty_prob=0.1, seed=seed, mcs_limit=mcs, flux=flux)
    with e.DeviceEngine(p, model, kernel=kernel) as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        eng.run(mcs, interval=1)
        got = eng.get_lattice()
        code = eng.draw_code()
        d = eng.describe()
    want = O.crs_run(init, L, H, model.matrix(), M, seed, 0, mcs, narrow=code, flux=flux)
    ok = np.array_equal(got, want)
    print("%-14s %s %dx%d M=%g: %s" % (sys.argv[1], d["kernel"], L, H, M, "bit-exact" if ok else "MISMATCH"))
    for k in (env or {}):
        del os.environ[k]
    assert ok


CASES = {
    "tile": lambda: run(64, 64, 1e-3, "tile"),
    "block": lambda: run(256, 128, 1e-3, "block"),
    "block_seam": lambda: run(66, 50, 1e-3, "block"),
    "block_reflect": lambda: run(96, 64, 1e-3, "block", flux=False),
    "slice": lambda: run(512, 96, 1e-2, "block", env={"ESCG_DRAW_FORMAT": "sliced"}),
    "slice_qcap": lambda: run(512, 96, 1e-2, "block", env={"ESCG_DRAW_FORMAT": "sliced", "ESCG_SLICE_QCAP": "1"}),
    "slice_lpi2": lambda: run(512, 96, 1e-2, "block", env={"ESCG_DRAW_FORMAT": "sliced", "ESCG_SLICE_LPI": "2"}),
    "ring": lambda: run(1024, 128, 1e-2, "ring", env={"ESCG_DRAW_FORMAT": "sliced"}),
    "ring_stop": lambda: run(1024, 64, 1e-2, "ring", mcs=4, env={"ESCG_DRAW_FORMAT": "sliced", "ESCG_RING_NB": "2"}),
}

if __name__ == "__main__":
    names = list(CASES) if sys.argv[1] == "all" else [sys.argv[1]]
    for n in names:
        sys.argv[1] = n
        CASES[n]()
