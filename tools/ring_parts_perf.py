"""Multi-part ring at L=3200 on one GPU (one launch over every part) vs the single-device ring:
the cost of the cross-part exchange (system-scope inbox words, flags, dual boundary writes).

    python tools/ring_parts_perf.py [L] [MCS]
"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402
from paper_2508_16639_b200.bands import RingGroup  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
model = e.make_circulant(3, [1])
with e.DeviceEngine(p, model, kernel="ring") as eng:
    eng.init_lattice()
    eng.advance(20)
    eng.advance(n)
    ms, _ = eng.last_timing()
    print("single ring  %3d CTAs: %.3f ms for %d MCS: %.3g attempts/s" % (eng.describe()["ctas"], ms, n, L * L * n / ms * 1e3))
for parts in (2, 4, 8):
    with RingGroup(p, model, parts) as grp:
        grp.init_lattice()
        grp.advance(20)
        grp.advance(n)
        ms = grp.last_ms()
        print("%d-part ring %3d CTAs: %.3f ms for %d MCS: %.3g attempts/s"
              % (parts, sum(grp.describe(i)["ctas"] for i in range(parts)), ms, n, L * L * n / ms * 1e3))
