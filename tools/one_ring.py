"""One ring-kernel launch at L=3200 (100 MCS advance) for ncu captures: tools/ring_ncu.sh."""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel=os.environ.get("ESCG_ONE_KERNEL", "ring")) as eng:
    eng.init_lattice()
    eng.advance(n)
    ms, launches = eng.last_timing()
    print(eng.describe(), "%.3f ms for %d MCS: %.3g attempts/s" % (ms, n, L * L * n / (ms / 1e3)))
