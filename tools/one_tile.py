"""Run a tile-kernel ensemble (profiling target): L, replicas, MCS."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 296
n = int(sys.argv[3]) if len(sys.argv) > 3 else 50
M = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-4
p = e.SimParams(length=L, height=L, species=3, mobility=M, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), n_replicas=reps, kernel="tile") as eng:
    eng.init_lattice()
    eng.advance(n)
    ms, launches = eng.last_timing()
    print("L=%d reps=%d mcs=%d ms=%.3f attempts/s=%.3e %s" % (L, reps, n, ms, L * L * n * reps / ms * 1e3, eng.describe()))
