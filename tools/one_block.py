"""Run a few block-kernel MCS at L=3200 (profiling target)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kernel = sys.argv[3] if len(sys.argv) > 3 else "block"  # or "auto"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), n_replicas=reps, kernel=kernel) as eng:
    eng.init_lattice()
    eng.advance(n)
    ms, launches = eng.last_timing()
    print("L=%d kernel=%s mcs=%d ms=%.3f attempts/s=%.3e" % (L, kernel, n, ms, L * L * n * reps / ms * 1e3))
