"""C2 (RPSLS L=1000, M=3e-5, p0=0) single lattice: one advance (profiling target for the byte block kernel)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = e.SimParams(length=1000, height=1000, species=5, mobility=3e-5, empty_prob=0.0, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_rpsls()) as eng:
    eng.init_lattice()
    eng.advance(n)
    ms, launches = eng.last_timing()
    print(eng.describe(), "mcs=%d ms=%.3f launches=%d attempts/s=%.3e" % (n, ms, launches, 1e6 * n / ms * 1e3))
