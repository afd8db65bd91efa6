"""Cost of MaxStep records on the ring kernel (L=3200): 900 MCS as advance (no records) vs run with
records every 9 MCS vs every 900."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402

p = e.SimParams(length=3200, height=3200, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1])) as eng:
    eng.init_lattice()
    eng.advance(900)
    for name, f in (("advance", lambda m: eng.advance(900)), ("run/9", lambda m: eng.run(m + 900, interval=9, record_trace=False)),
                    ("run/900", lambda m: eng.run(m + 900, interval=900, record_trace=False))):
        ts = []
        for _ in range(5):
            f(eng.mcs())
            ts.append(eng.last_timing()[0])
        print("%-8s %.3f ms per 900 MCS (min of 5), %.3g attempts/s" % (name, min(ts), 3200 * 3200 * 900 / min(ts) * 1e3))
