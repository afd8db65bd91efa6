import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e
L = 3200
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1])) as eng:
    eng.init_lattice()
    eng.advance(20)
    for rep in range(3):
        t0 = time.perf_counter(); eng.advance(900); w = time.perf_counter() - t0
        print("advance 900: dev %.1f ms wall %.1f ms launches %d" % (*eng.last_timing()[:1], w * 1e3, eng.last_timing()[1]))
        for interval in (9, 900, 1):
            m = eng.mcs()
            t0 = time.perf_counter(); eng.run(m + 900, interval=interval, record_trace=False); w = time.perf_counter() - t0
            ms, n = eng.last_timing()
            print("run 900 interval %d: dev %.1f ms wall %.1f ms launches %d" % (interval, ms, w * 1e3, n))
