"""Quick device-throughput probe (development tool; bench.py is the contract)."""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402


def probe(L, n_mcs, kernel="auto", reps=1, M=1e-4, p0=0.1, S=3):
    model = e.make_circulant(3, [1]) if S == 3 else e.make_rpsls()
    p = e.SimParams(length=L, height=L, species=S, mobility=M, empty_prob=p0, seed=1, mcs_limit=10 ** 9)
    with e.DeviceEngine(p, model, n_replicas=reps, kernel=kernel) as eng:
        eng.init_lattice()
        eng.advance(3)
        t0 = time.time()
        eng.advance(n_mcs)
        wall = time.time() - t0
        ms, launches = eng.last_timing()
        d = eng.describe()
    att = L * L * n_mcs * reps / (ms / 1e3)
    return dict(L=L, reps=reps, fmt=d["draw_format"], kernel=d["kernel"], ctas=d["ctas"], smem=d["smem_bytes"], mcs=n_mcs, ms=ms,
                wall_ms=wall * 1e3, launches=launches, attempts_per_s=att, mcs_per_s=n_mcs / (ms / 1e3),
                hbm_frac=att * 2 / 6537.3e9)


if __name__ == "__main__":
    out = []
    for args in [(3200, 200, "block"), (1000, 200, "block"), (16384, 10, "block"), (200, 500, "tile", 1),
                 (200, 200, "tile", 296), (100, 500, "tile", 1184), (400, 100, "tile", 148)]:
        r = probe(*args)
        print(json.dumps(r), flush=True)
        out.append(r)
