"""Bit-sliced vs NARROW block kernel throughput probe (development tool; bench.py is the contract).

    python tools/slice_perf.py [L ...]
"""
import json
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402


def probe(L, n_mcs, fmt, M=1e-4, p0=0.1):
    os.environ["ESCG_DRAW_FORMAT"] = fmt
    model = e.make_circulant(3, [1])
    p = e.SimParams(length=L, height=L, species=3, mobility=M, empty_prob=p0, seed=1, mcs_limit=10 ** 9)
    with e.DeviceEngine(p, model, kernel="block") as eng:
        eng.init_lattice()
        eng.advance(8)
        eng.advance(n_mcs)
        ms, launches = eng.last_timing()
        d = eng.describe()
    att = L * L * n_mcs / (ms / 1e3)
    return dict(L=L, fmt=d["draw_format"], ctas=d["ctas"], kmcs=d["kmcs"], smem=d["smem_bytes"], mcs=n_mcs, ms=round(ms, 3),
                launches=launches, attempts_per_s=att, mcs_per_s=n_mcs / (ms / 1e3), hbm_frac=att * 2 / 6537.3e9)


if __name__ == "__main__":
    fmts = ("narrow", "sliced")
    args = sys.argv[1:]
    M = 1e-4
    while args and args[0].startswith("--"):
        a = args.pop(0)
        if a.startswith("--fmt="):
            fmts = (a[6:],)
        elif a.startswith("--M="):
            M = float(a[4:])
    Ls = [int(a) for a in args] or [3200, 16384]
    for L in Ls:
        n = 400 if L <= 4096 else 20
        for fmt in fmts:
            print(json.dumps(dict(probe(L, n, fmt, M=M), M=M)), flush=True)
