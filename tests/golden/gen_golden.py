"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref/libescg_ref.so, built from
/root/reference/proj/src by oracle/Makefile).  Run in the build container (needs /root/reference at
build time only):

    python tests/golden/gen_golden.py            # kat/serial/rule/threshold fixtures (seconds)
    python tests/golden/gen_golden.py --stats    # + statistical ensembles (a few minutes, 8 procs)

The committed JSON files are what the tests (CPU and GPU box) read; /root/reference is never read at
test time.
"""
import json
import os
import sys
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Reference  # noqa: E402

_REF = None


def ref():
    global _REF
    if _REF is None:
        _REF = Reference()
    return _REF


def fnv1a64(cells):
    h = 1469598103934665603
    for v in np.asarray(cells, np.uint32).tolist():
        h = ((h ^ v) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def models():
    r = ref()
    return {
        "rps": r.circulant(3, [1]),
        "rpsls": r.circulant(5, [1, 2]),
        "ablated": r.rpsls_ablated(),
        "park8": r.park8(0.15, 0.75, 1.0),
    }


def gen_kat():
    r = ref()
    out = {}
    w = r.mt_raw(5489, 10000)
    out["mt19937_5489"] = {"first": int(w[0]), "10000th": int(w[-1]), "source": "SPEC.md:155,164"}
    out["seed_mix"] = [[s, k, int(r.lib.ref_seed_mix(s, k))] for s in (0, 1, 42, 5489, 2 ** 32 - 1) for k in (0, 1, 7)]
    out["stream_words"] = [{"seed": s, "count": c, "k": k, "words": r.stream_words(s, 8, count=c, k=k).tolist()}
                           for s in (1, 42, 7, 123456789012) for (c, k) in ((1, 0), (4, 2))]
    nb = []
    for (L, H, flux, arity) in [(4, 4, 1, 4), (4, 4, 0, 4), (5, 3, 1, 8), (5, 3, 0, 8), (2, 2, 1, 4), (2, 2, 0, 8)]:
        for i in range(L * H):
            for d in range(arity):
                nb.append([L, H, flux, arity, i, d, int(r.lib.ref_neighbor_index(i, d, arity, L, H, flux))])
    out["neighbor_index"] = nb
    out["align_num_randoms"] = [[a, b, int(r.lib.ref_align_num_randoms(a, b))] for (a, b) in
                                [(100000000, 40000), (100000000, 30000), (10, 3), (100000005, 90000), (5, 6),
                                 (100000000, 10240000), (100000000, 268435456)]]
    rates = []
    for (M, N) in [(3e-5, 160000), (1e-4, 40000), (3e-5, 10 ** 6), (1e-4, 3200 * 3200), (1e-4, 16384 ** 2), (0.0, 10 ** 4),
                   (1e-6, 40000)]:
        o = np.zeros(4)
        r.lib.ref_action_rates(M, N, o)
        rates.append([M, N, o.tolist()])
    out["action_rates"] = rates
    init = []
    for (L, H, S, p0, seed) in [(8, 8, 3, 0.0, 1), (10, 6, 5, 0.1, 42), (200, 200, 3, 0.0, 42), (16, 16, 8, 0.5, 3),
                                (6, 6, 3, 1.0, 9)]:
        c = r.init_lattice(L, H, S, p0, seed)
        init.append({"L": L, "H": H, "S": S, "p0": p0, "seed": seed, "first16": c[:16].tolist(), "fnv": fnv1a64(c)})
    out["init_lattice"] = init
    # Random123 Philox4x32-10 known-answer vectors (external; the device generator)
    out["philox4x32_10"] = [
        {"ctr": [0, 0, 0, 0], "key": [0, 0], "out": [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]},
        {"ctr": [0xffffffff] * 4, "key": [0xffffffff] * 2, "out": [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]},
        {"ctr": [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], "key": [0xa4093822, 0x299f31d0],
         "out": [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]},
    ]
    return out


SERIAL_CASES = [
    # L, H, mcs, seed, model, M, p0, arity, flux, tracked
    (8, 8, 10, 1, "rps", 1e-4, 0.0, 4, 1, 0),
    (50, 50, 100, 42, "rps", 1e-4, 0.1, 4, 1, 0),
    (64, 64, 200, 7, "rpsls", 3e-5, 0.0, 4, 1, 0),
    (40, 30, 60, 3, "ablated", 3e-3, 0.2, 8, 1, 4),
    (30, 22, 80, 11, "park8", 0.0, 0.0, 4, 0, 0),
    (21, 35, 50, 5, "rps", 1e-3, 0.1, 8, 0, 0),
    (12, 12, 400, 8, "rps", 5e-2, 0.3, 4, 1, 0),
]


def gen_serial():
    r = ref()
    ms = models()
    out = []
    for (L, H, mcs, seed, name, M, p0, arity, flux, tracked) in SERIAL_CASES:
        res = r.simulate(L, H, ms[name], M, p0, mcs, seed, mode=0, arity=arity, flux=bool(flux), tracked=tracked)
        out.append({"L": L, "H": H, "mcs": mcs, "seed": seed, "model": name, "M": M, "p0": p0, "arity": arity,
                    "flux": flux, "tracked": tracked, "status": res["status"], "n_records": int(res["n_records"]),
                    "final_counts": res["counts"][-1].tolist(), "record_steps_tail": res["steps"][-3:].tolist(),
                    "counts_at": {str(int(k)): res["counts"][k].tolist() for k in range(0, len(res["steps"]), max(1, len(res["steps"]) // 5))},
                    "fnv": fnv1a64(res["cells"])})
    return out


def gen_rule():
    """elementary_step outcomes (engine.hpp:108-141) for every (s, n) pair x direction x bucket edge."""
    r = ref()
    ms = models()
    rows = []
    for name, eps_N in [("rps", (1e-4, 40000)), ("park8", (0.0, 10000)), ("ablated", (3e-3, 10000))]:
        D = ms[name]
        S = D.shape[0]
        M, N = eps_N
        L = H = 4
        Meff = M * N / (L * H)
        # action words at every bucket / interaction edge (found by bisection on the reference's own
        # float/double expressions, mt19937.hpp:62 + engine.hpp:117-131) and their neighbours
        o = np.zeros(4)
        r.lib.ref_action_rates(Meff, L * H, o)
        mu, eps, total = o[0], o[2], o[3]

        def rr(x):
            return float(np.float32(np.float32(x) / np.float32(4294967295.0))) * total

        def edge(pred, lo=0, hi=2 ** 32):
            while lo < hi:
                mid = (lo + hi) // 2
                if pred(mid):
                    hi = mid
                else:
                    lo = mid + 1
            return lo

        xm = edge(lambda x: rr(x) >= eps)
        xi = edge(lambda x: rr(x) >= eps + mu)
        edges = {xm, xi}
        for dv in set(D.ravel().tolist()) - {0.0}:
            edges.add(edge(lambda x: (rr(x) - eps) / mu >= dv, xm, xi))
        words = sorted({w + k for w in edges for k in (-1, 0, 1) if 0 <= w + k < 2 ** 32} |
                       {0, 2 ** 31, 2 ** 32 - 1, (xm + xi) // 2})
        for s in range(S + 1):
            for n in range(S + 1):
                for d in (3, 0):
                    for x in words:
                        cells = np.zeros(16, np.int32)
                        cells[5] = s
                        nbi = int(r.lib.ref_neighbor_index(5, d, 4, L, H, 1))
                        cells[nbi] = n
                        act = np.float32(np.float32(x) / np.float32(4294967295.0))
                        rc = r.lib.ref_elementary_step(cells, L, H, S, 4, 1, np.ascontiguousarray(D.ravel()),
                                                       int(name == "park8"), Meff, 5, d, float(act))
                        rows.append([name, Meff, s, n, d, x, rc, int(cells[5]), int(cells[nbi])])
    return rows


# ---------------------------------------------------------------------------------------------
# Statistical ensembles (reference serial engine, MT19937): the distributions the GPU must match.
# ---------------------------------------------------------------------------------------------

def _ablated(seed):
    r = ref()
    res = r.simulate(200, 200, r.rpsls_ablated(), 3e-5, 0.0, 2000, seed, mode=0, tracked=4, want_cells=False)
    return int(res["steps"][-1]), res["status"]


def _probe(args):
    M, L, mcs, seed = args
    r = ref()
    res = r.simulate(L, L, r.circulant(3, [1]), M, 0.1, mcs, seed, mode=0, want_cells=False)
    last = res["counts"][-1]
    return int(np.sum(last[1:] > 0)), res["status"], int(res["steps"][-1])


def _traj(args):
    name, L, M, p0, mcs, seed, every = args
    r = ref()
    D = r.circulant(3, [1]) if name == "rps" else r.circulant(5, [1, 2])
    res = r.simulate(L, L, D, M, p0, mcs, seed, mode=0, want_cells=False)
    idx = list(range(0, len(res["steps"]), every))
    return [res["counts"][i].tolist() for i in idx], res["steps"][idx].tolist()


def _traj_lh(args):
    L, H, M, p0, mcs, seed, every = args
    r = ref()
    res = r.simulate(L, H, r.circulant(3, [1]), M, p0, mcs, seed, mode=0, want_cells=False)
    idx = list(range(0, len(res["steps"]), every))
    return [res["counts"][i].tolist() for i in idx], res["steps"][idx].tolist()


def gen_stats_seam(out):
    """Ensembles on periodic lattices whose sides are not divisible by 4 (device seam schedule)."""
    with Pool(8) as pool:
        for (L, H) in [(50, 50), (51, 45)]:
            tr = pool.map(_traj_lh, [(L, H, 1e-3, 0.1, 300, 4000 + s, 50) for s in range(64)])
            out["rps_L%dx%d_traj" % (L, H)] = {
                "desc": "RPS %dx%d periodic M=1e-3 p0=0.1: counts every 50 MCS to 300" % (L, H),
                "counts": [t[0] for t in tr], "steps": tr[0][1]}
    return out


def _park(seed):
    r = ref()
    res = r.simulate(100, 100, r.park8(0.15, 0.75, 1.0), 0.0, 0.0, 1000, seed, mode=0, want_cells=False)
    return res["counts"][-1].tolist()


def gen_stats():
    out = {}
    with Pool(8) as pool:
        seeds = list(range(1, 65))
        out["ablated_rpsls_L200"] = {
            "desc": "run_ablated_rpsls(200, ...) semantics: Paper (4) extinction MCS, reference serial engine",
            "seeds": seeds, "results": pool.map(_ablated, seeds)}
        probe = {}
        for M in (1e-4, 3e-4, 1e-3, 3e-3):
            args = [(M, 100, 3000, 1000 + s) for s in range(48)]
            probe[str(M)] = pool.map(_probe, args)
        out["coexistence_L100_3000mcs"] = {"desc": "RPS L=100 p0=0.1 3000 MCS: (alive species, status, last mcs)",
                                           "by_M": probe}
        tr = pool.map(_traj, [("rps", 200, 1e-4, 0.1, 600, 2000 + s, 100) for s in range(32)])
        out["rps_L200_traj"] = {"desc": "C1 config (RPS L=200 M=1e-4 p0=0.1): counts every 100 MCS to 600",
                                "counts": [t[0] for t in tr], "steps": tr[0][1]}
        tr = pool.map(_traj, [("rpsls", 200, 3e-5, 0.0, 400, 3000 + s, 100) for s in range(32)])
        out["rpsls_L200_traj"] = {"desc": "RPSLS L=200 M=3e-5 p0=0: counts every 100 MCS to 400",
                                  "counts": [t[0] for t in tr], "steps": tr[0][1]}
        out["park8_L100_1000"] = {"desc": "park8(0.15,0.75,1) L=100 M=0 1000 MCS final counts",
                                  "counts": pool.map(_park, list(range(1, 25)))}
    return out


# ---------------------------------------------------------------------------------------------
# Round-2 ensembles: the regimes the fast kernels run in (bit-sliced: P(migration) >= 0.996; byte
# block kernel below), with a spatial observable, and the C4 mobility sweep
# ---------------------------------------------------------------------------------------------

def _traj_corr(args):
    L, M, p0, mcs, seed, every = args
    import stats_ref

    r = ref()
    res = r.simulate(L, L, r.circulant(3, [1]), M, p0, mcs, seed, mode=0, want_cells=True)
    idx = list(range(0, len(res["steps"]), every))
    return ([res["counts"][i].tolist() for i in idx], res["steps"][idx].tolist(), res["status"],
            stats_ref.correlation_length(res["cells"], L, L))


C4_GRID = [1e-4, 2e-4, 3e-4, 4.5e-4, 6e-4, 8e-4, 1e-3, 1.5e-3, 3e-3]
C4_SEEDS = {100: 64, 200: 64, 300: 32, 400: 32}


def gen_stats2():
    out = {}
    with Pool(8) as pool:
        for key, L, M, mcs, nseed, s0 in (("rps_L512_M1e-3", 512, 1e-3, 2000, 64, 5000),
                                           ("rps_L1024_M3e-4", 1024, 3e-4, 1500, 48, 6000),
                                           ("rps_L1024_M3e-5", 1024, 3e-5, 1500, 48, 7000)):
            res = pool.map(_traj_corr, [(L, M, 0.1, mcs, s0 + s, 100) for s in range(nseed)])
            out[key] = {"desc": "RPS L=%d M=%g p0=0.1, reference serial engine: counts every 100 MCS to %d, final "
                                "status and correlation length (oracle/stats_ref.py)" % (L, M, mcs),
                        "steps": res[0][1], "counts": [r_[0] for r_ in res], "status": [r_[2] for r_ in res],
                        "corr_len": [r_[3] for r_ in res]}
            print("done", key, flush=True)
        c4 = {}
        for L, nseed in C4_SEEDS.items():
            by_m = {}
            for i, M in enumerate(C4_GRID):
                by_m[str(M)] = pool.map(_probe, [(M, L, 10000, 100000 + 1000 * i + L + s) for s in range(nseed)])
            c4[str(L)] = by_m
            print("done C4 L=%d" % L, flush=True)
        out["c4_sweep_1e4mcs"] = {"desc": "C4: RPS L in 100..400, p0=0.1, 1e4 MCS, reference serial engine: "
                                          "(alive species, status, last mcs) per seed", "grid": C4_GRID, "by_L": c4}
    return out


def gen_stats3():
    """C1 at its own length: RPS L=200, M=1e-4, p0=0.1 to 1e4 MCS, 64 reference seeds."""
    out = {}
    with Pool(8) as pool:
        L, M, mcs, nseed, s0 = 200, 1e-4, 10000, 64, 8000
        res = pool.map(_traj_corr, [(L, M, 0.1, mcs, s0 + s, 500) for s in range(nseed)])
        out["rps_L200_M1e-4_1e4"] = {"desc": "C1: RPS L=200 M=1e-4 p0=0.1, reference serial engine: counts every "
                                             "500 MCS to 1e4, final status and correlation length",
                                     "steps": res[0][1], "counts": [r_[0] for r_ in res],
                                     "status": [r_[2] for r_ in res], "corr_len": [r_[3] for r_ in res]}
    return out


if __name__ == "__main__":
    def dump(name, obj):
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(obj, f, separators=(",", ":"))
        print("wrote", name)

    dump("kat.json", gen_kat())
    dump("serial.json", gen_serial())
    dump("rule.json", gen_rule())
    if "--stats3" in sys.argv:
        dump("stats3.json", gen_stats3())
        sys.exit(0)
    if "--stats2" in sys.argv:
        dump("stats2.json", gen_stats2())
        sys.exit(0)
    if "--stats" in sys.argv:
        dump("stats.json", gen_stats_seam(gen_stats()))
    elif "--stats-seam" in sys.argv:
        dump("stats.json", gen_stats_seam(json.load(open(os.path.join(HERE, "stats.json")))))
