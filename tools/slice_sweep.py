"""Sweep the bit-sliced kernel's launch geometry at one lattice size (development tool).

    python tools/slice_sweep.py L [lpi ...]
Prints one JSON line per (lanes per item, MCS per launch, split) with attempts/s.
"""
import json
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402


def run(L, n_mcs, lpi, k, split):
    os.environ["ESCG_DRAW_FORMAT"] = "sliced"
    os.environ["ESCG_SLICE_LPI"] = str(lpi)
    os.environ["ESCG_BLOCK_K"] = str(k)
    if split:
        os.environ["ESCG_SLICE_SPLIT"] = split
    else:
        os.environ.pop("ESCG_SLICE_SPLIT", None)
    p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
    with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
        eng.init_lattice()
        eng.advance(8)
        best = 0.0
        for _ in range(2):
            eng.advance(n_mcs)
            ms, _ = eng.last_timing()
            best = max(best, L * L * n_mcs / (ms / 1e3))
        d = eng.describe()
    return dict(L=L, lpi=lpi, k=d["kmcs"], split=split, ctas=d["ctas"], smem=d["smem_bytes"], attempts_per_s=best)


if __name__ == "__main__":
    L = int(sys.argv[1])
    lpis = [int(a) for a in sys.argv[2:]] or [1, 2]
    GL = L // 128
    n = 200 if L <= 4096 else 10
    splits = [None]
    for nbx in range(1, GL + 1):
        gw = -(-GL // nbx) + 1
        if gw > 17 or (nbx > 1 and -(-GL // (nbx - 1)) + 1 == gw):
            continue
        nby = max(1, 148 // nbx)
        splits.append("%d,%d" % (nby, nbx))
    for lpi in lpis:
        for k in (1, 2, 3, 4):
            for sp in splits:
                try:
                    print(json.dumps(run(L, n, lpi, k, sp)), flush=True)
                except Exception as ex:  # noqa: BLE001
                    print(json.dumps(dict(L=L, lpi=lpi, k=k, split=sp, error=str(ex))), flush=True)
