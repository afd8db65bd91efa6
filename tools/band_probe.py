"""Throughput of a BandGroup (virtual row bands on one GPU, wall clock; development probe).

    python tools/band_probe.py L n_bands kmcs mcs
"""
import sys, time, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2508_16639_b200 as e
from paper_2508_16639_b200.bands import BandGroup
import torch
L = int(sys.argv[1]); nb = int(sys.argv[2]); k = int(sys.argv[3]); mcs = int(sys.argv[4])
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10**9)
with BandGroup(p, e.make_circulant(3, [1]), nb, kmcs=k) as g:
    g.init_lattice(); g.advance(2); torch.cuda.synchronize()
    t = time.perf_counter(); g.advance(mcs); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(json.dumps({"L": L, "bands": nb, "kmcs": k, "mcs": mcs, "s": dt, "attempts_per_s": L * L * mcs / dt, "fmt": os.environ.get("ESCG_DRAW_FORMAT", "auto")}))
