"""Fraction of von Neumann neighbour pairs holding equal codes in the bench lattice (L=3200 RPS, M=1e-4)
after n MCS: an undecided bit-sliced attempt on an equal pair is a no-op (development tool)."""
import json
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2508_16639_b200 as e  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
    eng.init_lattice()
    done = 0
    for n in (0, 100, 1000, 5000, 20000):
        eng.advance(n - done)
        done = n
        a = np.asarray(eng.get_lattice()).reshape(L, L)
        eq = ((a == np.roll(a, 1, 0)).mean() + (a == np.roll(a, 1, 1)).mean()) / 2
        print(json.dumps(dict(L=L, mcs=n, equal_pair_frac=float(eq), counts=[int(c) for c in eng.counts()])))
