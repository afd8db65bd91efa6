"""CPU: the oracle restatement (oracle/escg_oracle.c) pinned against the reference's golden vectors
(tests/golden/*.json, generated from the unmodified reference by tests/golden/gen_golden.py) and,
where the reference library is built (oracle/_ref), against the reference directly."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def fnv1a64(cells):
    h = 1469598103934665603
    for v in np.asarray(cells, np.uint32).tolist():
        h = ((h ^ v) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def model(oracle, name):
    S = {"rps": 3, "rpsls": 5, "ablated": 5, "park8": 8}[name]
    D = np.zeros((S, S))
    if name == "rps":
        for i in range(3):
            D[i, (i + 1) % 3] = 1
    elif name in ("rpsls", "ablated"):
        for i in range(5):
            for k in (1, 2):
                D[i, (i + k) % 5] = 1
        if name == "ablated":
            D[0, 1] = 0  # experiments.cpp:57
    else:  # experiments.cpp:61-76
        for i in range(1, 9):
            D[i - 1, i % 8] = 1.0
            D[i - 1, (i + 1) % 8] = 0.15
        D[0, 4] = 0.75
        D[2, 6] = 0.75
    return D


def test_mt19937_kat(oracle):
    k = gold("kat.json")["mt19937_5489"]
    w = oracle.mt_words(5489, 10000)
    assert int(w[0]) == k["first"] == 3499211612
    assert int(w[-1]) == k["10000th"] == 4123659995


def test_seed_mix_and_streams(oracle):
    k = gold("kat.json")
    for s, i, v in k["seed_mix"]:
        assert oracle.lib.orc_seed_mix(s, i) == v
    for row in k["stream_words"]:
        assert oracle.stream_words(row["seed"], row["k"], 8).tolist() == row["words"]


def test_neighbor_index(oracle):
    for L, H, flux, arity, i, d, want in gold("kat.json")["neighbor_index"]:
        assert oracle.neighbor_index(i, d, arity, L, H, flux) == want
    # SPEC.md:86-88
    assert oracle.neighbor_index(0, 0, 4, 4, 4, True) == 12
    assert oracle.neighbor_index(5, 3, 4, 4, 4, True) == 6
    assert oracle.neighbor_index(0, 0, 4, 4, 4, False) == 4
    assert oracle.neighbor_index(0, 4, 4, 4, 4, True) == -1  # ConfigError: direction out of range


def test_align_and_rates(oracle):
    k = gold("kat.json")
    for a, b, want in k["align_num_randoms"]:
        assert oracle.lib.orc_align_num_randoms(a, b) == want
    for M, N, want in k["action_rates"]:
        assert oracle.action_rates(M, N).tolist() == want  # bit-identical doubles


def test_init_lattice(oracle):
    for row in gold("kat.json")["init_lattice"]:
        st = oracle.lib
        init, *_ = oracle.serial_draws(row["L"], row["H"], row["S"], row["p0"], row["seed"], 0)
        assert init[:16].tolist() == row["first16"]
        assert fnv1a64(init) == row["fnv"]


def test_philox_kat(oracle):
    for row in gold("kat.json")["philox4x32_10"]:
        assert oracle.philox(row["ctr"], row["key"]).tolist() == row["out"]


@pytest.mark.parametrize("case", range(7))
def test_serial_runs_match_reference_goldens(oracle, case):
    g = gold("serial.json")[case]
    D = model(oracle, g["model"])
    res = oracle.run_serial(g["L"], g["H"], D, g["M"], g["p0"], g["mcs"], g["seed"], arity=g["arity"],
                            flux=bool(g["flux"]), tracked=g["tracked"])
    assert res["status"] == g["status"]
    assert len(res["steps"]) == g["n_records"]
    assert res["counts"][-1].tolist() == g["final_counts"]
    for k, v in g["counts_at"].items():
        assert res["counts"][int(k)].tolist() == v
    assert fnv1a64(res["cells"]) == g["fnv"]


def test_rule_table_matches_reference(oracle):
    rows = gold("rule.json")
    for name, Meff, s, n, d, x, rc, s2, n2 in rows:
        D = model(oracle, name)
        cells = np.zeros(16, np.int32)
        cells[5] = s
        nbi = oracle.neighbor_index(5, d, 4, 4, 4, True)
        cells[nbi] = n
        got = oracle.apply_draws(cells, 4, 4, D, Meff, np.array([5], np.uint32), np.array([d], np.uint32),
                                 np.array([x], np.uint32))
        assert (int(got[5]), int(got[nbi])) == (s2, n2), (name, s, n, d, x)


def test_rule_table_shape_rps(oracle):
    """interaction with an empty site is a no-op, reproduction only into an empty site,
    migration swaps any unequal pair."""
    rows = [r for r in gold("rule.json") if r[0] == "rps"]
    for name, Meff, s, n, d, x, rc, s2, n2 in rows:
        if s == n:
            assert (s2, n2) == (s, n)


def test_is_save_mcs(oracle):
    want = [m for m in range(0, 2001) if oracle.lib.orc_is_save_mcs(m, 2000)]
    assert want[:12] == [0, 1, 2, 5, 10, 20, 50, 100, 200, 500, 1000, 2000]


def test_crs_round_and_init_are_pure_functions(oracle):
    """Device schedule spec: round parameters and init depend only on (seed, mcs)."""
    a = [oracle.crs_round(7, m) for m in range(64)]
    assert a == [oracle.crs_round(7, m) for m in range(64)]
    perms = {tuple(p) for _, _, p in a}
    assert all(sorted(p) == [0, 1, 2, 3] for p in perms) and len(perms) > 10
    assert {(oy, ox) for oy, ox, _ in a} == {(0, 0), (0, 1), (1, 0), (1, 1)}
    c = oracle.crs_init(40, 40, 5, 0.1, 99)
    assert np.array_equal(c, oracle.crs_init(40, 40, 5, 0.1, 99))
    frac_empty = (c == 0).mean()
    assert 0.05 < frac_empty < 0.15
    assert oracle.lib.orc_seed32(5) == 5 and oracle.lib.orc_seed32(5 + (1 << 32)) != 5


@pytest.mark.parametrize("flux,arity,narrow", [(True, 4, False), (True, 4, True), (True, 8, False), (False, 4, False),
                                               (False, 8, False)])
def test_crs_schedule_conserves_lattice_invariants(oracle, flux, arity, narrow):
    """Colouring makes each phase an exact sequential update: values stay in [0, S], counts sum to N,
    the run is deterministic and resumable (MCS split points do not change the result)."""
    L, H = (48, 32) if flux else (21, 15)
    D = model(oracle, "rps")
    init = oracle.crs_init(L, H, 3, 0.1, 5)
    a = oracle.crs_run(init, L, H, D, 1e-2, 5, 0, 10, arity=arity, flux=flux, narrow=narrow)
    b = oracle.crs_run(oracle.crs_run(init, L, H, D, 1e-2, 5, 0, 4, arity=arity, flux=flux, narrow=narrow), L, H, D,
                       1e-2, 5, 4, 6, arity=arity, flux=flux, narrow=narrow)
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() <= 3 and a.size == L * H
    assert not np.array_equal(a, init)


def test_crs_tiles_are_disjoint():
    """Same-colour 2x2 tiles have disjoint von-Neumann/Moore footprints on periodic lattices with
    L, H ≡ 0 (mod 4) and on reflecting lattices of any size."""
    for (L, H, periodic) in [(8, 8, True), (12, 20, True), (7, 9, False), (2, 3, False), (10, 6, False)]:
        for oy in (0, 1):
            for ox in (0, 1):
                Ty = H // 2 if periodic else (H + oy + 1) // 2
                Tx = L // 2 if periodic else (L + ox + 1) // 2
                for cy in (0, 1):
                    for cx in (0, 1):
                        seen = {}
                        for ty in range(cy, Ty, 2):
                            for tx in range(cx, Tx, 2):
                                for dy in range(-1, 3):
                                    for dx in range(-1, 3):
                                        y, x = 2 * ty - oy + dy, 2 * tx - ox + dx
                                        if periodic:
                                            y, x = y % H, x % L
                                        elif not (0 <= y < H and 0 <= x < L):
                                            if y == -1:
                                                y = 1
                                            if x == -1:
                                                x = 1
                                            if y == H:
                                                y = H - 2
                                            if x == L:
                                                x = L - 2
                                            if not (0 <= y < H and 0 <= x < L):
                                                continue
                                        key = (y, x)
                                        assert seen.get(key, (ty, tx)) == (ty, tx), (L, H, periodic, oy, ox, key)
                                        seen[key] = (ty, tx)


def _axis_colours(n):
    """tiles and colours of a periodic axis (mirror of escg_oracle.c crs_axis)."""
    T = n // 2 if n % 4 == 0 else (n + 1) // 2
    seam = -1 if n % 4 == 0 else (T - 2 if n % 4 == 3 else T - 1)
    return T, [2 if t == seam else (t & 1) for t in range(T)]


@pytest.mark.parametrize("n", list(range(4, 41)) + [50, 101, 102, 103, 200])
def test_seam_colouring_gives_disjoint_footprints(n):
    """Periodic axes of any length >= 4: same-colour tiles have disjoint 1-D footprints (their cells
    +-1, modulo n) for both tiling origins, footprints never wrap onto themselves, and every cell
    belongs to exactly one tile.  The 2-D (von Neumann / Moore) footprint is the product of the two
    axes' footprints, so the 2-D colour classes (cy, cx) are disjoint too."""
    T, col = _axis_colours(n)
    for o in (0, 1):
        owner = {}
        foot = []
        for t in range(T):
            cells = [(2 * t + d - o) % n for d in (0, 1) if 2 * t + d < n]
            for c in cells:
                assert c not in owner
                owner[c] = t
            f = {(c + e) % n for c in cells for e in (-1, 0, 1)}
            assert len(f) == len(cells) + 2
            foot.append(f)
        assert len(owner) == n
        for t in range(T):
            for u in range(t + 1, T):
                if col[t] == col[u]:
                    assert not (foot[t] & foot[u]), (n, o, t, u)


def test_crs_round_generic_permutations(oracle):
    for ncy, ncx in [(2, 2), (2, 3), (3, 2), (3, 3)]:
        seen = set()
        for m in range(200):
            oy, ox, perm = oracle.crs_round_g(11, m, ncy, ncx)
            assert sorted(perm) == list(range(ncy * ncx))
            seen.add(tuple(perm))
            if ncy * ncx == 4:
                assert (oy, ox, perm) == oracle.crs_round(11, m)
        assert len(seen) > (10 if ncy * ncx == 4 else 50)


@pytest.mark.parametrize("L,H,arity", [(50, 50, 4), (21, 15, 4), (7, 6, 8), (13, 20, 8), (4, 5, 4)])
def test_crs_seam_schedule_invariants(oracle, L, H, arity):
    D = model(oracle, "rps")
    init = oracle.crs_init(L, H, 3, 0.1, 8)
    a = oracle.crs_run(init, L, H, D, 1e-2, 8, 0, 12, arity=arity)
    b = oracle.crs_run(oracle.crs_run(init, L, H, D, 1e-2, 8, 0, 5, arity=arity), L, H, D, 1e-2, 8, 5, 7, arity=arity)
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() <= 3 and not np.array_equal(a, init)


def test_oracle_matches_compiled_reference(oracle, ref):
    """Direct cross-check with the reference library (only where oracle/_ref was built)."""
    D = ref.circulant(3, [1])
    a = oracle.run_serial(32, 24, D, 1e-3, 0.1, 30, 77)
    b = ref.simulate(32, 24, D, 1e-3, 0.1, 30, 77)
    assert np.array_equal(a["cells"], b["cells"]) and np.array_equal(a["counts"], b["counts"])
    assert np.array_equal(ref.init_lattice(20, 20, 5, 0.2, 3), oracle.serial_draws(20, 20, 5, 0.2, 3, 0)[0])


def test_slice3_thresholds_track_the_exact_powers(oracle):
    """SLICED3 run thresholds (escg_oracle.c orc_slice3_table): T[g-1] within g of floor((1-2^-K)^g 2^32)."""
    from fractions import Fraction

    for K in (6, 8, 10, 12, 14, 16):
        t = oracle.slice3_table(K)
        for g in range(1, 33):
            exact = int(Fraction(2 ** K - 1, 2 ** K) ** g * 2 ** 32)
            assert exact - g <= int(t[g - 1]) <= exact, (K, g)


@pytest.mark.parametrize("K", [6, 8])
def test_slice3_masks_are_iid_bernoulli(oracle, K):
    """The SLICED3 undecided mask of an attempt has i.i.d. Bernoulli(2^-K) bits: the count of set bits
    per mask is Binomial(32, 2^-K) and every bit position is equally likely (chi-square)."""
    import math

    q = 2.0 ** -K
    n = 40000
    pos = np.zeros(32)
    zeros = ones = multi = 0
    for i in range(n):
        u = oracle.slice3_mask(77, i, 5, i % 4, i % 4, K)
        c = bin(u).count("1")
        zeros += c == 0
        ones += c == 1
        multi += c >= 2
        for b in range(32):
            pos[b] += (u >> b) & 1
    p0 = (1 - q) ** 32
    p1 = 32 * q * (1 - q) ** 31
    for k, p in ((zeros, p0), (ones, p1), (multi, 1 - p0 - p1)):
        assert abs(k - n * p) < 5 * math.sqrt(n * p * (1 - p)) + 1, (K, k, n * p)
    exp = pos.sum() / 32
    chi2 = ((pos - exp) ** 2 / exp).sum()
    assert chi2 < 70, chi2  # 31 dof, p ~ 1e-4
