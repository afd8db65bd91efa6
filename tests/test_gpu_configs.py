"""GPU parity at the configurations the bench and BASELINE.json name (VERDICT r01 "what's missing" 1).

Every test runs the engine exactly as AUTO plans it for that configuration (kernel, draw format,
block split, MCS per launch, record cadence) and compares each lattice and each density record with
oracle/escg_oracle.c:orc_crs_run + densities(), the sequential definition of the coloured schedule
(the reference rule engine.hpp:108-141 on the same Philox draws; the MaxStep loop engine.cpp:165-192
supplies the record cadence align(numRandoms, N)/N).

  C3  RPS L=3200, M=1e-4, p0=0.1, MaxStep (numRandoms 1e8 -> 9 MCS per record): the bench workload
  C2  RPSLS L=1000, M=3e-5 (the reference's default mobility), Serial cadence (record every MCS)
  C5  RPS L=16384, M=1e-4, p0=0.1: the large-lattice plan, 2 MCS

The oracle runs ~1.7 s per MCS at L=3200 and ~45 s at L=16384 on one host core.
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run_records(oracle, init, L, H, dom, M, seed, code, S, mcs0, bounds):
    """Oracle states at each record MCS in `bounds` (ascending, starting at mcs0)."""
    cur, t, out = init, mcs0, []
    for b in bounds:
        if b > t:
            cur = oracle.crs_run(cur, L, H, dom, M, seed, t, b - t, narrow=code)
            t = b
        out.append((cur, oracle.densities(cur, S).tolist()))
    return out


def test_c3_bench_configuration_matches_oracle(escg, oracle):
    """The bench kernel as planned (bit-sliced, K=10, 2 MCS per launch) with the bench's own record
    cadence: advance(4), then run to MCS 22 with interval 9 (records at 4, 13, 22), every record and
    both lattices against the oracle."""
    L, M, p0, seed = 3200, 1e-4, 0.1, 20240601
    model = escg.make_circulant(3, [1])
    p = escg.SimParams(length=L, height=L, species=3, mobility=M, empty_prob=p0, num_randoms=100000000,
                       max_step=True, seed=seed, mcs_limit=22)
    interval = escg.align_num_randoms(p.num_randoms, L * L) // (L * L)
    assert interval == 9
    with escg.DeviceEngine(p, model) as eng:
        d = eng.describe()
        code = eng.draw_code()
        assert code >> 8 == 10 and code & 0xFF in (2, 3), hex(code)  # bit-sliced, K = 10 action bits
        assert d["kernel"] in ("block", "ring") and d["draw_format"] == "sliced", d
        eng.init_lattice()
        init = eng.get_lattice()
        assert np.array_equal(init, oracle.crs_init(L, L, 3, p0, seed))
        eng.advance(4)
        got4 = eng.get_lattice()
        st = eng.run(22, interval=interval)
        fin = eng.get_lattice()
        steps, counts = eng.read_trace()
    assert int(st[0]) == int(escg.RunStatus.Completed)
    want4 = oracle.crs_run(init, L, L, model.matrix(), M, seed, 0, 4, narrow=code)
    assert np.array_equal(got4, want4)
    assert steps.tolist() == [4, 13, 22]
    recs = _run_records(oracle, want4, L, L, model.matrix(), M, seed, code, 3, 4, [4, 13, 22])
    for (lat, dens), c in zip(recs, counts.tolist()):
        assert c == dens
    assert np.array_equal(fin, recs[-1][0])


def test_c3_bench_plan_is_the_measured_one(escg):
    """The plan the r01 bench numbers were measured on (or the ring kernel that replaces it)."""
    L = 3200
    p = escg.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10)
    with escg.DeviceEngine(p, escg.make_circulant(3, [1])) as eng:
        d = eng.describe()
    if d["kernel"] == "block":
        assert d["ctas"] == 145 and d["kmcs"] == 2 and d["threads"] == 256, d
    else:
        assert d["kernel"] == "ring", d


def test_c2_rpsls_l1000_matches_oracle(escg, oracle):
    """RPSLS L=1000 at the default mobility 3e-5 (P(migration) 0.968: the byte-level block kernel,
    WIDE draws, planner split), Serial cadence: advance(3), then run(10, interval=1) with a record
    every MCS, each record and the final lattice against the oracle."""
    L, M, p0, seed = 1000, 3e-5, 0.0, 5
    model = escg.make_rpsls()
    p = escg.SimParams(length=L, height=L, species=5, mobility=M, empty_prob=p0, seed=seed, mcs_limit=10)
    with escg.DeviceEngine(p, model) as eng:
        d = eng.describe()
        code = eng.draw_code()
        assert d["kernel"] == "block" and code == 0, (d, code)
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(3)
        got3 = eng.get_lattice()
        st = eng.run(10, interval=1)
        fin = eng.get_lattice()
        steps, counts = eng.read_trace()
    assert int(st[0]) == int(escg.RunStatus.Completed)
    want3 = oracle.crs_run(init, L, L, model.matrix(), M, seed, 0, 3, narrow=code)
    assert np.array_equal(got3, want3)
    assert steps.tolist() == list(range(3, 11))
    recs = _run_records(oracle, want3, L, L, model.matrix(), M, seed, code, 5, 3, list(range(3, 11)))
    for (lat, dens), c in zip(recs, counts.tolist()):
        assert c == dens
    assert np.array_equal(fin, recs[-1][0])


def test_c5_l16384_matches_oracle(escg, oracle):
    """RPS L=16384 (268M cells) with its own AUTO plan: 2 MCS against the oracle, plus the record."""
    L, M, p0, seed = 16384, 1e-4, 0.1, 99
    model = escg.make_circulant(3, [1])
    p = escg.SimParams(length=L, height=L, species=3, mobility=M, empty_prob=p0, seed=seed, mcs_limit=2)
    with escg.DeviceEngine(p, model) as eng:
        d = eng.describe()
        code = eng.draw_code()
        assert d["draw_format"] == "sliced", d
        eng.init_lattice()
        init = eng.get_lattice()
        st = eng.run(2, interval=2)
        fin = eng.get_lattice()
        steps, counts = eng.read_trace()
    assert int(st[0]) == int(escg.RunStatus.Completed)
    want = oracle.crs_run(init, L, L, model.matrix(), M, seed, 0, 2, narrow=code)
    del init
    assert np.array_equal(fin, want)
    assert steps.tolist() == [0, 2]
    assert counts.tolist()[1] == oracle.densities(want, 3).tolist()
