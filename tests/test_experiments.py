"""Experiments harness: CPU format pins against the reference, GPU runs."""
import ctypes as C
import os
import random

import numpy as np
import pytest


def test_format_double_matches_reference(ref):
    from paper_2508_16639_b200.experiments import format_double

    f = ref.lib.ref_format_double
    f.argtypes = [C.c_double, C.c_char_p, C.c_int]
    f.restype = C.c_int
    buf = C.create_string_buffer(64)
    rng = random.Random(3)
    vals = [0.0, -0.0, 1.0, 0.1, 3e-5, 100000.0, 1e16, 1e21, 1e-7, 2 / 3, 0.15, 12345678.0, 1e5, 5e-324, 1e-5,
            123456.0, 1234567.0, 0.001, 0.0001, 1e22, 1e15, 1.5e-5, 0.875, 0.020833333333333332]
    vals += [rng.uniform(-1e6, 1e6) for _ in range(200)] + [10 ** rng.uniform(-30, 30) for _ in range(300)]
    vals += [float(rng.randint(0, 10 ** 9)) for _ in range(100)]
    for v in vals:
        f(v, buf, 64)
        assert format_double(v) == buf.value.decode(), v


def ref_tool():
    tool = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "ref_csv_tool")
    if not os.path.exists(tool):
        pytest.skip("oracle/_ref/ref_csv_tool not built")
    return tool


def test_csv_writers_match_reference(tmp_path):
    """experiments.cpp:242-285 run out of process by oracle/_ref/ref_csv_tool."""
    import subprocess

    from paper_2508_16639_b200 import experiments as X

    tool = ref_tool()
    st = X.ExtinctionStats(times=[156, 2000, 141], censored=[False, True, False], budget=2000)
    X.write_extinction_csv(st, tmp_path / "a.csv")
    subprocess.run([tool, "extinction", str(tmp_path / "b.csv"), "156", "0", "2000", "1", "141", "0"], check=True)
    assert (tmp_path / "a.csv").read_text() == (tmp_path / "b.csv").read_text()
    r = X.CoexistenceResult(trials=48, coexisting=13, probability=13 / 48)
    X.write_coexistence_csv(r, 1e-3, 100, 3000, tmp_path / "c.csv")
    subprocess.run([tool, "coexistence", str(tmp_path / "d.csv"), "48", "13", repr(13 / 48), "0.001", "100", "3000"],
                   check=True)
    assert (tmp_path / "c.csv").read_text() == (tmp_path / "d.csv").read_text()


def test_stats_helpers():
    from paper_2508_16639_b200 import experiments as X

    m = X.mean_std([1.0, 2.0, 3.0, 4.0])
    assert m.mean == 2.5 and abs(m.std_dev - 1.2909944487358056) < 1e-15 and m.n == 4
    assert X.mean_std([5.0]).std_dev == 0.0
    st = X.ExtinctionStats(times=[100, 250, 700, 2000], censored=[False, False, False, True], budget=2000)
    assert st.in_window(200, 600) == 1 and st.summary().n == 3
    assert X.parse_engine_mode("maxstep") == X.EngineMode.MaxStep and X.engine_mode_name(X.EngineMode.ParallelMcs) == "parallel"
    with pytest.raises(X.ConfigError):
        X.parse_engine_mode("turbo")
    assert X.trial_seed(10, 3) == 13


@pytest.mark.gpu
def test_ablated_rpsls_harness_matches_engine(escg, tmp_path):
    from paper_2508_16639_b200 import experiments as X

    st = X.run_ablated_rpsls(48, 12, 3000, seed=100)
    assert len(st.times) == 12 and st.budget == 3000
    p = escg.SimParams(length=48, height=48, species=5, mcs_limit=3000, seed=100)
    with escg.DeviceEngine(p, escg.make_rpsls_ablated(), n_replicas=12, seeds=range(100, 112), kernel="tile") as eng:
        eng.init_lattice()
        s = eng.run(3000, interval=1, tracked=4, record_trace=False)
        for r in range(12):
            m, status, last = eng.replica_result(r)
            assert (st.times[r], st.censored[r]) == ((m, False) if status == 2 else (3000, True))
    X.write_extinction_csv(st, tmp_path / "e.csv")
    assert (tmp_path / "e.csv").read_text().startswith("trial,extinction_mcs,censored\n0,")


@pytest.mark.gpu
def test_coexistence_and_park_sweep(escg, tmp_path):
    from paper_2508_16639_b200 import experiments as X

    lo = X.run_coexistence_probe(1e-4, 64, 300, 16, seed=7)
    hi = X.run_coexistence_probe(3e-2, 64, 300, 16, seed=7)
    assert lo.trials == 16 and lo.probability >= hi.probability
    tab = X.run_park_sweep(X.SweepSpec(alphas=[0.15, 0.5], length=40, trials=6, mcs=200, seed=3))
    assert len(tab.cells) == 16 and all(0.0 <= c.survival_prob <= 1.0 for c in tab.cells)
    X.write_sweep_csv(tab, tmp_path / "s.csv")
    assert (tmp_path / "s.csv").read_text().splitlines()[0] == "alpha,species,survival_prob,std,n"
    rows = X.run_bench_matrix([64], [X.EngineMode.Serial, X.EngineMode.MaxStep], 50, 2, 1, seed=1)
    assert len(rows) == 2 and all(r.mean_s > 0 for r in rows)
    X.write_bench_csv(rows, 50, tmp_path / "b.csv")
    tune = X.run_tuning_curve(64, [1, 5], 20, seed=1)
    assert [t.num_randoms for t in tune] == [64 * 64, 5 * 64 * 64]
