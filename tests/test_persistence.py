"""Checkpoint / CSV formats: byte-compatible with the reference (round trip
through the reference's own load_checkpoint/save_checkpoint, out of process), and device resume from
a checkpoint is bit-identical to an uninterrupted run."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_csv_tool")


def need_tool():
    if not os.path.exists(TOOL):
        pytest.skip("oracle/_ref/ref_csv_tool not built")


@pytest.mark.parametrize("model_name", ["rps", "park8"])
def test_checkpoint_round_trips_through_reference(escg, tmp_path, model_name):
    need_tool()
    from paper_2508_16639_b200 import persistence as P

    model = escg.make_circulant(3, [1]) if model_name == "rps" else escg.make_park8(0.15, 0.75, 1.0)
    S = model.size
    params = escg.SimParams(length=12, height=7, species=S, mobility=3e-5 if S == 3 else 0.0, empty_prob=0.1,
                            seed=123456789012345, mcs_limit=500, max_step=True, num_randoms=1000)
    rng = np.random.default_rng(2)
    lat = escg.Lattice(12, 7, rng.integers(0, S + 1, 84).astype(np.int32))
    P.save_checkpoint(tmp_path / "a", params, lat, model, 250)
    r = subprocess.run([TOOL, "roundtrip", str(tmp_path / "a"), str(tmp_path / "b")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for f in ("params.csv", "grid.csv", "dominance.csv"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes(), f
    cp = P.load_checkpoint(tmp_path / "b")
    assert cp.saved_mcs == 250 and cp.params.seed == 123456789012345 and cp.params.max_step
    assert np.array_equal(cp.lattice.cells, lat.cells) and np.array_equal(cp.dominance.entries, model.entries)


def test_densities_and_dirname_match_reference(escg, tmp_path):
    need_tool()
    from paper_2508_16639_b200 import persistence as P

    tr = escg.DensityTrace()
    tr.append(0, [10, 20, 30, 40])
    tr.append(9, [11, 19, 31, 39])
    P.export_densities(tr, tmp_path / "d.csv")
    args = [TOOL, "densities", str(tmp_path / "e.csv"), "0", "3"] + [str(x) for x in (0, 10, 20, 30, 40, 9, 11, 19, 31, 39)]
    subprocess.run(args, check=True)
    assert (tmp_path / "d.csv").read_text() == (tmp_path / "e.csv").read_text()
    P.export_densities(tr, tmp_path / "d.csv", append=True)
    subprocess.run(args[:3] + ["1"] + args[4:], check=True)
    assert (tmp_path / "d.csv").read_text() == (tmp_path / "e.csv").read_text()
    for (L, H, n, M, flux, S) in [(200, 200, 4, 3e-5, 1, 3), (100, 50, 8, 0.0, 0, 8), (3200, 3200, 4, 1e-4, 1, 3)]:
        want = subprocess.run([TOOL, "dirname", str(L), str(H), str(n), repr(M), str(flux), str(S)], capture_output=True,
                              text=True).stdout.strip()
        p = escg.SimParams(length=L, height=H, neighbourhood=escg.Neighbourhood(n), mobility=M, flux=bool(flux), species=S)
        assert P.output_dir_name(p) == want
    assert P.output_dir_name(escg.SimParams()) == "L200_H200_n4_m3e-05_flux1_s3"


def test_format_errors(escg, tmp_path):
    from paper_2508_16639_b200 import persistence as P

    (tmp_path / "g.csv").write_text("1,0\n2\n7\n")
    with pytest.raises(escg.FormatError, match="ragged row at line 2"):
        P.import_grid(tmp_path / "g.csv")
    (tmp_path / "g.csv").write_text("1,0\n2,2\n")
    with pytest.raises(escg.FormatError, match="missing saved-MCS trailer"):
        P.import_grid(tmp_path / "g.csv")
    (tmp_path / "g.csv").write_text("1,0\n2,2\n7\n")
    lat, mcs = P.import_grid(tmp_path / "g.csv")
    assert mcs == 7 and lat.cells.tolist() == [1, 0, 2, 2]
    (tmp_path / "dm.csv").write_text("0,1\n1\n")
    with pytest.raises(escg.FormatError, match="not square"):
        P.import_dominance(tmp_path / "dm.csv")
    with pytest.raises(escg.IoError):
        P.import_params(tmp_path / "missing.csv")


@pytest.mark.gpu
def test_device_resume_from_checkpoint_is_bit_exact(escg, tmp_path):
    from paper_2508_16639_b200 import persistence as P

    model = escg.make_rpsls()
    p = escg.SimParams(length=64, height=64, species=5, mobility=1e-3, seed=99, mcs_limit=60)
    full = escg.simulate(p, model, escg.EngineMode.ParallelMcs)
    half = escg.simulate(escg.SimParams(**{**p.__dict__, "mcs_limit": 25}), model, escg.EngineMode.ParallelMcs)
    P.save_checkpoint(tmp_path / "cp", p, half.state.lattice, model, half.state.current_mcs)
    cp = P.load_checkpoint(tmp_path / "cp")
    rest = escg.simulate(cp.params, cp.dominance, escg.EngineMode.ParallelMcs, resume_from=P.resume_state(cp))
    assert rest.state.current_mcs == 60
    assert np.array_equal(rest.state.lattice.cells, full.state.lattice.cells)
    assert rest.state.trace.counts[-1].tolist() == full.state.trace.counts[-1].tolist()


def test_parse_int_follows_from_chars(escg):
    from paper_2508_16639_b200 import persistence as P

    assert P._parse_int("-12", "x") == -12 and P._parse_int("007", "x") == 7
    for bad in ["", "-", "+5", " 5", "5 ", "1e3", "²", "9223372036854775808", "--1"]:
        with pytest.raises(escg.FormatError):
            P._parse_int(bad, "x")
    assert P._parse_int("9223372036854775807", "x") == (1 << 63) - 1
