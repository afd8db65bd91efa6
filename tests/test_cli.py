"""CLI: defaults = Tables 3.1/3.2, alignment, usage errors / exit codes; GPU run+resume."""
import io
import os

import numpy as np
import pytest


def test_defaults_match_tables(escg):
    from paper_2508_16639_b200 import cli

    ns = cli.build_parser().parse_args(["run"])
    p = cli.params_from(ns)
    assert (p.length, p.height, p.mcs_limit, int(p.neighbourhood), p.print_frequency, p.mobility, p.species, p.flux,
            p.empty_prob, p.save, p.dominance_import, p.resume, p.num_randoms, p.max_step) == \
        (200, 200, 100000, 4, 200, 3e-05, 3, True, 0.0, False, False, False, 100000000, False)


def test_num_randoms_aligned_after_parsing(escg):
    from paper_2508_16639_b200 import cli

    p = cli.params_from(cli.build_parser().parse_args(["run", "--length", "300", "--height", "300", "--numRandoms", "100000005"]))
    assert p.num_randoms == 99990000


def test_usage_errors_and_exit_codes(escg, capsys):
    from paper_2508_16639_b200 import cli

    assert cli.main(["run", "--neighbourhood", "5"]) == 2
    assert "neighbourhood" in capsys.readouterr().err
    assert cli.main(["run", "--length", "x"]) == 2
    assert cli.main(["run", "--length", "1"]) == 2            # ConfigError from validate
    assert cli.main(["run", "--numRandoms", "10"]) == 2       # numRandoms < N
    assert cli.main(["resume", "--out", "/nonexistent/dir"]) == 3  # IoError


@pytest.mark.gpu
def test_run_save_resume(escg, tmp_path):
    from paper_2508_16639_b200 import cli
    from paper_2508_16639_b200 import persistence as P

    out = io.StringIO()
    assert cli.main(["run", "--length", "64", "--height", "64", "--mcs", "40", "--printFrequency", "20", "--seed", "5",
                     "--save", "true", "--out", str(tmp_path)], out=out) == 0
    lines = out.getvalue().splitlines()
    assert [ln.split(",")[0] for ln in lines] == ["0", "20", "40"]
    d = tmp_path / "L64_H64_n4_m3e-05_flux1_s3"
    cp = P.load_checkpoint(d)
    assert cp.saved_mcs == 40
    assert cli.main(["resume", "--out", str(d), "--mcs", "60"], out=io.StringIO()) == 0
    assert P.load_checkpoint(d).saved_mcs == 60
    assert (d / "densities.csv").read_text().splitlines()[0] == "mcs,count_0,count_1,count_2,count_3"
