"""CPU: the C-ABI library (libescg_b200.so) without a GPU — loads, exports every symbol declared in
include/escg_dev.h, host-side precomputation is exact against the oracle/reference, validation mirrors
the reference's ConfigError behaviour, and the device path fails loudly (no CPU fallback)."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "escg_dev.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"ESCG_API\s+[\w\s\*]+?\b(escg_\w+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for s in ("escg_dev_create", "escg_dev_run", "escg_dev_replay", "escg_simulate", "escg_dev_last_error"):
        assert s in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol(escg):
    from paper_2508_16639_b200 import _lib

    lib = _lib.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2508_16639_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"#include\s*[<\"][^>\"]*oracle|import\s+pyoracle|from\s+pyoracle|liboracle|libescg_ref",
                                     text), f


def test_action_rates_and_align_match_reference(escg):
    k = json.load(open(os.path.join(ROOT, "tests", "golden", "kat.json")))
    for M, N, want in k["action_rates"]:
        r = escg.action_rates(M, N)
        assert [r.mu, r.sigma, r.epsilon, r.total] == want
    for a, b, want in k["align_num_randoms"]:
        if want < 0:
            with pytest.raises(escg.ConfigError):
                escg.align_num_randoms(a, b)
        else:
            assert escg.align_num_randoms(a, b) == want


@pytest.mark.parametrize("M,N", [(1e-4, 40000), (3e-5, 10 ** 6), (1e-4, 3200 * 3200), (1e-4, 16384 ** 2), (0.0, 10000),
                                 (3e-3, 10000), (1e-6, 40000)])
def test_bucket_thresholds_equal_reference_double_path(escg, oracle, M, N):
    """X_mig / X_int reproduce the reference's float/double bucketing (engine.hpp:117-123): dense
    check around both edges plus a strided sweep of the whole 2^32 range."""
    xm, xi, _ = escg.thresholds(M, N, escg.make_circulant(3, [1]))
    thr = np.array([xm, xi], np.uint32)
    for x in (xm, xi):
        lo, hi = max(0, x - 5000), min(2 ** 32 - 1, x + 5000)
        assert oracle.lib.orc_check_bucket_thresholds(thr, M, N, lo, hi, 1) == 0
    assert oracle.lib.orc_check_bucket_thresholds(thr, M, N, 0, 2 ** 32 - 1, 65537) == 0


def test_survey_threshold_table(escg):
    """SURVEY §A.3 values (measured there with the oracle's exact expressions)."""
    rps = escg.make_circulant(3, [1])
    assert escg.thresholds(1e-4, 40000, rps)[:2] == (3435973761, 3865470593)
    assert escg.thresholds(3e-5, 10 ** 6, escg.make_rpsls())[:2] == (4156419968, 4225693568)
    assert escg.thresholds(1e-4, 3200 * 3200, rps)[:2] == (4290776960, 4292872064)
    assert escg.thresholds(1e-4, 16384 ** 2, rps)[:2] == (4294807424, 4294887296)
    assert escg.thresholds(0.0, 10000, escg.make_park8(0.15, 0.75, 1.0))[:2] == (0, 2147483584)


@pytest.mark.parametrize("M,N", [(0.0, 10000), (1e-4, 40000), (3e-3, 16)])
def test_interaction_thresholds_equal_reference(escg, oracle, M, N):
    """T[a][b]: u < D[a][b] (engine.hpp:125-131) ⇔ x < T — checked at every edge and neighbours."""
    park = escg.make_park8(0.15, 0.75, 1.0)
    xm, xi, T = escg.thresholds(M, N, park)
    D = park.matrix()
    for a in range(1, 9):
        for b in range(1, 9):
            t = int(T[a, b])
            for x in {t - 2, t - 1, t, t + 1, xm, xi - 1, (xm + xi) // 2}:
                if not (xm <= x < xi):
                    continue
                want = oracle.lib.orc_interaction(x, M, N, np.ascontiguousarray(D.ravel()), 8, a, b)
                fires = x < t
                if D[a - 1, b - 1] > 0:
                    assert fires == (want == 1), (a, b, x)
                else:
                    assert not fires


def test_validation_matches_reference_messages(escg):
    cases = [
        (dict(length=1), "lattice dimensions must be at least 2x2"),
        (dict(mcs_limit=-1), "mcs limit must be non-negative"),
        (dict(print_frequency=0), "print frequency must be positive"),
        (dict(mobility=-1.0), "mobility must be non-negative"),
        (dict(species=65), "species count must be in [1, 64]"),
        (dict(length=65536, height=65536), "lattice exceeds the supported cell count"),
        (dict(empty_prob=1.5), "empty probability must be in [0, 1]"),
        (dict(num_randoms=0), "numRandoms must be positive"),
    ]
    for kw, msg in cases:
        with pytest.raises(escg.ConfigError, match=re.escape(msg)):
            escg.SimParams(**kw).validate()
    bad = escg.DominanceModel(3, escg.DominanceModel.Kind.Binary, np.array([0, 1, 0.5, 0, 0, 1, 1, 0, 0]))
    with pytest.raises(escg.ConfigError, match="binary dominance entries must be 0 or 1"):
        bad.validate()
    diag = escg.DominanceModel(2, escg.DominanceModel.Kind.Binary, np.array([1.0, 0, 0, 0]))
    with pytest.raises(escg.ConfigError, match="dominance diagonal must be zero"):
        diag.validate()
    with pytest.raises(escg.ConfigError, match="circulant offset 3 out of range"):
        escg.make_circulant(3, [3])


def test_presets_match_reference(escg, ref):
    assert np.array_equal(escg.make_circulant(3, [1]).matrix(), ref.circulant(3, [1]))
    assert np.array_equal(escg.make_rpsls().matrix(), ref.circulant(5, [1, 2]))
    assert np.array_equal(escg.make_rpsls_ablated().matrix(), ref.rpsls_ablated())
    assert np.array_equal(escg.make_park8(0.15, 0.75, 1.0).matrix(), ref.park8(0.15, 0.75, 1.0))


def test_save_schedule(escg):
    assert [m for m in range(2001) if escg.is_save_mcs(m, 2000)][:8] == [0, 1, 2, 5, 10, 20, 50, 100]


def test_device_path_fails_loudly_without_gpu(escg):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(escg.EngineError, match="no CPU fallback"):
        escg.DeviceEngine(escg.SimParams(seed=1), escg.make_circulant(3, [1]))
    with pytest.raises(escg.EngineError):
        escg.simulate(escg.SimParams(seed=1, mcs_limit=1), escg.make_circulant(3, [1]))


def test_build_targets_sm100a():
    """The in-tree library carries sm_100a SASS (cuobjdump), no PTX-JIT fallback."""
    import subprocess

    lib = os.path.join(ROOT, "paper_2508_16639_b200", "libescg_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_densities_mirror_reference_semantics(escg):
    """engine.cpp:70-94: counts per value in [0, S]; a value outside raises EngineError."""
    lat = escg.Lattice(3, 2, np.array([0, 1, 2, 2, 3, 0], np.int32))
    assert escg.densities(lat, 3).tolist() == [2, 1, 2, 1]
    with pytest.raises(escg.EngineError, match="corrupt lattice value 4"):
        escg.densities(escg.Lattice(2, 1, np.array([1, 4], np.int32)), 3)
    with pytest.raises(escg.EngineError, match="corrupt lattice value -1"):
        escg.densities(escg.Lattice(2, 1, np.array([-1, 0], np.int32)), 3)
