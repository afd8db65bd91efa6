"""GPU parity of the persistent bit-sliced ring kernel (csrc/ring.cu).

The ring kernel computes the same coloured schedule with the same draws as the overlapped-tile
bit-sliced kernel, so oracle/escg_oracle.c orc_crs_run (fmt = 2 | K << 8) is its definition too:
every lattice, record and stop decision must match bit for bit — for any number of bands (the draws
depend only on global coordinates), with the bands' boundary rows exchanged through the L2
mailboxes every colour phase (engine.hpp:108-141 per tile; records engine.cpp:47-57, 165-192).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RING_CASES = [
    # L, H, S, M, p0, model, bands (ESCG_RING_NB; None = one per SM up to H/8), expected K
    (1024, 256, 3, 1.0, 0.1, "rps", None, 16),   # 32 bands of 8 rows
    (1024, 256, 3, 1.0, 0.1, "rps", "2", 16),    # two bands of 128 rows: warps loop over slabs
    (1024, 200, 3, 1e-1, 0.0, "rps", "7", 14),   # uneven bands (28 or 29 rows)
    (512, 96, 3, 1e-2, 0.1, "rps", "5", 8),      # 4 groups per row, bands of 19-20 rows
    (512, 96, 5, 1e-2, 0.1, "rpsls", "3", 8),    # 3 bit planes
    (128, 64, 3, 3e-2, 0.2, "rps", "4", None),   # one group: every row wraps onto its own lane
    (3200, 160, 3, 1e-3, 0.1, "rps", None, None),  # 25 groups (the bench's row width), 20 bands of 8
]


def _model(escg, name):
    return {"rps": lambda: escg.make_circulant(3, [1]), "rpsls": escg.make_rpsls}[name]()


def _params(escg, L, H, S, M, p0, seed, mcs):
    return escg.SimParams(length=L, height=H, species=S, mobility=M, empty_prob=p0, seed=seed, mcs_limit=mcs)


@pytest.mark.parametrize("qcap,draws", [(None, "3"), ("1", "3"), (None, "2")])
@pytest.mark.parametrize("case", RING_CASES, ids=[f"{c[0]}x{c[1]}_{c[5]}_nb{c[6]}" for c in RING_CASES])
def test_ring_matches_crs_oracle(escg, oracle, case, qcap, draws, monkeypatch):
    """advance(3), advance(4), then run(12, interval=2): lattices and every record against the
    oracle.  qcap=1 shrinks the per-warp deferred-tile queue so the in-place replay runs."""
    L, H, S, M, p0, name, nb, K = case
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    monkeypatch.setenv("ESCG_SLICE_DRAWS", draws)  # SLICED3 (default) and SLICED
    if nb:
        monkeypatch.setenv("ESCG_RING_NB", nb)
    if qcap:
        monkeypatch.setenv("ESCG_SLICE_QCAP", qcap)
    model = _model(escg, name)
    seed = 0xBEEF + L + H
    with escg.DeviceEngine(_params(escg, L, H, S, M, p0, seed, 12), model, kernel="ring") as eng:
        d = eng.describe()
        code = eng.draw_code()
        assert d["kernel"] == "ring" and code & 0xFF == int(draws) and (K is None or code >> 8 == K), (d, hex(code))
        if nb:
            assert d["ctas"] == int(nb)
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(3)
        got3 = eng.get_lattice()
        eng.advance(4)
        got7 = eng.get_lattice()
        st = eng.run(12, interval=2)
        fin = eng.get_lattice()
        steps, counts = eng.read_trace()
    want3 = oracle.crs_run(init, L, H, model.matrix(), M, seed, 0, 3, narrow=code)
    assert np.array_equal(got3, want3)
    want7 = oracle.crs_run(want3, L, H, model.matrix(), M, seed, 3, 4, narrow=code)
    assert np.array_equal(got7, want7)
    assert steps.tolist() == [7, 9, 11, 12] and int(st[0]) == int(escg.RunStatus.Completed)
    cur = want7
    for t0, t1, c in zip([7, 7, 9, 11], [7, 9, 11, 12], counts.tolist()):
        cur = oracle.crs_run(cur, L, H, model.matrix(), M, seed, t0, t1 - t0, narrow=code) if t1 > t0 else cur
        assert c == oracle.densities(cur, S).tolist()
    assert np.array_equal(fin, cur)


def test_ring_is_auto_choice_for_bench_lattice(escg):
    """AUTO: a single L=3200 RPS lattice at M=1e-4 runs on the ring kernel, one band per SM."""
    p = _params(escg, 3200, 3200, 3, 1e-4, 0.1, 1, 10)
    with escg.DeviceEngine(p, escg.make_circulant(3, [1])) as eng:
        d = eng.describe()
    assert d["kernel"] == "ring" and d["draw_format"] == "sliced" and d["threads"] == 256, d
    assert d["ctas"] >= 100, d


def test_ring_stops_mid_run_like_oracle(escg, oracle, monkeypatch):
    """Tracked extinction inside a run: species 2 starts with a few cells among species 1 (its
    predator), records every MCS.  The run must stop at the oracle's first record without species 2
    and return that record's lattice (the band snapshot), not a later one."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    monkeypatch.setenv("ESCG_RING_NB", "6")
    L, H, M, seed = 512, 64, 3e-3, 4242
    model = escg.make_circulant(3, [1])
    rng = np.random.default_rng(5)
    cells = np.where(rng.random(L * H) < 0.1, 0, 1).astype(np.int32)
    cells[rng.choice(L * H, 6, replace=False)] = 2
    with escg.DeviceEngine(_params(escg, L, H, 3, M, 0.0, seed, 2000), model, kernel="ring") as eng:
        code = eng.draw_code()
        eng.set_lattice(cells)
        st = eng.run(2000, interval=1, tracked=2)
        got = eng.get_lattice()
        mcs = eng.mcs()
        steps, counts = eng.read_trace()
    cur, t = cells, 0
    while oracle.densities(cur, 3)[2] > 0 and t < 2000:
        cur = oracle.crs_run(cur, L, H, model.matrix(), M, seed, t, 1, narrow=code)
        t += 1
    assert t < 2000, "species 2 survived the oracle run; pick another seed"
    assert int(st[0]) == int(escg.RunStatus.Stopped) and mcs == t
    assert steps.tolist() == list(range(0, t + 1))
    assert counts.tolist()[-1] == oracle.densities(cur, 3).tolist()
    assert np.array_equal(got, cur)


def test_ring_stasis_at_first_record(escg, monkeypatch):
    """One species left: stasis at the run's first record, before the ring kernel steps."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    L, H = 1024, 64
    cells = np.ones(L * H, np.int32)
    cells[::7] = 0
    with escg.DeviceEngine(_params(escg, L, H, 3, 1.0, 0.0, 1, 50), escg.make_circulant(3, [1]), kernel="ring") as eng:
        eng.set_lattice(cells)
        st = eng.run(50, interval=5)
        assert int(st[0]) == int(escg.RunStatus.Stasis) and eng.mcs() == 0
        assert np.array_equal(eng.get_lattice(), cells)


@pytest.mark.parametrize("draws", ["2", "3"])
def test_ring_long_run_equals_block_slice_kernel(escg, monkeypatch, draws):
    """200 MCS with 9-MCS records at the bench's row width: the ring kernel and the overlapped-tile
    bit-sliced kernel (both the oracle's schedule) give the same trace and lattice, for either
    sliced draw format (each kernel's default differs, so the format is pinned here)."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    monkeypatch.setenv("ESCG_SLICE_DRAWS", draws)
    L, H, M, seed = 3200, 256, 1e-4, 77
    model = escg.make_circulant(3, [1])
    out = []
    for kernel in ("ring", "block"):
        with escg.DeviceEngine(_params(escg, L, H, 3, M, 0.1, seed, 200), model, kernel=kernel) as eng:
            assert eng.describe()["kernel"] == kernel
            eng.init_lattice()
            st = eng.run(200, interval=9)
            out.append((int(st[0]), eng.read_trace(), eng.get_lattice()))
    (s1, (t1, c1), l1), (s2, (t2, c2), l2) = out
    assert s1 == s2 == int(escg.RunStatus.Completed)
    assert t1.tolist() == t2.tolist() and np.array_equal(c1, c2)
    assert np.array_equal(l1, l2)


# ---- multi-part ring (escg_dev_create_ring_part; bands.RingGroup) ------------------------------

RING_PART_CASES = [
    # L, H, parts, ctas per part (0: the device's SMs shared by the parts), M, model
    (1024, 256, 2, 0, 1e-2, "rps"),
    (1024, 256, 3, 0, 1e-2, "rps"),
    (1024, 256, 4, 3, 3e-2, "rps"),    # few fat bands per part: interior slabs too
    (512, 96, 2, 1, 1e-2, "rps"),      # one band per part: every band is both boundary bands of its part
    (3200, 320, 2, 0, 1e-3, "rps"),    # the bench's row width
    (1024, 200, 3, 2, 1e-2, "rpsls"),  # 3 bit planes, parts of 64-68 rows, uneven bands
    (640, 136, 8, 1, 3e-2, "rps"),     # the most parts, 16-20 rows each
]


@pytest.mark.parametrize("case", RING_PART_CASES, ids=[f"{c[0]}x{c[1]}_p{c[2]}_c{c[3]}_{c[5]}" for c in RING_PART_CASES])
def test_ring_parts_match_crs_oracle(escg, oracle, case):
    """A lattice split into parts whose ring kernels exchange boundary rows through each other's
    inboxes and planes (one launch over all parts: the single-GPU form of the multi-GPU ring).
    Consecutive advances alternate the inbox sets and hand the final boundary rows over by flag;
    a host write in between restarts from the neighbours' rows.  Lattices and counts against the
    oracle (draw format 2 | K << 8, the same as the single ring's)."""
    from paper_2508_16639_b200.bands import RingGroup

    L, H, n, ctas, M, name = case
    model = _model(escg, name)
    S = model.size
    seed = 4000 + L + n
    p = _params(escg, L, H, S, M, 0.1, seed, 100)
    with RingGroup(p, model, n, ctas=ctas) as grp:
        d = grp.describe()
        code = d["draw_code"]
        assert d["kernel"] == "ring" and code & 0xFF == 2, d
        grp.init_lattice()
        init = grp.get_lattice()
        assert np.array_equal(init, oracle.crs_init(L, H, S, 0.1, seed))
        cur, t = init, 0
        for step in (3, 1, 2, 5):
            grp.advance(step)
            cur = oracle.crs_run(cur, L, H, model.matrix(), M, seed, t, step, narrow=code)
            t += step
            assert np.array_equal(grp.get_lattice(), cur), ("after MCS", t)
        assert grp.counts().tolist() == oracle.densities(cur, S).tolist()
        # host write between advances: the next launch reads the neighbours' rows directly
        rng = np.random.default_rng(n)
        cells = rng.integers(0, S + 1, L * H).astype(np.int32)
        grp.set_lattice(cells, mcs=t)
        grp.advance(2)
        grp.advance(3)
        want = oracle.crs_run(cells, L, H, model.matrix(), M, seed, t, 5, narrow=code)
        assert np.array_equal(grp.get_lattice(), want)


def test_ring_parts_equal_single_ring(escg):
    """40 MCS at the bench's row width: a 4-part ring equals the single-device ring."""
    from paper_2508_16639_b200.bands import RingGroup

    L, H, M, seed = 3200, 512, 1e-4, 91
    model = escg.make_circulant(3, [1])
    p = _params(escg, L, H, 3, M, 0.1, seed, 40)
    with escg.DeviceEngine(p, model, kernel="ring") as eng:
        eng.init_lattice()
        eng.advance(40)
        want = eng.get_lattice()
    with RingGroup(p, model, 4) as grp:
        grp.init_lattice()
        for _ in range(4):
            grp.advance(10)
        got = grp.get_lattice()
    assert np.array_equal(got, want)


@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2")
def test_ring_parts_on_two_gpus(escg, oracle):
    """Parts on two GPUs of one process: one launch per GPU, rows cross over NVLink peer stores."""
    from paper_2508_16639_b200.bands import RingGroup

    L, H, M, seed = 1024, 256, 1e-2, 5150
    model = escg.make_circulant(3, [1])
    with RingGroup(_params(escg, L, H, 3, M, 0.1, seed, 10), model, 2, devices=[0, 1]) as grp:
        code = grp.describe()["draw_code"]
        grp.init_lattice()
        init = grp.get_lattice()
        grp.advance(3)
        grp.advance(4)
        got = grp.get_lattice()
    assert np.array_equal(got, oracle.crs_run(init, L, H, model.matrix(), M, seed, 0, 7, narrow=code))


def test_ring_part_without_neighbour_times_out(escg, monkeypatch):
    """One rank's part launched while its neighbour never runs (a dead rank): the kernel's bounded
    waits give up (ESCG_RING_TIMEOUT_S) and the host raises instead of hanging."""
    import ctypes as C

    from paper_2508_16639_b200 import _lib
    from paper_2508_16639_b200.bands import RingGroup

    monkeypatch.setenv("ESCG_RING_TIMEOUT_S", "0.5")
    p = _params(escg, 1024, 128, 3, 1e-2, 0.1, 77, 10)
    with RingGroup(p, escg.make_circulant(3, [1]), 2) as grp:
        grp.init_lattice()
        h = grp._h[0]
        _lib.check(_lib.lib().escg_dev_advance(h, 2))  # part 1 never launches
        out = np.zeros(64 * 1024, np.int32)
        m = C.c_int64(0)
        with pytest.raises(escg.EngineError, match="stopped answering"):
            _lib.check(_lib.lib().escg_dev_get_lattice(h, 0, out.ctypes.data_as(C.c_void_p), C.byref(m)))


def test_ring_parts_reject_band_entry_points(escg):
    """A ring part is advanced only by ring launches: run, band step and band-group advance refuse it."""
    import ctypes as C

    from paper_2508_16639_b200 import _lib
    from paper_2508_16639_b200.bands import RingGroup

    p = _params(escg, 1024, 128, 3, 1e-2, 0.1, 78, 10)
    with RingGroup(p, escg.make_circulant(3, [1]), 2) as grp:
        h = grp._h[0]
        L = _lib.lib()
        with pytest.raises(escg.ConfigError, match="ring parts"):
            _lib.check(L.escg_dev_run(h, 5, 1, 0, -1, 0, None))
        with pytest.raises(escg.ConfigError, match="not a band engine"):
            _lib.check(L.escg_dev_band_step(h, 1))
        arr = (C.c_void_p * 2)(*[x.value for x in grp._h])
        with pytest.raises(escg.ConfigError, match="ring parts"):
            _lib.check(L.escg_group_advance(arr, 2, 1))
