"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact.

1. Serial replay of injected reference MT19937 draws == reference run_serial (north_star clause
   "given an injected identical random draw sequence ... bit-exact against the reference").
2. Coloured schedule (tile and block kernels) == oracle/escg_oracle.c:orc_crs_run, which applies
   the same Philox draws through the reference's double-precision elementary_step.
3. Device init == oracle crs_init; fused density records == densities() of the exported lattice.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # L, H, S, M, p0, arity, flux, model
    (8, 8, 3, 1e-4, 0.0, 4, True, "rps"),
    (64, 64, 3, 1e-4, 0.1, 4, True, "rps"),
    (48, 32, 5, 3e-5, 0.0, 4, True, "rpsls"),
    (40, 40, 5, 3e-3, 0.2, 8, True, "ablated"),
    (30, 22, 8, 0.0, 0.0, 4, False, "park8"),
    (21, 35, 3, 1e-3, 0.1, 8, False, "rps"),
]


def model_of(escg, name):
    return {
        "rps": lambda: escg.make_circulant(3, [1]),
        "rpsls": escg.make_rpsls,
        "ablated": escg.make_rpsls_ablated,
        "park8": lambda: escg.make_park8(0.15, 0.75, 1.0),
    }[name]()


def params(escg, L, H, S, M, p0, arity, flux, seed=1, mcs=100):
    return escg.SimParams(length=L, height=H, species=S, mobility=M, empty_prob=p0,
                          neighbourhood=escg.Neighbourhood(arity), flux=flux, seed=seed, mcs_limit=mcs)


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}_{c[7]}_n{c[5]}_{'flux' if c[6] else 'refl'}" for c in CASES])
def test_replay_matches_reference_serial(escg, oracle, ref, case):
    L, H, S, M, p0, arity, flux, name = case
    model = model_of(escg, name)
    seed, n_mcs = 11, 5
    n = L * H * n_mcs
    init, wc, wd, wa = oracle.serial_draws(L, H, S, p0, seed, n)
    # the injected draws are exactly the reference's own stream (random_batch.hpp:44-53)
    assert np.array_equal(init, ref.init_lattice(L, H, S, p0, seed))
    expect = oracle.apply_draws(init, L, H, model.matrix(), M, wc, wd, wa, arity=arity, flux=flux)
    if flux and arity == 4 and name == "rps":
        got_ref = ref.simulate(L, H, model.matrix(), M, p0, n_mcs, seed, arity=arity, flux=flux)["cells"]
        assert np.array_equal(expect, got_ref)
    with escg.DeviceEngine(params(escg, L, H, S, M, p0, arity, flux), model, kernel="tile" if L * H < 40000 else "auto") as eng:
        eng.set_lattice(init)
        eng.replay(wc, wd, wa)
        got = eng.get_lattice()
    assert np.array_equal(got, expect)


@pytest.mark.parametrize("name,eps", [("rps", 8.0), ("park8", 0.0), ("ablated", 60.0), ("rps", 2048.0),
                                      ("rps", 53687.0912), ("park8", 3.0)])
def test_replay_threshold_edges(escg, oracle, name, eps):
    """One injected attempt per (s, n) pair per action word at every threshold X-1, X, X+1
    (bucket edges and every interaction edge), all applied in a single device replay."""
    model = model_of(escg, name)
    S = model.size
    L, H0 = 300, 8
    # thresholds depend on (M, N) only through eps = 2MN; pick M for the target eps
    probe_N = L * H0
    xm, xi, T = escg.thresholds(eps / (2 * probe_N), probe_N, model)
    edges = sorted({int(v) + d for v in [xm, xi, *T.ravel().tolist()] for d in (-1, 0, 1) if 0 <= int(v) + d < 2 ** 32})
    edges += [0, 2 ** 32 - 1]
    pairs = [(s, nb, x) for s in range(S + 1) for nb in range(S + 1) for x in edges]
    H = max(4, -(-3 * len(pairs) // L))
    H += (-H) % 4
    N = L * H
    M = eps / (2 * N)
    rng = np.random.default_rng(5)
    lat = rng.integers(0, S + 1, N).astype(np.int32)
    wc = np.zeros(len(pairs), np.uint32)
    wd = np.full(len(pairs), 3, np.uint32)  # right neighbour
    wa = np.zeros(len(pairs), np.uint32)
    for k, (s, nb, x) in enumerate(pairs):
        c = 3 * k
        lat[c], lat[c + 1] = s, nb
        wc[k], wa[k] = c, x
    want = oracle.apply_draws(lat, L, H, model.matrix(), M, wc, wd, wa)
    with escg.DeviceEngine(params(escg, L, H, S, M, 0.0, 4, True), model, kernel="block") as eng:
        eng.set_lattice(lat)
        eng.replay(wc, wd, wa)
        got = eng.get_lattice()
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [pairs[i // 3] for i in bad[:5]]


CRS_CASES = [
    (8, 8, 3, 1e-4, 0.1, 4, True, "rps"),
    (64, 48, 3, 1e-4, 0.1, 4, True, "rps"),
    (100, 100, 5, 3e-5, 0.0, 4, True, "rpsls"),
    (40, 36, 5, 3e-3, 0.2, 8, True, "ablated"),
    (30, 22, 8, 0.0, 0.0, 4, False, "park8"),
    (21, 35, 3, 1e-3, 0.1, 8, False, "rps"),
    (13, 6, 3, 1e-2, 0.3, 4, False, "rps"),
    # periodic lattices with seams (L or H not divisible by 4: 6 or 9 colour phases)
    (50, 50, 3, 3e-5, 0.1, 4, True, "rps"),
    (21, 15, 3, 1e-3, 0.1, 8, True, "rps"),
    (7, 6, 5, 1e-2, 0.0, 4, True, "rpsls"),
    (102, 33, 3, 1e-4, 0.1, 4, True, "rps"),
    (4, 5, 3, 1e-2, 0.2, 8, True, "rps"),
    (13, 40, 8, 0.0, 0.0, 4, True, "park8"),
]


@pytest.mark.parametrize("case", CRS_CASES, ids=[f"{c[0]}x{c[1]}_{c[7]}_n{c[5]}_{'flux' if c[6] else 'refl'}" for c in CRS_CASES])
def test_tile_kernel_matches_crs_oracle(escg, oracle, case):
    L, H, S, M, p0, arity, flux, name = case
    model = model_of(escg, name)
    seed = 0x1234567890AB
    p = params(escg, L, H, S, M, p0, arity, flux, seed=seed)
    with escg.DeviceEngine(p, model, kernel="tile") as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        assert np.array_equal(init, oracle.crs_init(L, H, S, p0, seed))
        eng.advance(3)
        got3 = eng.get_lattice()
        eng.advance(4)
        got7 = eng.get_lattice()
        narrow = eng.draw_code()
    want3 = oracle.crs_run(init, L, H, model.matrix(), M, seed, 0, 3, arity=arity, flux=flux, narrow=narrow)
    assert np.array_equal(got3, want3)
    want7 = oracle.crs_run(want3, L, H, model.matrix(), M, seed, 3, 4, arity=arity, flux=flux, narrow=narrow)
    assert np.array_equal(got7, want7)


@pytest.mark.parametrize("table", ["0", "1"])
@pytest.mark.parametrize("fmt", ["wide", "narrow"])
@pytest.mark.parametrize("LH", [(64, 64), (200, 200), (96, 160), (8, 8), (100, 36)])
@pytest.mark.parametrize("arity", [4, 8])
def test_block_kernel_matches_crs_oracle(escg, oracle, LH, arity, fmt, table, monkeypatch):
    L, H = LH
    monkeypatch.setenv("ESCG_DRAW_FORMAT", fmt)
    monkeypatch.setenv("ESCG_PHASE_TABLE", table)  # both phase-geometry paths of block_phases
    model = escg.make_circulant(3, [1])
    seed = 99
    M = 1e-2 if fmt == "narrow" else 1e-3
    p = params(escg, L, H, 3, M, 0.1, arity, True, seed=seed)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(5)
        got = eng.get_lattice()
        narrow = eng.draw_code()
    assert narrow == (fmt == "narrow" and L % 8 == 0)
    want = oracle.crs_run(init, L, H, model.matrix(), M, seed, 0, 5, arity=arity, narrow=narrow)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("LH", [(64, 64), (200, 200), (96, 160), (8, 8)])
def test_tile_kernel_narrow_matches_crs_oracle(escg, oracle, LH, monkeypatch):
    L, H = LH
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "narrow")
    model = escg.make_rpsls()
    seed = 4242
    p = params(escg, L, H, 5, 3e-3, 0.0, 4, True, seed=seed)
    with escg.DeviceEngine(p, model, kernel="tile") as eng:
        assert eng.draw_code()
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(6)
        got = eng.get_lattice()
    assert np.array_equal(got, oracle.crs_run(init, L, H, model.matrix(), 3e-3, seed, 0, 6, narrow=True))


def test_block_equals_tile_kernel(escg):
    L = 200
    model = escg.make_rpsls()
    p = params(escg, L, L, 5, 3e-5, 0.0, 4, True, seed=2024)
    outs = []
    for kernel in ("tile", "block"):
        with escg.DeviceEngine(p, model, kernel=kernel) as eng:
            eng.init_lattice()
            eng.advance(40)
            outs.append(eng.get_lattice())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("kernel", ["tile", "block"])
def test_run_records_and_stop_rules(escg, oracle, kernel):
    """escg_dev_run: records at the reference cadence, counts == densities(), status rules."""
    L = 64
    model = escg.make_circulant(3, [1])
    p = params(escg, L, L, 3, 1e-4, 0.1, 4, True, seed=5, mcs=23)
    with escg.DeviceEngine(p, model, kernel=kernel) as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        st = eng.run(23, interval=5)
        steps, counts = eng.read_trace()
        final = eng.get_lattice()
        assert st[0] == escg.RunStatus.Completed
        assert steps.tolist() == [0, 5, 10, 15, 20, 23]
        assert eng.mcs() == 23
        narrow = eng.draw_code()
    want = oracle.crs_run(init, L, L, model.matrix(), 1e-4, 5, 0, 23, narrow=narrow)
    assert np.array_equal(final, want)
    assert np.array_equal(counts[-1], oracle.densities(want, 3))
    assert np.array_equal(counts[0], oracle.densities(init, 3))


def test_tracked_extinction_stops_like_on_record(escg, oracle):
    """Ablated RPSLS: stop at the first record where Paper (4) is extinct (experiments.cpp:107-113)."""
    L = 48
    model = escg.make_rpsls_ablated()
    p = params(escg, L, L, 5, 3e-5, 0.0, 4, True, seed=3, mcs=3000)
    with escg.DeviceEngine(p, model, kernel="tile") as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        st = eng.run(3000, interval=1, tracked=4)
        steps, counts = eng.read_trace()
        t = eng.mcs()
        final = eng.get_lattice()
        narrow = eng.draw_code()
    assert st[0] == escg.RunStatus.Stopped
    assert counts[-1][4] == 0 and all(c[4] > 0 for c in counts[:-1])
    assert steps[-1] == t
    assert np.array_equal(final, oracle.crs_run(init, L, L, model.matrix(), 3e-5, 3, 0, t, narrow=narrow))


def test_replicas_equal_single_runs(escg):
    L = 32
    model = escg.make_circulant(3, [1])
    seeds = [7, 8, 9, 10]
    p = params(escg, L, L, 3, 1e-3, 0.1, 4, True)
    with escg.DeviceEngine(p, model, n_replicas=4, seeds=seeds, kernel="tile") as eng:
        eng.init_lattice()
        eng.advance(50)
        batch = [eng.get_lattice(r) for r in range(4)]
    for r, s in enumerate(seeds):
        p1 = params(escg, L, L, 3, 1e-3, 0.1, 4, True, seed=s)
        with escg.DeviceEngine(p1, model, kernel="block") as eng:
            eng.init_lattice()
            eng.advance(50)
            assert np.array_equal(eng.get_lattice(), batch[r])


def test_simulate_one_call_matches_handle_path(escg, oracle):
    L = 64
    model = escg.make_circulant(3, [1])
    p = params(escg, L, L, 3, 1e-4, 0.1, 4, True, seed=77, mcs=40)
    res = escg.simulate(p, model, escg.EngineMode.ParallelMcs)
    assert res.status == escg.RunStatus.Completed and res.state.current_mcs == 40
    assert len(res.state.trace.steps) == 41
    init = oracle.crs_init(L, L, 3, 0.1, 77)
    want = oracle.crs_run(init, L, L, model.matrix(), 1e-4, 77, 0, 40)
    assert np.array_equal(res.state.lattice.cells, want)
    # hooks path (host-driven record_and_check) gives the same trajectory
    seen = []
    res2 = escg.simulate(p, model, escg.EngineMode.ParallelMcs,
                         hooks=escg.RunHooks(on_record=lambda st: seen.append(st.current_mcs) or True))
    assert seen == list(range(41))
    assert np.array_equal(res2.state.lattice.cells, want)


def test_device_replica_runner_matches_single_engine(escg):
    """dist.device_replica_runner (the per-rank body of a sharded ensemble) == per-seed engines."""
    from paper_2508_16639_b200.dist import device_replica_runner, run_sharded

    p = params(escg, 32, 32, 3, 1e-3, 0.1, 4, True, mcs=30)
    model = escg.make_circulant(3, [1])
    res = run_sharded([5, 6, 7], device_replica_runner(p, model))
    for s, (m, st, counts) in zip([5, 6, 7], res):
        q = params(escg, 32, 32, 3, 1e-3, 0.1, 4, True, seed=s, mcs=30)
        with escg.DeviceEngine(q, model, kernel="block") as eng:
            eng.init_lattice()
            eng.run(30, interval=1, record_trace=False)
            assert eng.replica_result(0)[2].tolist() == counts and m == 30


@pytest.mark.parametrize("LH,arity", [((320, 320), 4), ((256, 384), 8)])
def test_persistent_block_kernel_matches_oracle_and_launch_path(escg, oracle, LH, arity, monkeypatch):
    """Persistent cooperative mode (one launch per run, grid barrier between chunks) == oracle ==
    one-launch-per-chunk mode, for advance and for run() with records."""
    L, H = LH
    model = escg.make_circulant(3, [1])
    p = params(escg, L, H, 3, 3e-3, 0.1, arity, True, seed=321, mcs=11)
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ESCG_PERSISTENT", mode)
        with escg.DeviceEngine(p, model, kernel="block") as eng:
            d = eng.describe()
            assert d["persistent"] == (mode == "1"), d
            eng.init_lattice()
            init = eng.get_lattice()
            eng.advance(5)
            a5 = eng.get_lattice()
            st = eng.run(11, interval=3)
            steps, counts = eng.read_trace()
            outs[mode] = (a5, eng.get_lattice(), steps.tolist(), counts.tolist(), int(st[0]), eng.mcs(),
                          eng.draw_code())
    assert all((np.array_equal(x, y) if isinstance(x, np.ndarray) else x == y)
               for x, y in zip(outs["1"][:6], outs["0"][:6]))
    a5, fin, steps, counts, st, m, narrow = outs["1"]
    assert steps == [5, 8, 11] and st == int(escg.RunStatus.Completed) and m == 11
    want5 = oracle.crs_run(init, L, H, model.matrix(), 3e-3, 321, 0, 5, arity=arity, narrow=narrow)
    assert np.array_equal(a5, want5)
    want11 = oracle.crs_run(want5, L, H, model.matrix(), 3e-3, 321, 5, 6, arity=arity, narrow=narrow)
    assert np.array_equal(fin, want11)
    assert counts[-1] == oracle.densities(want11, 3).tolist()


def test_persistent_tracked_stop(escg, monkeypatch):
    """Early stop inside a persistent run: ablated RPSLS until Paper dies; same MCS/lattice as the
    per-launch path."""
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ESCG_PERSISTENT", mode)
        p = params(escg, 256, 256, 5, 3e-4, 0.0, 4, True, seed=9, mcs=3000)
        with escg.DeviceEngine(p, escg.make_rpsls_ablated(), kernel="block") as eng:
            eng.init_lattice()
            st = eng.run(3000, interval=1, tracked=4)
            res[mode] = (int(st[0]), eng.mcs(), eng.get_lattice(), eng.read_trace()[1][-1].tolist())
    assert res["1"][0] == res["0"][0] and res["1"][1] == res["0"][1]
    assert np.array_equal(res["1"][2], res["0"][2]) and res["1"][3] == res["0"][3]


@pytest.mark.parametrize("n_bands,kmcs,LH", [(2, 1, (96, 128)), (3, 2, (160, 160)), (4, 1, (200, 208)), (2, 2, (320, 192))])
def test_band_group_equals_single_lattice(escg, oracle, n_bands, kmcs, LH):
    """Row-band sharding (virtual bands on one GPU): bit-identical to the single-lattice engine and
    to the oracle schedule — halos, global tile ids and init offsets are exact."""
    from paper_2508_16639_b200.bands import BandGroup

    L, H = LH
    model = escg.make_circulant(3, [1])
    p = params(escg, L, H, 3, 1e-2, 0.1, 4, True, seed=555)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(7)
        single = eng.get_lattice()
        narrow = eng.draw_code()
    with BandGroup(p, model, n_bands, kmcs=kmcs) as grp:
        grp.init_lattice()
        assert np.array_equal(grp.get_lattice(), init)
        grp.advance(3)
        grp.advance(4)
        banded = grp.get_lattice()
        assert np.array_equal(grp.counts(), np.bincount(banded, minlength=4).astype(np.uint64))
    assert np.array_equal(banded, single)
    assert np.array_equal(single, oracle.crs_run(init, L, H, model.matrix(), 1e-2, 555, 0, 7, narrow=narrow))


@pytest.mark.gpu
@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2")
@pytest.mark.parametrize("fmt", ["wide", "sliced"])
def test_band_group_on_two_gpus(escg, oracle, fmt, monkeypatch):
    """Bands on two GPUs of one process: halos by peer copies between the devices (escg_group_advance),
    bit-identical to the oracle schedule (byte and bit-sliced kernels)."""
    from paper_2508_16639_b200.bands import BandGroup

    monkeypatch.setenv("ESCG_DRAW_FORMAT", fmt)
    L, H, M, seed = 512, 256, 1e-2, 909
    model = escg.make_circulant(3, [1])
    p = params(escg, L, H, 3, M, 0.1, 4, True, seed=seed)
    with BandGroup(p, model, 2, devices=[0, 1], kmcs=2) as grp:
        grp.init_lattice()
        init = grp.get_lattice()
        grp.advance(3)
        grp.advance(4)
        got = grp.get_lattice()
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        narrow = eng.draw_code()
    assert np.array_equal(got, oracle.crs_run(init, L, H, model.matrix(), M, seed, 0, 7, narrow=narrow))


@pytest.mark.gpu
@pytest.mark.parametrize("n_bands,kmcs,L,H,S", [(2, 1, 256, 128, 3), (3, 2, 384, 240, 3), (4, 2, 128, 208, 5)])
def test_sliced_band_group_equals_single_lattice(escg, oracle, n_bands, kmcs, L, H, S, monkeypatch):
    """Row bands on the bit-sliced kernel: the group stays in plane form across chunks (halos move as
    plane rows) and equals the single-lattice bit-sliced run and the oracle's SLICED schedule."""
    from paper_2508_16639_b200.bands import BandGroup

    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    model = escg.make_circulant(3, [1]) if S == 3 else escg.make_rpsls()
    p = params(escg, L, H, S, 1e-2, 0.1, 4, True, seed=808)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        assert eng.draw_format() == "sliced"
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(9)
        single = eng.get_lattice()
        narrow = eng.draw_code()
    with BandGroup(p, model, n_bands, kmcs=kmcs) as grp:
        grp.init_lattice()
        grp.advance(4)
        grp.advance(5)
        banded = grp.get_lattice()
        assert np.array_equal(grp.counts(), np.bincount(banded, minlength=S + 1).astype(np.uint64))
    assert np.array_equal(banded, single)
    assert np.array_equal(single, oracle.crs_run(init, L, H, model.matrix(), 1e-2, 808, 0, 9, narrow=narrow))


@pytest.mark.gpu
def test_sliced_band_primitives_match_single_lattice(escg, monkeypatch):
    """The multi-process band path (escg_dev_band_rows + escg_dev_band_step, byte halos) on the
    bit-sliced kernel, bands in one process: equals the single-lattice run bit for bit."""
    import torch

    from paper_2508_16639_b200._lib import check, lib
    from paper_2508_16639_b200.bands import DistributedBand

    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    L, H, n_bands, kmcs = 256, 192, 3, 2
    p = params(escg, L, H, 3, 1e-2, 0.1, 4, True, seed=32)
    model = escg.make_circulant(3, [1])
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        assert eng.draw_format() == "sliced"
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(7)
        want = eng.get_lattice()
    bands = [DistributedBand(p, model, rank=g, world=n_bands, device=0, kmcs=kmcs) for g in range(n_bands)]
    try:
        for b in bands:
            s, r = b.info["start"], b.info["rows"]
            b.set_band(init[s * L:(s + r) * L], 0)
        done = 0
        while done < 7:
            chunk = min(kmcs, 7 - done)
            views = [b.halo_views() for b in bands]
            for g in range(n_bands):
                up, dn = views[(g - 1) % n_bands], views[(g + 1) % n_bands]
                views[g][0].copy_(up[2])
                views[g][3].copy_(dn[1])
            torch.cuda.synchronize()
            for b in bands:
                check(lib().escg_dev_band_step(b._h, chunk))
            done += chunk
        got = np.concatenate([b.get_band() for b in bands])
        assert np.array_equal(got, want)
    finally:
        for b in bands:
            b.close()


def test_band_group_resume_from_host_lattice(escg):
    from paper_2508_16639_b200.bands import BandGroup

    L, H = 128, 128
    model = escg.make_rpsls()
    p = params(escg, L, H, 5, 3e-3, 0.0, 8, True, seed=77)
    rng = np.random.default_rng(1)
    start = rng.integers(0, 6, L * H).astype(np.int32)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        eng.set_lattice(start, mcs=40)
        eng.advance(6)
        single = eng.get_lattice()
    with BandGroup(p, model, 3, kmcs=2) as grp:
        grp.set_lattice(start, mcs=40)
        grp.advance(6)
        assert np.array_equal(grp.get_lattice(), single)


@pytest.mark.gpu
def test_seam_lattice_ensemble_matches_oracle(escg, oracle):
    """Replicas of a seam lattice (odd size) on the tile kernel = independent oracle runs."""
    L, H, S = 31, 29, 3
    model = escg.make_circulant(3, [1])
    p = params(escg, L, H, S, 1e-3, 0.1, 4, True, seed=5)
    with escg.DeviceEngine(p, model, n_replicas=6, seeds=range(50, 56), kernel="tile") as eng:
        assert eng.describe()["kernel"] == "tile"
        eng.init_lattice()
        init = [eng.get_lattice(r) for r in range(6)]
        eng.advance(9)
        for r in range(6):
            want = oracle.crs_run(init[r], L, H, model.matrix(), 1e-3, 50 + r, 0, 9)
            assert np.array_equal(eng.get_lattice(r), want)


@pytest.mark.gpu
def test_periodic_lattices_need_four_cells_per_side(escg):
    p = params(escg, 3, 8, 3, 1e-4, 0.1, 4, True)
    with pytest.raises(escg.ConfigError, match=">= 4"):
        escg.DeviceEngine(p, escg.make_circulant(3, [1]))


@pytest.mark.parametrize("LH,arity,kmcs,name", [((64, 64), 4, 2, "rps"), ((101, 67), 8, 1, "rps"), ((13, 6), 4, 1, "rps"),
                                                 ((600, 500), 4, 2, "rps"), ((603, 498), 8, 3, "park8"),
                                                 ((1000, 31), 4, 4, "rpsls"), ((2, 2), 4, 1, "rps")])
def test_block_kernel_reflect_matches_crs_oracle(escg, oracle, LH, arity, kmcs, name, monkeypatch):
    """Mirror-reflecting lattices (flux=false) on the block kernel: clipped windows, reflect tiling,
    boundary pairs through the explicit-coordinate path — bit-exact with the sequential oracle."""
    L, H = LH
    monkeypatch.setenv("ESCG_BLOCK_MCS", str(kmcs))
    model = model_of(escg, name)
    S = model.size
    M = 0.0 if name == "park8" else 1e-3
    p = params(escg, L, H, S, M, 0.1, arity, False, seed=4242)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        assert eng.describe()["kernel"] == "block" and eng.draw_format() == "wide"
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(7)
        got = eng.get_lattice()
        st = eng.run(12, interval=3, record_trace=True)
        steps, counts = eng.read_trace(0)
        final = eng.get_lattice()
    want = oracle.crs_run(init, L, H, model.matrix(), M, 4242, 0, 7, arity=arity, flux=False)
    assert np.array_equal(got, want)
    if st[0] == escg.RunStatus.Stasis:  # tiny lattices collapse at the first record
        assert np.array_equal(final, want) and steps.tolist() == [7]
        return
    want12 = oracle.crs_run(want, L, H, model.matrix(), M, 4242, 7, 5, arity=arity, flux=False)
    assert np.array_equal(final, want12)
    assert steps.tolist()[-1] == 12
    assert counts[-1].tolist() == np.bincount(want12, minlength=S + 1).tolist()


@pytest.mark.parametrize("LH,arity,kmcs,name", [((1002, 1000), 4, 1, "rps"), ((501, 463), 8, 1, "park8"),
                                                 ((50, 50), 4, 2, "rps"), ((21, 15), 8, 1, "rps"),
                                                 ((7, 6), 4, 1, "rpsls"), ((1000, 30), 4, 2, "rps"),
                                                 ((30, 1001), 8, 1, "rps")])
def test_block_kernel_seams_match_crs_oracle(escg, oracle, LH, arity, kmcs, name, monkeypatch):
    """Periodic lattices with seams on the block kernel (per-axis tile lists, 6/9 phases, margin
    3 x phases x MCS; small lattices make windows wrap several times) — bit-exact with the oracle."""
    L, H = LH
    monkeypatch.setenv("ESCG_BLOCK_MCS", str(kmcs))
    model = model_of(escg, name)
    S = model.size
    M = 0.0 if name == "park8" else 1e-3
    p = params(escg, L, H, S, M, 0.1, arity, True, seed=777)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        assert eng.describe()["kernel"] == "block" and eng.draw_format() == "wide"
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(5)
        got = eng.get_lattice()
        st = eng.run(9, interval=2, record_trace=True)
        steps, counts = eng.read_trace(0)
        final = eng.get_lattice()
    want = oracle.crs_run(init, L, H, model.matrix(), M, 777, 0, 5, arity=arity)
    assert np.array_equal(got, want)
    if st[0] == escg.RunStatus.Stasis:
        return
    want9 = oracle.crs_run(want, L, H, model.matrix(), M, 777, 5, 4, arity=arity)
    assert np.array_equal(final, want9)
    assert steps.tolist()[-1] == 9 and counts[-1].tolist() == np.bincount(want9, minlength=S + 1).tolist()


@pytest.mark.parametrize("n_bands,kmcs", [(2, 2), (3, 1), (4, 3)])
def test_band_primitives_match_single_lattice(escg, n_bands, kmcs):
    """The multi-process band path in one process: halo rows moved between band buffers with torch
    device copies (what NCCL send/recv does across ranks) through escg_dev_band_rows, then
    escg_dev_band_step — equals the single-lattice run bit for bit."""
    import torch

    from paper_2508_16639_b200._lib import check, lib
    from paper_2508_16639_b200.bands import DistributedBand

    L, H = 96, 192
    p = params(escg, L, H, 3, 1e-2, 0.1, 4, True, seed=31)
    model = escg.make_circulant(3, [1])
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(11)
        want = eng.get_lattice()
    bands = [DistributedBand(p, model, rank=g, world=n_bands, device=0, kmcs=kmcs) for g in range(n_bands)]
    try:
        for b in bands:
            s, r = b.info["start"], b.info["rows"]
            b.set_band(init[s * L:(s + r) * L], 0)
        done = 0
        while done < 11:
            chunk = min(kmcs, 11 - done)
            views = [b.halo_views() for b in bands]
            for g in range(n_bands):
                up, dn = views[(g - 1) % n_bands], views[(g + 1) % n_bands]
                views[g][0].copy_(up[2])  # top halo ← the band above's last rows
                views[g][3].copy_(dn[1])  # bottom halo ← the band below's first rows
            torch.cuda.synchronize()
            for b in bands:
                check(lib().escg_dev_band_step(b._h, chunk))
            done += chunk
        got = np.concatenate([b.get_band() for b in bands])
        assert np.array_equal(got, want)
        assert sum(b.counts() for b in bands).tolist() == np.bincount(want, minlength=4).tolist()
    finally:
        for b in bands:
            b.close()


@pytest.mark.parametrize("L,H,flux,arity,kernel,fmt", [(64, 64, True, 4, "tile", "narrow"), (48, 40, True, 8, "tile", "wide"),
                                                       (1024, 512, True, 4, "block", "narrow"),
                                                       (1024, 512, True, 4, "block", "sliced"),
                                                       (1000, 520, True, 4, "block", "wide"),
                                                       (501, 463, True, 8, "block", "wide"),
                                                       (333, 200, False, 4, "block", "wide"),
                                                       (51, 45, True, 4, "tile", "wide")])
def test_pure_exchange_conserves_every_species(escg, L, H, flux, arity, kernel, fmt, monkeypatch):
    """SURVEY §4.3 (criteria 3/11): with no predation (D = 0) and no empty cells only exchanges can
    fire, so every species count is conserved exactly — the invariant the reference's racy
    parallel engines violate.  Covers every kernel mode (periodic NARROW/WIDE, seams, reflect)."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", fmt)
    D = escg.DominanceModel(3, escg.DominanceModel.Kind.Binary, np.zeros(9))
    p = params(escg, L, H, 3, 1e-1, 0.0, arity, flux, seed=5)
    with escg.DeviceEngine(p, D, kernel=kernel) as eng:
        eng.init_lattice()
        c0 = eng.counts()
        init = eng.get_lattice()
        eng.advance(40)
        assert eng.counts().tolist() == c0.tolist()
        assert not np.array_equal(eng.get_lattice(), init)
        assert c0[0] == 0


def test_device_init_lattice_is_uniform(escg, ref):
    """SURVEY §4.3 criterion 12: device init_lattice species frequencies pass the reference's own
    chi-square uniformity test (stats.cpp chi_square_uniform_pvalue) and the empty fraction matches."""
    L = 2048
    p = params(escg, L, L, 5, 1e-4, 0.2, 4, True, seed=12345)
    with escg.DeviceEngine(p, escg.make_rpsls(), kernel="block") as eng:
        eng.init_lattice()
        c = eng.counts()
    n = L * L
    assert abs(c[0] / n - 0.2) < 5 * np.sqrt(0.2 * 0.8 / n)
    assert ref.chi_square_uniform(c[1:]) > 1e-3


def test_auto_kernel_choice(escg):
    """AUTO: replicas that fill the device run one CTA each (tile); a few lattices spread over all
    SMs (block) — the faster choice on B200 in both regimes (engine.cpp create_impl)."""
    p = params(escg, 200, 200, 3, 1e-4, 0.1, 4, True)
    model = escg.make_circulant(3, [1])
    with escg.DeviceEngine(p, model) as eng:
        assert eng.describe()["kernel"] == "block"
    with escg.DeviceEngine(p, model, n_replicas=296, seeds=range(296)) as eng:
        assert eng.describe()["kernel"] == "tile"
    with escg.DeviceEngine(params(escg, 3200, 3200, 3, 1e-4, 0.1, 4, True), model) as eng:
        assert eng.describe()["kernel"] == "ring"  # one bit-sliced lattice of 25 groups per row


def _fnv1a_i32(cells):
    h = 1469598103934665603
    for b in np.ascontiguousarray(cells, "<i4").tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_reference_simulate_dispatches_to_device_engine(escg, ref):
    """INTEGRATION.md §1 compiled for real: the unmodified reference with the EngineMode::Device case
    (oracle/device_patch.py) runs escg::simulate() on this engine through the C ABI; the result equals
    this package's simulate() from the same MT19937-initialised lattice, bit for bit."""
    import os
    import subprocess

    demo = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                        "escg_device_demo")
    if not os.path.exists(demo):
        pytest.skip("oracle/_ref/escg_device_demo not built (needs /root/reference at build time)")
    L, H, mcs = 64, 48, 120
    out = subprocess.run([demo, str(L), str(H), str(mcs)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    got = dict(kv.split("=") for kv in out.stdout.split())
    init = ref.init_lattice(L, H, 3, 0.1, 77)
    assert int(got["init_fnv"], 16) == _fnv1a_i32(init)
    p = escg.SimParams(length=L, height=H, species=3, mobility=1e-3, empty_prob=0.1, seed=77, mcs_limit=mcs,
                       print_frequency=1000000)
    res = escg.simulate(p, escg.make_circulant(3, [1]), escg.EngineMode.Serial,
                        resume_from=escg.RunState(lattice=escg.Lattice(L, H, init), current_mcs=0))
    assert int(got["status"]) == int(res.status) and int(got["mcs"]) == res.state.current_mcs
    assert int(got["records"]) == len(res.state.trace.counts)
    assert int(got["total"]) == L * H
    assert int(got["final_fnv"], 16) == _fnv1a_i32(res.state.lattice.cells)


# ---- bit-sliced block kernel (draw format SLICED, csrc/slice.cu) -----------------------------------

SLICED_CASES = [
    # L, H, S, M, p0, model, forced split "nby,nbx" (None: planner), ESCG_BLOCK_MCS, expected K
    (128, 128, 3, 1e-2, 0.1, "rps", None, None, 6),      # one group per row: the window wraps onto itself
    (256, 64, 3, 3e-2, 0.1, "rps", "2,2", "1", 8),
    (384, 200, 3, 1e-2, 0.0, "rps", "3,3", "2", 8),      # 3 column blocks of one group, uneven row blocks
    (512, 96, 5, 1e-2, 0.1, "rpsls", "2,3", "4", 8),     # 3 bit planes (S = 5), 4 MCS per launch
    (256, 256, 3, 5e-2, 0.2, "rps", "4,2", "3", 10),
    (1024, 128, 3, 1e-1, 0.1, "rps", "1,3", "2", 12),    # column blocks of 2, 3, 3 groups
    (1024, 256, 3, 1.0, 0.1, "rps", None, None, 16),
]


@pytest.mark.parametrize("lpi,qcap,draws", [("1", None, "3"), ("1", "1", "3"), ("2", None, "3"), ("2", "3", "3"),
                                             ("1", None, "2"), ("2", None, "2")])
@pytest.mark.parametrize("case", SLICED_CASES, ids=[f"{c[0]}x{c[1]}_{c[5]}_K{c[8]}" for c in SLICED_CASES])
def test_slice_kernel_matches_crs_oracle(escg, oracle, case, lpi, qcap, draws, monkeypatch):
    """The bit-sliced block kernel == oracle orc_crs_run with the SLICED3 (default) or SLICED draw
    spec, bit for bit: advance in two calls (bytes -> planes -> bytes between them), then run() with
    records.  One and two lanes per item; a 3-entry deferred-tile queue forces the in-place overflow
    path."""
    L, H, S, M, p0, name, split, kmax, K = case
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    monkeypatch.setenv("ESCG_SLICE_DRAWS", draws)
    monkeypatch.setenv("ESCG_SLICE_LPI", lpi)
    if qcap:
        monkeypatch.setenv("ESCG_SLICE_QCAP", qcap)
    if split:
        monkeypatch.setenv("ESCG_SLICE_SPLIT", split)
    if kmax:
        monkeypatch.setenv("ESCG_BLOCK_MCS", kmax)
    model = model_of(escg, name)
    seed = 0xC0FFEE + L
    p = params(escg, L, H, S, M, p0, 4, True, seed=seed, mcs=12)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        code = eng.draw_code()
        assert code == int(draws) | (K << 8), hex(code)
        if split:
            assert eng.describe()["ctas"] == int(split.split(",")[0]) * int(split.split(",")[1])
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


@pytest.mark.parametrize("kforce,kwant", [("10", 10), ("7", 6), ("4", 16), ("18", 16)])
def test_slice_kernel_forced_action_planes(escg, oracle, kforce, kwant, monkeypatch):
    """ESCG_SLICE_K (experiments) lowers K to an even value in [6, leading ones of X_mig]; anything
    else is ignored.  The forced format is still the oracle's SLICED definition with that K."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    monkeypatch.setenv("ESCG_SLICE_K", kforce)
    L, H, M = 1024, 256, 1.0  # X_mig has >= 16 leading ones
    model = escg.make_circulant(3, [1])
    p = params(escg, L, H, 3, M, 0.1, 4, True, seed=29, mcs=4)
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        code = eng.draw_code()
        assert code == 3 | (kwant << 8), hex(code)
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(3)
        got = eng.get_lattice()
    assert np.array_equal(got, oracle.crs_run(init, L, H, model.matrix(), M, 29, 0, 3, narrow=code))


def test_slice_kernel_replicas_and_stops(escg, oracle, monkeypatch):
    """Replica batches on the bit-sliced kernel: every replica equals its single run; a tracked
    extinction stop leaves the lattice of the stopping record (plane buffer named by `cur`)."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    L, H, M = 256, 128, 2e-2
    model = escg.make_circulant(3, [1])
    seeds = [17, 18, 19]
    p = params(escg, L, H, 3, M, 0.1, 4, True, seed=17, mcs=9)
    with escg.DeviceEngine(p, model, n_replicas=3, seeds=seeds, kernel="block") as eng:
        assert eng.draw_format() == "sliced"
        eng.init_lattice()
        inits = [eng.get_lattice(r) for r in range(3)]
        eng.advance(5)
        got = [eng.get_lattice(r) for r in range(3)]
        code = eng.draw_code()
    for r in range(3):
        assert np.array_equal(got[r], oracle.crs_run(inits[r], L, H, model.matrix(), M, seeds[r], 0, 5, narrow=code))
    # species 2 starts extinct: the run stops at its first record (MCS 0, before any step)
    cells = inits[0].copy()
    cells[cells == 2] = 1
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        eng.set_lattice(cells)
        st = eng.run(9, interval=3, tracked=2)
        assert int(st[0]) == int(escg.RunStatus.Stopped) and eng.mcs() == 0
        assert np.array_equal(eng.get_lattice(), cells)


@pytest.mark.parametrize("L,H,kmcs", [(4480, 3364, 2), (16384, 1024, 2), (1024, 512, 1)])
def test_band_engines_keep_their_chunk(escg, L, H, kmcs):
    """Band engines run exactly the chunk (halo depth) they were created with — the planner searches
    only the split — so every band of a lattice exchanges halos at the same cadence (ADVICE r01:
    4480 x 3364 in 2 bands used to plan k=2 and k=1 for its two bands)."""
    from paper_2508_16639_b200 import bands

    p = escg.SimParams(length=L, height=H, species=3, mobility=1e-4, empty_prob=0.1, seed=3, mcs_limit=10)
    with bands.BandGroup(p, escg.make_circulant(3, [1]), 2, kmcs=kmcs) as g:
        assert [i["kmcs"] for i in g.info] == [kmcs, kmcs], g.info
        assert [i["halo"] for i in g.info] == [12 * kmcs, 12 * kmcs], g.info


def test_simulate_reuses_engine_with_new_seed(escg, oracle):
    """escg_simulate caches its engine by shape, model and environment, not by seed: a new seed on
    the cached engine gives that seed's run (equal to a fresh engine's), and the old seed again
    reproduces the first result."""
    L = 128
    p1 = escg.SimParams(length=L, height=L, species=3, mobility=1e-3, empty_prob=0.1, seed=11, mcs_limit=30)
    p2 = escg.SimParams(length=L, height=L, species=3, mobility=1e-3, empty_prob=0.1, seed=12, mcs_limit=30)
    model = escg.make_circulant(3, [1])
    r1 = escg.simulate(p1, model, escg.EngineMode.Serial).state.lattice.cells
    r2 = escg.simulate(p2, model, escg.EngineMode.Serial).state.lattice.cells
    r1b = escg.simulate(p1, model, escg.EngineMode.Serial).state.lattice.cells
    assert not np.array_equal(r1, r2)
    assert np.array_equal(r1, r1b)
    with escg.DeviceEngine(p2, model) as eng:
        eng.init_lattice()
        eng.run(30, interval=1)
        assert np.array_equal(eng.get_lattice(), r2)


@pytest.mark.parametrize("fmt", ["narrow", "sliced"])
def test_band_steps_ordered_on_the_caller_stream(escg, fmt, monkeypatch):
    """Device-ordered band stepping (escg_dev_set_stream, what bands.DistributedBand does with NCCL):
    halo copies and band steps enqueued on one torch stream with no host synchronisation between
    them give the single-lattice run bit for bit."""
    import torch

    from paper_2508_16639_b200._lib import check, lib
    from paper_2508_16639_b200.bands import DistributedBand

    monkeypatch.setenv("ESCG_DRAW_FORMAT", fmt)
    L, H, n_bands, kmcs, T = 1024, 256, 3, 2, 9
    p = params(escg, L, H, 3, 5e-2, 0.1, 4, True, seed=41)
    model = escg.make_circulant(3, [1])
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        assert eng.draw_format() == fmt
        eng.init_lattice()
        init = eng.get_lattice()
        eng.advance(T)
        want = eng.get_lattice()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        bands = [DistributedBand(p, model, rank=g, world=n_bands, device=0, kmcs=kmcs) for g in range(n_bands)]
    try:
        for b in bands:
            s, r = b.info["start"], b.info["rows"]
            b.set_band(init[s * L:(s + r) * L], 0)
        with torch.cuda.stream(stream):
            done = 0
            while done < T:
                chunk = min(kmcs, T - done)
                views = [b.halo_views() for b in bands]
                for g in range(n_bands):
                    up, dn = views[(g - 1) % n_bands], views[(g + 1) % n_bands]
                    views[g][0].copy_(up[2])
                    views[g][3].copy_(dn[1])
                for b in bands:
                    check(lib().escg_dev_band_step(b._h, chunk))
                done += chunk
        got = np.concatenate([b.get_band() for b in bands])
        assert np.array_equal(got, want)
    finally:
        for b in bands:
            b.close()


@pytest.mark.gpu
def test_sliced_state_stays_in_planes_across_calls(escg, oracle, monkeypatch):
    """A single bit-sliced lattice keeps its state in bit planes between run/advance calls (no
    conversion per call); every mix of run, advance, reads, counts and host writes must still be the
    oracle's schedule."""
    monkeypatch.setenv("ESCG_DRAW_FORMAT", "sliced")
    L, H, M, seed = 512, 128, 1e-2, 4321
    model = escg.make_circulant(3, [1])
    p = params(escg, L, H, 3, M, 0.1, 4, True, seed=seed)
    D = model.matrix()
    with escg.DeviceEngine(p, model, kernel="block") as eng:
        code = eng.draw_code()
        assert code & 0xFF in (2, 3)
        eng.init_lattice()
        cur = eng.get_lattice()
        t = 0
        for op, n in (("run", 5), ("advance", 3), ("advance", 2), ("run", 4), ("get", 0), ("run", 3), ("advance", 1)):
            if op == "run":
                st = eng.run(t + n, interval=2)
                assert int(st[0]) == int(escg.RunStatus.Completed)
            elif op == "advance":
                eng.advance(n)
            if n:
                cur = oracle.crs_run(cur, L, H, D, M, seed, t, n, narrow=code)
                t += n
            if op == "get" or op == "advance":
                assert np.array_equal(eng.get_lattice(), cur), (op, t)
        assert np.array_equal(eng.counts(), np.bincount(cur, minlength=4).astype(np.uint64))
        cells = np.random.default_rng(3).integers(0, 4, L * H).astype(np.int32)
        eng.set_lattice(cells, mcs=t)
        eng.advance(2)
        assert np.array_equal(eng.get_lattice(), oracle.crs_run(cells, L, H, D, M, seed, t, 2, narrow=code))
