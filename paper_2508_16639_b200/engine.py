"""Host-side mirror of the reference's C++ simulation API over the B200 engine.

Reference interface (paths under /root/reference/proj):
  SimParams            include/escg/params.hpp:18-49
  ActionRates          include/escg/params.hpp:53-70
  DominanceModel       include/escg/dominance.hpp:13-39, src/dominance.cpp:8-42
  Lattice              include/escg/lattice.hpp:14-27
  DensityTrace/stasis  include/escg/engine.hpp:24-43
  RunState/RunHooks    include/escg/engine.hpp:45-67
  simulate             include/escg/engine.hpp:164-171, src/engine.cpp:194-240
  record_and_check     src/engine.cpp:47-57

`simulate(..., mode)` keeps the reference's record cadence for `mode` (Serial/ParallelMcs record
every MCS, MaxStep every align(numRandoms, N)/N MCS) while the update itself always runs the
device's coloured random-sequential kernel.  Draws come from counter-based Philox streams keyed by
the seed, so trajectories are statistically (not bitwise) equivalent to the reference's MT19937
runs; `DeviceEngine.replay` is the bit-exact path for injected reference draws.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import random
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import Params, check, lib, ptr
from .errors import ConfigError, EngineError


class Neighbourhood(enum.IntEnum):
    VonNeumann4 = 4
    Moore8 = 8


class EngineMode(enum.IntEnum):
    """engine.hpp:18 — selects the record cadence; the device update is the same for all."""

    Serial = 0
    ParallelMcs = 1
    MaxStep = 2


class RunStatus(enum.IntEnum):
    """engine.hpp:20"""

    Completed = 0
    Stasis = 1
    Stopped = 2


@dataclass
class SimParams:
    """params.hpp:18-49 (defaults = Table 3.1/3.2)."""

    length: int = 200
    height: int = 200
    mcs_limit: int = 100000
    neighbourhood: Neighbourhood = Neighbourhood.VonNeumann4
    print_frequency: int = 200
    mobility: float = 3e-05
    species: int = 3
    flux: bool = True
    empty_prob: float = 0.0
    save: bool = False
    dominance_import: bool = False
    resume: bool = False
    num_randoms: int = 100000000
    max_step: bool = False
    seed: Optional[int] = None

    def cells(self) -> int:
        return int(self.length) * int(self.height)

    def to_c(self, seed: Optional[int] = None) -> Params:
        p = Params()
        p.length, p.height, p.mcs_limit = int(self.length), int(self.height), int(self.mcs_limit)
        p.neighbourhood = int(self.neighbourhood)
        p.print_frequency = int(self.print_frequency)
        p.mobility = float(self.mobility)
        p.species = int(self.species)
        p.flux = 1 if self.flux else 0
        p.empty_prob = float(self.empty_prob)
        p.save, p.dominance_import, p.resume = int(self.save), int(self.dominance_import), int(self.resume)
        p.num_randoms = int(self.num_randoms)
        p.max_step = int(self.max_step)
        s = self.seed if seed is None else seed
        p.has_seed = 0 if s is None else 1
        p.seed = 0 if s is None else int(s) & 0xFFFFFFFFFFFFFFFF
        return p

    def validate(self) -> None:
        """params.hpp:37-48 (ConfigError with the reference's messages)."""
        check(_validate_params(self))


def _validate_params(p: SimParams) -> int:
    # validation is done by the library together with a dummy 1x1 model of matching size
    dom = np.zeros(int(p.species) * int(p.species)) if 1 <= int(p.species) <= 64 else np.zeros(1)
    return lib().escg_validate(C.byref(p.to_c()), dom, int(p.species), 0)


@dataclass
class ActionRates:
    """params.hpp:53-58"""

    mu: float = 1.0
    sigma: float = 1.0
    epsilon: float = 0.0
    total: float = 2.0


def action_rates(mobility: float, cells: int) -> ActionRates:
    """params.hpp:61-70 — ε = 2MN."""
    out = np.zeros(4)
    check(lib().escg_action_rates(float(mobility), int(cells), out))
    return ActionRates(*out.tolist())


def align_num_randoms(requested: int, cells: int) -> int:
    """random_batch.hpp:32-38"""
    v = lib().escg_align_num_randoms(int(requested), int(cells))
    if v < 0:
        raise ConfigError(lib().escg_dev_last_error().decode())
    return int(v)


@dataclass
class DominanceModel:
    """dominance.hpp:13-39 — flat S x S entries, row = attacker - 1."""

    class Kind(enum.IntEnum):
        Binary = 0
        Rated = 1

    size: int = 0
    kind: "DominanceModel.Kind" = 0
    entries: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def entry(self, a: int, b: int) -> float:
        return float(self.entries[(a - 1) * self.size + (b - 1)])

    def win_rate(self, a: int, b: int) -> float:
        for v in (a, b):
            if v < 0 or v > self.size:
                raise EngineError("corrupt lattice value %d" % v)
        if a == 0 or b == 0:
            return 0.0
        return self.entry(a, b)

    def dominates(self, a: int, b: int) -> bool:
        return self.win_rate(a, b) == 1.0

    def matrix(self) -> np.ndarray:
        return np.asarray(self.entries, np.float64).reshape(self.size, self.size)

    def validate(self) -> None:
        """dominance.cpp:8-21"""
        if self.size < 1 or self.size > 64:
            raise ConfigError("dominance size must be in [1, 64]")
        if np.asarray(self.entries).size != self.size * self.size:
            raise ConfigError("dominance entry count does not match size")
        p = SimParams(species=self.size)
        check(lib().escg_validate(C.byref(p.to_c()), np.ascontiguousarray(self.entries, np.float64), self.size,
                                  int(self.kind)))


def make_circulant(species: int, offsets: Sequence[int]) -> DominanceModel:
    """dominance.cpp:23-42 — C(S, K): i dominates j iff (j - i + S) mod S ∈ K."""
    if species < 2:
        raise ConfigError("circulant network needs at least 2 species")
    if len(offsets) == 0:
        raise ConfigError("circulant offset set must not be empty")
    for k in offsets:
        if k < 1 or k >= species:
            raise ConfigError("circulant offset %d out of range [1, %d]" % (k, species - 1))
    e = np.zeros(species * species)
    for i in range(species):
        for k in offsets:
            e[i * species + (i + k) % species] = 1.0
    return DominanceModel(species, DominanceModel.Kind.Binary, e)


def make_rpsls() -> DominanceModel:
    """experiments.cpp:53"""
    return make_circulant(5, [1, 2])


PAPER_SPECIES = 4  # experiments.hpp:25 kPaperSpecies


def make_rpsls_ablated() -> DominanceModel:
    """experiments.cpp:55-59 — Rock no longer crushes Scissors."""
    m = make_rpsls()
    m.entries[(1 - 1) * 5 + (2 - 1)] = 0.0
    return m


def make_park8(alpha: float, beta: float, gamma: float) -> DominanceModel:
    """experiments.cpp:61-76"""
    for rate in (alpha, beta, gamma):
        if not (0.0 <= rate <= 1.0):
            raise ConfigError("park8 rates must lie in [0, 1]")
    e = np.zeros(64)

    def edge(a, b, r):
        e[(a - 1) * 8 + (b - 1)] = r

    for i in range(1, 9):
        edge(i, i % 8 + 1, gamma)
        edge(i, (i + 1) % 8 + 1, alpha)
    edge(1, 5, beta)
    edge(3, 7, beta)
    m = DominanceModel(8, DominanceModel.Kind.Rated, e)
    m.validate()
    return m


@dataclass
class Lattice:
    """lattice.hpp:14-27 — flat row-major int32 cells, 0 = empty."""

    length: int = 0
    height: int = 0
    cells: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def size(self) -> int:
        return self.length * self.height

    def at(self, row: int, col: int) -> int:
        return int(self.cells[row * self.length + col])

    def __eq__(self, other) -> bool:
        return (isinstance(other, Lattice) and self.length == other.length and self.height == other.height
                and np.array_equal(self.cells, other.cells))


@dataclass
class DensityTrace:
    """engine.hpp:24-36"""

    steps: List[int] = field(default_factory=list)
    counts: List[np.ndarray] = field(default_factory=list)
    alive: List[int] = field(default_factory=list)

    def append(self, mcs: int, row) -> None:
        row = np.asarray(row, np.uint64)
        self.alive = [s for s in range(1, row.size) if row[s] > 0]
        self.steps.append(int(mcs))
        self.counts.append(row)


def densities(lattice: Lattice, species: int) -> np.ndarray:
    """engine.cpp:70-94 — counts[v] for v in [0, S] of a host lattice; EngineError on a value outside
    [0, S].  (Device lattices are counted in the kernels: DeviceEngine.counts.)"""
    cells = np.asarray(lattice.cells)
    bad = (cells < 0) | (cells > species)
    if bad.any():
        raise EngineError("corrupt lattice value %d" % int(cells[np.argmax(bad)]))
    return np.bincount(cells.astype(np.int64), minlength=species + 1).astype(np.uint64)


def stasis(trace: DensityTrace) -> bool:
    """engine.hpp:40-43"""
    if not trace.counts:
        raise ConfigError("stasis needs at least one density record")
    return len(trace.alive) <= 1


@dataclass
class RunState:
    """engine.hpp:45-51.  In the hooks-driven path `lattice` is exported lazily from the device."""

    lattice: Optional[Lattice] = None
    current_mcs: int = 0
    trace: DensityTrace = field(default_factory=DensityTrace)
    rates: ActionRates = field(default_factory=ActionRates)
    model: Optional[DominanceModel] = None


@dataclass
class RunHooks:
    """engine.hpp:63-67"""

    on_record: Optional[Callable[[RunState], bool]] = None
    on_save: Optional[Callable[[RunState], None]] = None
    console: Optional[io.TextIOBase] = None


@dataclass
class SimulationResult:
    """engine.hpp:164-167"""

    state: RunState
    status: RunStatus = RunStatus.Completed


def is_save_mcs(mcs: int, limit: int) -> bool:
    """engine.cpp:14-19"""
    if mcs == 0 or mcs == limit:
        return True
    lead = mcs
    while lead >= 10 and lead % 10 == 0:
        lead //= 10
    return lead in (1, 2, 5)


def print_density_line(out, mcs: int, counts, n: int) -> None:
    """engine.cpp:21-30"""
    out.write(str(mcs) + "".join(",%.6f" % (float(c) / float(n)) for c in counts) + "\n")


class DeviceEngine:
    """Handle over `escg_dev` (include/escg_dev.h): R independent lattices of one shape on one GPU."""

    def __init__(self, params: SimParams, model: DominanceModel, n_replicas: int = 1, seeds=None, device: int = 0,
                 kernel: str = "auto"):
        self.params = params
        self.model = model
        self.n_replicas = int(n_replicas)
        self.S = int(model.size)
        kern = {"auto": 0, "tile": 1, "block": 2, "ring": 3}[kernel]
        seeds_arr = None
        if seeds is not None:
            seeds_arr = np.ascontiguousarray([int(s) & 0xFFFFFFFFFFFFFFFF for s in seeds], np.uint64)
            if seeds_arr.size != self.n_replicas:
                raise ConfigError("one seed per replica required")
        seed = params.seed
        if seed is None:
            seed = random.SystemRandom().getrandbits(64)  # engine.cpp:210 random_device
        self._h = C.c_void_p()
        check(lib().escg_dev_create(C.byref(params.to_c(seed)), np.ascontiguousarray(model.entries, np.float64),
                                    self.S, int(model.kind), int(device), self.n_replicas, ptr(seeds_arr), kern,
                                    C.byref(self._h)))
        self.N = params.cells()

    def close(self) -> None:
        if self._h:
            check(lib().escg_dev_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --- lattice -----------------------------------------------------------------------------
    def init_lattice(self) -> None:
        check(lib().escg_dev_init_lattice(self._h))

    def set_lattice(self, cells, replica: int = 0, mcs: int = 0) -> None:
        cells = np.ascontiguousarray(np.asarray(cells).ravel(), np.int32)
        if cells.size != self.N:
            raise ConfigError("lattice size does not match params")
        check(lib().escg_dev_set_lattice(self._h, int(replica), cells, int(mcs)))

    def get_lattice(self, replica: int = 0) -> np.ndarray:
        out = np.zeros(self.N, np.int32)
        m = C.c_int64(0)
        check(lib().escg_dev_get_lattice(self._h, int(replica), ptr(out), C.byref(m)))
        return out

    def mcs(self, replica: int = 0) -> int:
        m = C.c_int64(0)
        check(lib().escg_dev_get_lattice(self._h, int(replica), None, C.byref(m)))
        return m.value

    def counts(self, replica: int = 0) -> np.ndarray:
        out = np.zeros(self.S + 1, np.uint64)
        check(lib().escg_dev_counts(self._h, int(replica), out))
        return out

    # --- stepping ----------------------------------------------------------------------------
    def advance(self, n_mcs: int) -> None:
        check(lib().escg_dev_advance(self._h, int(n_mcs)))

    def run(self, mcs_limit: int, interval: int = 1, stop_stasis: bool = True, tracked: int = 0,
            record_trace: bool = True) -> np.ndarray:
        flags = (_lib.ESCG_STOP_STASIS if stop_stasis else 0) | (_lib.ESCG_STOP_TRACKED if tracked >= 1 else 0)
        status = np.zeros(self.n_replicas, np.int32)
        check(lib().escg_dev_run(self._h, int(mcs_limit), int(interval), flags, int(tracked), int(record_trace),
                                 ptr(status)))
        return status

    def read_trace(self, replica: int = 0):
        n = C.c_int64(0)
        check(lib().escg_dev_read_trace(self._h, int(replica), None, None, 0, C.byref(n)))
        steps = np.zeros(max(n.value, 1), np.int64)
        counts = np.zeros(max(n.value, 1) * (self.S + 1), np.uint64)
        check(lib().escg_dev_read_trace(self._h, int(replica), ptr(steps), ptr(counts), n.value, C.byref(n)))
        k = n.value
        return steps[:k], counts[: k * (self.S + 1)].reshape(k, self.S + 1)

    def replica_result(self, replica: int = 0):
        m = C.c_int64(0)
        st = C.c_int32(0)
        last = np.zeros(self.S + 1, np.uint64)
        check(lib().escg_dev_replica_result(self._h, int(replica), C.byref(m), C.byref(st), last))
        return m.value, st.value, last

    def replay(self, w_cell, w_dir, w_act) -> None:
        a = [np.ascontiguousarray(w, np.uint32) for w in (w_cell, w_dir, w_act)]
        check(lib().escg_dev_replay(self._h, a[0], a[1], a[2], a[0].size))

    def last_timing(self):
        ms = C.c_double(0)
        n = C.c_int64(0)
        check(lib().escg_dev_last_timing(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def draw_code(self) -> int:
        """The draw format as the oracle names it (oracle/escg_oracle.c orc_crs_run `fmt`):
        0 WIDE, 1 NARROW, 2 | K << 8 SLICED with K action bit planes, 3 | K << 8 SLICED3 (undecided masks
        drawn directly)."""
        v = C.c_int32(0)
        check(lib().escg_dev_draw_format(self._h, C.byref(v)))
        return int(v.value)

    def draw_format(self) -> str:
        """'wide', 'narrow' or 'sliced' — which attempt-word layout this engine's
        draws use."""
        return {0: "wide", 1: "narrow", 2: "sliced", 3: "sliced"}[self.draw_code() & 0xFF]

    def describe(self):
        vals = [C.c_int32(0) for _ in range(4)]
        check(lib().escg_dev_describe(self._h, *[C.byref(v) for v in vals]))
        kernel, ctas, threads, smem = (v.value for v in vals)
        k, pers = C.c_int32(0), C.c_int32(0)
        check(lib().escg_dev_block_mode(self._h, C.byref(k), C.byref(pers)))
        return dict(kernel={1: "tile", 2: "block", 3: "ring"}[kernel], ctas=ctas, threads=threads, smem_bytes=smem,
                    draw_format=self.draw_format(), kmcs=k.value, persistent=bool(pers.value))


def thresholds(mobility: float, cells: int, model: DominanceModel):
    """Integer thresholds equivalent to the reference's double bucketing (escg_thresholds)."""
    xmx = np.zeros(2, np.uint32)
    T = np.zeros((model.size + 1) ** 2, np.uint32)
    check(lib().escg_thresholds(float(mobility), int(cells), np.ascontiguousarray(model.entries, np.float64),
                                int(model.size), xmx, T))
    return int(xmx[0]), int(xmx[1]), T.reshape(model.size + 1, model.size + 1)


def _interval(params: SimParams, mode: EngineMode) -> int:
    n = params.cells()
    if mode == EngineMode.MaxStep:
        return align_num_randoms(params.num_randoms, n) // n
    if mode == EngineMode.ParallelMcs:
        align_num_randoms(params.num_randoms, n)  # engine.cpp:142 (same ConfigError)
    return 1


def simulate(params: SimParams, model: DominanceModel, mode: EngineMode = EngineMode.MaxStep, pool=None,
             hooks: Optional[RunHooks] = None, streams=None, resume_from: Optional[RunState] = None,
             device: int = 0) -> SimulationResult:
    """engine.cpp:194-240 on the B200 engine (signature of engine.hpp:169-171; `pool`/`streams` are
    accepted for drop-in compatibility and ignored — the device owns its parallelism and RNG)."""
    check(_validate_params(params))
    model.validate()
    if model.size != params.species:
        raise ConfigError("species count (%d) does not match dominance size (%d)" % (params.species, model.size))
    hooks = hooks or RunHooks()
    interval = _interval(params, EngineMode(mode))
    n = params.cells()
    rates = action_rates(params.mobility, n)
    state = RunState(current_mcs=0, rates=rates, model=model)
    start_cells = None
    if resume_from is not None:
        start_cells = np.ascontiguousarray(resume_from.lattice.cells, np.int32)
        state.current_mcs = int(resume_from.current_mcs)
        state.trace = resume_from.trace if resume_from.trace is not None else DensityTrace()

    if hooks.on_record is None and hooks.on_save is None:
        # Fast path: one C-ABI call, records/stop checks on device; console lines replayed.
        S = model.size
        cap = (params.mcs_limit - state.current_mcs) // interval + 2
        steps = np.zeros(max(cap, 1), np.int64)
        counts = np.zeros(max(cap, 1) * (S + 1), np.uint64)
        cells = np.zeros(n, np.int32)
        out_mcs, n_rec, status = C.c_int64(0), C.c_int64(0), C.c_int32(0)
        seed = params.seed if params.seed is not None else random.SystemRandom().getrandbits(64)
        check(lib().escg_simulate(C.byref(params.to_c(seed)), np.ascontiguousarray(model.entries, np.float64), S,
                                  int(model.kind), int(mode), int(device), ptr(start_cells), state.current_mcs, 0, 0,
                                  ptr(cells), C.byref(out_mcs), ptr(steps), ptr(counts), cap, C.byref(n_rec),
                                  C.byref(status)))
        k = min(n_rec.value, cap)
        counts = counts[: k * (S + 1)].reshape(k, S + 1)
        for i in range(k):
            state.trace.append(int(steps[i]), counts[i].copy())
            if hooks.console is not None and steps[i] % params.print_frequency == 0:
                print_density_line(hooks.console, int(steps[i]), counts[i], n)
        state.lattice = Lattice(params.length, params.height, cells)
        state.current_mcs = out_mcs.value
        return SimulationResult(state, RunStatus(status.value))

    # Hooks path: the host drives record_and_check (engine.cpp:47-57) between device advances.
    eng = DeviceEngine(params, model, 1, device=device)
    try:
        if start_cells is not None:
            eng.set_lattice(start_cells, 0, state.current_mcs)
        else:
            eng.init_lattice()
        while True:
            state.trace.append(state.current_mcs, eng.counts(0))
            state.lattice = Lattice(params.length, params.height, eng.get_lattice(0))
            if hooks.console is not None and state.current_mcs % params.print_frequency == 0:
                print_density_line(hooks.console, state.current_mcs, state.trace.counts[-1], n)
            if params.save and hooks.on_save is not None and is_save_mcs(state.current_mcs, params.mcs_limit):
                hooks.on_save(state)
            if hooks.on_record is not None and not hooks.on_record(state):
                return SimulationResult(state, RunStatus.Stopped)
            if state.current_mcs >= params.mcs_limit:
                return SimulationResult(state, RunStatus.Completed)
            if stasis(state.trace):
                return SimulationResult(state, RunStatus.Stasis)
            adv = min(interval, params.mcs_limit - state.current_mcs)
            eng.advance(adv)
            state.current_mcs += adv
    finally:
        eng.close()
