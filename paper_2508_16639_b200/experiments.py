"""Replica-batched experiment harness on the device.

Mirror of the reference's experiments module (include/escg/experiments.hpp, src/experiments.cpp).
The reference runs IID trials sequentially (experiments.cpp:98-117).  Here every trial is a replica
lattice with seed `seed + t` (experiments.cpp:26 trial_seed):

* replicas of one configuration run concurrently (one CTA per lattice for small L);
* the `on_record` predicates the reference installs become on-device stop rules:
  Paper extinction → Stopped (experiments.cpp:106-113), stasis, limit;
* under torch.distributed the trials are sharded across ranks with no data-path collective
  (`dist.run_sharded`).

The CSV writers reproduce experiments.cpp:242-285 byte-for-byte (format_double =
persistence.cpp:57-62, std::to_chars shortest round-trip).
"""
from __future__ import annotations

import decimal
import math
import statistics
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import dist
from .engine import (PAPER_SPECIES, DeviceEngine, EngineMode, RunStatus, SimParams, _interval, make_circulant,
                     make_park8, make_rpsls_ablated, simulate)
from .errors import ConfigError, IoError

# replicas per engine (bounded so the per-replica trace/counts buffers stay small)
MAX_REPLICAS_PER_ENGINE = 4096


# ---------------------------------------------------------------------------------------------
# stats.cpp:9-21 and persistence.cpp:57-62
# ---------------------------------------------------------------------------------------------

@dataclass
class MeanStd:
    """stats.hpp:8-12: sample mean / std (n-1), std 0 when n < 2."""

    mean: float = 0.0
    std_dev: float = 0.0
    n: int = 0


def mean_std(xs: Sequence[float]) -> MeanStd:
    """stats.cpp:9-21"""
    r = MeanStd(n=len(xs))
    if not xs:
        return r
    s = 0.0
    for x in xs:
        s += x
    r.mean = s / len(xs)
    if len(xs) < 2:
        return r
    sq = 0.0
    for x in xs:
        sq += (x - r.mean) * (x - r.mean)
    r.std_dev = math.sqrt(sq / (len(xs) - 1))
    return r


def format_double(v: float) -> str:
    """persistence.cpp:57-62: std::to_chars(double) — shortest round-trip digits, fixed or scientific
    notation, whichever is shorter (fixed on ties)."""
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    if math.isinf(v) or math.isnan(v):
        return ("-" if v < 0 else "") + ("inf" if math.isinf(v) else "nan")
    sign = "-" if v < 0 else ""
    t = decimal.Decimal(repr(abs(v))).normalize().as_tuple()
    d = "".join(str(x) for x in t.digits)
    e = t.exponent
    point = len(d) + e  # digits before the decimal point
    if e >= 0:  # integral at shortest precision: printf-%f style prints the exact integer value
        fixed = str(int(abs(v)))
    elif point > 0:
        fixed = d[:point] + "." + d[point:]
    else:
        fixed = "0." + "0" * (-point) + d
    se = point - 1
    sci = d[0] + ("." + d[1:] if len(d) > 1 else "") + "e" + ("+" if se >= 0 else "-") + "%02d" % abs(se)
    return sign + (fixed if len(fixed) <= len(sci) else sci)


# ---------------------------------------------------------------------------------------------
# Result types (experiments.hpp)
# ---------------------------------------------------------------------------------------------

@dataclass
class ExtinctionStats:
    """experiments.hpp:37-44"""

    times: List[int] = field(default_factory=list)
    censored: List[bool] = field(default_factory=list)
    budget: int = 0

    def in_window(self, lo: int, hi: int) -> int:
        """experiments.cpp:78-83"""
        return sum(1 for t, c in zip(self.times, self.censored) if not c and lo <= t <= hi)

    def summary(self) -> MeanStd:
        """experiments.cpp:85-90"""
        return mean_std([float(t) for t, c in zip(self.times, self.censored) if not c])


@dataclass
class CoexistenceResult:
    """experiments.hpp:51-55"""

    trials: int = 0
    coexisting: int = 0
    probability: float = 0.0


@dataclass
class SweepSpec:
    """experiments.hpp:63-72"""

    alphas: List[float] = field(default_factory=list)
    beta: float = 0.75
    gamma: float = 1.0
    length: int = 100
    trials: int = 20
    mcs: int = 0  # 0 selects the L^2 default
    mode: EngineMode = EngineMode.Serial
    seed: int = 1


@dataclass
class SurvivalCell:
    alpha: float = 0.0
    species: int = 0
    survival_prob: float = 0.0
    std_dev: float = 0.0
    trials: int = 0
    single_trial: bool = False


@dataclass
class SurvivalTable:
    cells: List[SurvivalCell] = field(default_factory=list)


@dataclass
class BenchRow:
    """experiments.hpp:90-99 (workers = GPUs used)"""

    length: int = 0
    mode: EngineMode = EngineMode.Serial
    mean_s: float = 0.0
    std_s: float = 0.0
    median_s: float = 0.0
    runs: int = 0
    workers: int = 1
    seed: int = 0


@dataclass
class TuneRow:
    multiplier: int = 0
    num_randoms: int = 0
    seconds: float = 0.0


def trial_seed(base: int, trial: int) -> int:
    """experiments.cpp:26"""
    return (int(base) + int(trial)) & 0xFFFFFFFFFFFFFFFF


def engine_mode_name(mode: EngineMode) -> str:
    """experiments.cpp:37-44"""
    return {EngineMode.Serial: "serial", EngineMode.ParallelMcs: "parallel", EngineMode.MaxStep: "maxstep"}[
        EngineMode(mode)]


def parse_engine_mode(name: str) -> EngineMode:
    """experiments.cpp:46-51"""
    table = {"serial": EngineMode.Serial, "parallel": EngineMode.ParallelMcs, "maxstep": EngineMode.MaxStep}
    if name not in table:
        raise ConfigError("unknown engine mode '%s'" % name)
    return table[name]


# ---------------------------------------------------------------------------------------------
# Replica runner (one configuration, many seeds) — sharded over ranks when distributed
# ---------------------------------------------------------------------------------------------

def run_replicas(params: SimParams, model, seeds: Sequence[int], mode: EngineMode = EngineMode.Serial,
                 tracked: int = 0, device: Optional[int] = None):
    """Run one lattice per seed to params.mcs_limit under `mode`'s record cadence with the device stop
    rules; returns [(stop MCS, RunStatus, final counts)] in seed order (all ranks' results on rank 0)."""
    interval = _interval(params, EngineMode(mode))

    def runner(part):
        out = []
        for b in range(0, len(part), MAX_REPLICAS_PER_ENGINE):
            chunk = list(part[b:b + MAX_REPLICAS_PER_ENGINE])
            dev = device
            if dev is None:
                try:
                    import torch

                    dev = torch.cuda.current_device() if torch.cuda.is_available() else 0
                except Exception:
                    dev = 0
            with DeviceEngine(params, model, n_replicas=len(chunk), seeds=chunk, device=dev) as eng:
                eng.init_lattice()
                eng.run(params.mcs_limit, interval=interval, tracked=tracked, record_trace=False)
                for r in range(len(chunk)):
                    m, st, last = eng.replica_result(r)
                    out.append((int(m), RunStatus(st), [int(c) for c in last]))
        return out

    return dist.run_sharded(list(seeds), runner)


def run_ablated_rpsls(length: int, trials: int, mcs: int, seed: int, mode: EngineMode = EngineMode.Serial,
                      pool=None, device: Optional[int] = None) -> ExtinctionStats:
    """experiments.cpp:92-119 — Paper (species 4) extinction MCS per trial; censored at the budget."""
    if trials < 1:
        raise ConfigError("trials must be at least 1")
    params = SimParams(length=length, height=length, species=5, mcs_limit=mcs, seed=seed)
    res = run_replicas(params, make_rpsls_ablated(), [trial_seed(seed, t) for t in range(trials)], mode,
                       tracked=PAPER_SPECIES, device=device)
    st = ExtinctionStats(budget=mcs)
    for m, status, last in res:
        extinct = status == RunStatus.Stopped
        st.times.append(m if extinct else mcs)
        st.censored.append(not extinct)
    return st


def run_coexistence_probe(mobility: float, length: int, mcs: int, trials: int, seed: int = 1,
                          mode: EngineMode = EngineMode.Serial, pool=None,
                          device: Optional[int] = None) -> CoexistenceResult:
    """experiments.cpp:121-141 — three species, empty 0.1; success = all three alive at the end."""
    if trials < 1:
        raise ConfigError("trials must be at least 1")
    params = SimParams(length=length, height=length, species=3, mobility=mobility, empty_prob=0.1, mcs_limit=mcs,
                       seed=seed)
    res = run_replicas(params, make_circulant(3, [1]), [trial_seed(seed, t) for t in range(trials)], mode,
                       device=device)
    r = CoexistenceResult(trials=trials)
    r.coexisting = sum(1 for _, _, last in res if sum(1 for c in last[1:] if c > 0) == 3)
    r.probability = r.coexisting / trials
    return r


def run_park_sweep(spec: SweepSpec, pool=None, device: Optional[int] = None) -> SurvivalTable:
    """experiments.cpp:143-178 — park8 immobile variant, survival probability per species per alpha."""
    if spec.trials < 1:
        raise ConfigError("trials must be at least 1")
    if not spec.alphas:
        raise ConfigError("sweep needs at least one alpha value")
    mcs = spec.mcs if spec.mcs > 0 else spec.length * spec.length
    table = SurvivalTable()
    for alpha in spec.alphas:
        model = make_park8(alpha, spec.beta, spec.gamma)
        params = SimParams(length=spec.length, height=spec.length, species=8, mobility=0.0, mcs_limit=mcs,
                           seed=spec.seed)
        res = run_replicas(params, model, [trial_seed(spec.seed, t) for t in range(spec.trials)], spec.mode,
                           device=device)
        for s in range(1, 9):
            stat = mean_std([1.0 if last[s] > 0 else 0.0 for _, _, last in res])
            table.cells.append(SurvivalCell(alpha=alpha, species=s, survival_prob=stat.mean, std_dev=stat.std_dev,
                                            trials=spec.trials, single_trial=spec.trials == 1))
    return table


def _run_timed(params, model, mode, device):
    """experiments.cpp:28-33 — wall time of one simulate() call."""
    t0 = time.perf_counter()
    simulate(params, model, mode, device=device or 0)
    return time.perf_counter() - t0


def run_bench_matrix(sizes: Sequence[int], modes: Sequence[EngineMode], mcs: int, runs: int, warmups: int,
                     seed: int, pool=None, num_randoms: int = 0, device: Optional[int] = None) -> List[BenchRow]:
    """experiments.cpp:180-213 on the device engine (workers = 1 GPU)."""
    if runs < 1:
        raise ConfigError("bench needs at least one measured run")
    rows = []
    model = make_circulant(3, [1])
    for length in sizes:
        for mode in modes:
            params = SimParams(length=length, height=length, mcs_limit=mcs, seed=seed,
                               num_randoms=num_randoms if num_randoms > 0 else 100 * length * length)
            for _ in range(warmups):
                _run_timed(params, model, mode, device)
            secs = [_run_timed(params, model, mode, device) for _ in range(runs)]
            st = mean_std(secs)
            rows.append(BenchRow(length=length, mode=EngineMode(mode), mean_s=st.mean, std_s=st.std_dev,
                                 median_s=sorted(secs)[len(secs) // 2], runs=runs, workers=1, seed=seed))
    return rows


def run_tuning_curve(length: int, multipliers: Sequence[int], mcs: int, seed: int, pool=None, warmups: int = 1,
                     device: Optional[int] = None) -> List[TuneRow]:
    """experiments.cpp:215-240.  On the device numRandoms only sets the record cadence (MaxStep)."""
    if not multipliers:
        raise ConfigError("tuning curve needs at least one multiplier")
    model = make_circulant(3, [1])
    rows, warmed = [], False
    for mult in multipliers:
        params = SimParams(length=length, height=length, mcs_limit=mcs, num_randoms=mult * length * length,
                           max_step=True, seed=seed)
        if not warmed:
            for _ in range(warmups):
                _run_timed(params, model, EngineMode.MaxStep, device)
            warmed = True
        rows.append(TuneRow(multiplier=mult, num_randoms=params.num_randoms,
                            seconds=_run_timed(params, model, EngineMode.MaxStep, device)))
    return rows


# ---------------------------------------------------------------------------------------------
# CSV emission (experiments.cpp:242-285)
# ---------------------------------------------------------------------------------------------

def _open_csv(path):
    try:
        return open(path, "w", newline="")
    except OSError:
        raise IoError("cannot open %s for writing" % path)


def write_extinction_csv(stats: ExtinctionStats, path) -> None:
    with _open_csv(path) as out:
        out.write("trial,extinction_mcs,censored\n")
        for i, (t, c) in enumerate(zip(stats.times, stats.censored)):
            out.write("%d,%d,%d\n" % (i, t, 1 if c else 0))


def write_coexistence_csv(result: CoexistenceResult, mobility: float, length: int, mcs: int, path) -> None:
    with _open_csv(path) as out:
        out.write("mobility,length,mcs,trials,coexisting,probability\n")
        out.write("%s,%d,%d,%d,%d,%s\n" % (format_double(mobility), length, mcs, result.trials, result.coexisting,
                                           format_double(result.probability)))


def write_sweep_csv(table: SurvivalTable, path) -> None:
    """experiments.cpp:257 (the defined 2-argument form; the header's 3-argument declaration does not
    link in the reference)."""
    with _open_csv(path) as out:
        out.write("alpha,species,survival_prob,std,n\n")
        for c in table.cells:
            out.write("%s,%d,%s,%s,%d\n" % (format_double(c.alpha), c.species, format_double(c.survival_prob),
                                            format_double(c.std_dev), c.trials))


def write_bench_csv(rows: Sequence[BenchRow], mcs: int, path) -> None:
    with _open_csv(path) as out:
        out.write("length,mode,mcs,mean_s,std_s,median_s,runs,workers,seed\n")
        for r in rows:
            out.write("%d,%s,%d,%s,%s,%s,%d,%d,%d\n" % (r.length, engine_mode_name(r.mode), mcs, format_double(r.mean_s),
                                                      format_double(r.std_s), format_double(r.median_s), r.runs,
                                                      r.workers, r.seed))


def write_tuning_csv(rows: Sequence[TuneRow], length: int, mcs: int, path) -> None:
    with _open_csv(path) as out:
        out.write("length,mcs,multiplier,num_randoms,seconds\n")
        for r in rows:
            out.write("%d,%d,%d,%d,%s\n" % (length, mcs, r.multiplier, r.num_randoms, format_double(r.seconds)))
