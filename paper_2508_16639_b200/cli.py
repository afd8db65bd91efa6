"""Command-line surface (flags of PAPER.md Tables 3.1/3.2) over the device engine.

    python -m paper_2508_16639_b200 run    [--length 200 --height 200 --mcs 100000 --neighbourhood 4
                                            --printFrequency 200 --mobility 3e-05 --species 3 --flux true
                                            --empty 0.0 --save false --dominance false --numRandoms 100000000
                                            --maxStep false --seed S --mode serial|parallel|maxstep
                                            --out DIR --dominanceFile dominance.csv --device 0]
    python -m paper_2508_16639_b200 resume --out DIR          (or: run --resume true)
    python -m paper_2508_16639_b200 sweep  --alphas 0.1,0.2 --length 100 --trials 20 [--mcs 0]
    python -m paper_2508_16639_b200 bench  --sizes 100,200 --mcs 1000 --runs 3
    python -m paper_2508_16639_b200 tune   --length 200 --multipliers 1,5,10 --mcs 1000

Exit codes: 0 completed/stasis/stopped, 2 usage/config, 3 I/O, 4 format, 5 engine.
Console: "mcs,<density_0>,...,<density_S>" every printFrequency MCS (engine.cpp:21-30).
"""
from __future__ import annotations

import argparse
import os
import sys

from . import experiments as X
from . import persistence as P
from .engine import (EngineMode, Neighbourhood, RunHooks, SimParams, align_num_randoms, make_circulant, simulate)
from .errors import ConfigError, EngineError, FormatError, IoError

EXIT = {ConfigError: 2, IoError: 3, FormatError: 4, EngineError: 5}


class UsageError(ConfigError):
    pass


def _bool(text: str) -> bool:
    if text in ("true", "1"):
        return True
    if text in ("false", "0"):
        return False
    raise UsageError("invalid boolean '%s'" % text)


def _nb(text: str) -> Neighbourhood:
    try:
        v = int(text)
    except ValueError:
        raise UsageError("invalid neighbourhood '%s'" % text)
    if v not in (4, 8):
        raise UsageError("neighbourhood must be 4 or 8 (got '%s')" % text)
    return Neighbourhood(v)


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="paper_2508_16639_b200", description="B200 ESCG Monte Carlo engine")
    sub = ap.add_subparsers(dest="cmd")
    run = sub.add_parser("run")
    resume = sub.add_parser("resume")
    for p in (run, resume):
        d = SimParams()
        p.add_argument("--length", type=int, default=d.length)
        p.add_argument("--height", type=int, default=d.height)
        p.add_argument("--mcs", type=int, default=d.mcs_limit)
        p.add_argument("--neighbourhood", type=_nb, default=d.neighbourhood)
        p.add_argument("--printFrequency", type=int, default=d.print_frequency)
        p.add_argument("--mobility", type=float, default=d.mobility)
        p.add_argument("--species", type=int, default=d.species)
        p.add_argument("--flux", type=_bool, default=d.flux)
        p.add_argument("--empty", type=float, default=d.empty_prob)
        p.add_argument("--save", type=_bool, default=d.save)
        p.add_argument("--dominance", type=_bool, default=d.dominance_import)
        p.add_argument("--resume", type=_bool, default=d.resume)
        p.add_argument("--numRandoms", type=int, default=d.num_randoms)
        p.add_argument("--maxStep", type=_bool, default=d.max_step)
        p.add_argument("--seed", type=int, default=None)
        p.add_argument("--mode", default=None, choices=["serial", "parallel", "maxstep"])
        p.add_argument("--out", default=".")
        p.add_argument("--dominanceFile", default="dominance.csv")
        p.add_argument("--device", type=int, default=0)
    sw = sub.add_parser("sweep")
    sw.add_argument("--alphas", required=True)
    sw.add_argument("--beta", type=float, default=0.75)
    sw.add_argument("--gamma", type=float, default=1.0)
    sw.add_argument("--length", type=int, default=100)
    sw.add_argument("--trials", type=int, default=20)
    sw.add_argument("--mcs", type=int, default=0)
    sw.add_argument("--seed", type=int, default=1)
    sw.add_argument("--csv", default="sweep.csv")
    be = sub.add_parser("bench")
    be.add_argument("--sizes", default="100,200")
    be.add_argument("--modes", default="serial,maxstep")
    be.add_argument("--mcs", type=int, default=1000)
    be.add_argument("--runs", type=int, default=3)
    be.add_argument("--warmups", type=int, default=1)
    be.add_argument("--seed", type=int, default=1)
    be.add_argument("--csv", default="bench.csv")
    tu = sub.add_parser("tune")
    tu.add_argument("--length", type=int, default=200)
    tu.add_argument("--multipliers", default="1,5,10,50")
    tu.add_argument("--mcs", type=int, default=1000)
    tu.add_argument("--seed", type=int, default=1)
    tu.add_argument("--csv", default="tune.csv")
    return ap


def params_from(ns) -> SimParams:
    """Flags → SimParams; numRandoms is aligned right after parsing."""
    p = SimParams(length=ns.length, height=ns.height, mcs_limit=ns.mcs, neighbourhood=ns.neighbourhood,
                  print_frequency=ns.printFrequency, mobility=ns.mobility, species=ns.species, flux=ns.flux,
                  empty_prob=ns.empty, save=ns.save, dominance_import=ns.dominance, resume=ns.resume,
                  num_randoms=ns.numRandoms, max_step=ns.maxStep, seed=ns.seed)
    p.validate()
    p.num_randoms = align_num_randoms(p.num_randoms, p.cells())
    return p


def _mode(ns, p: SimParams) -> EngineMode:
    if ns.mode:
        return X.parse_engine_mode(ns.mode)
    return EngineMode.MaxStep if p.max_step else EngineMode.Serial


def cmd_run(ns, out=sys.stdout) -> int:
    resume_state = None
    if ns.cmd == "resume" or ns.resume:
        cp = P.load_checkpoint(ns.out)
        p, model = cp.params, cp.dominance
        if ns.mcs != SimParams().mcs_limit:
            p.mcs_limit = ns.mcs
        resume_state = P.resume_state(cp)
        p.num_randoms = align_num_randoms(p.num_randoms, p.cells())
    else:
        p = params_from(ns)
        model = P.import_dominance(ns.dominanceFile) if p.dominance_import else make_circulant(p.species, [1]) \
            if p.species >= 2 else None
        if model is None:
            from .engine import DominanceModel
            import numpy as np

            model = DominanceModel(1, DominanceModel.Kind.Binary, np.zeros(1))
    odir = None
    if p.save:
        odir = ns.out if resume_state is not None else os.path.join(ns.out, P.output_dir_name(p))
        os.makedirs(odir, exist_ok=True)
    res = simulate(p, model, _mode(ns, p), hooks=RunHooks(console=out), resume_from=resume_state, device=ns.device)
    if odir:
        P.export_densities(res.state.trace, os.path.join(odir, "densities.csv"), append=resume_state is not None)
        P.save_checkpoint(odir, p, res.state.lattice, model, res.state.current_mcs)
    return 0


def main(argv=None, out=sys.stdout) -> int:
    try:
        ns = build_parser().parse_args(argv)
        if ns.cmd in (None, "run", "resume"):
            if ns.cmd is None:
                ns = build_parser().parse_args(["run"] + list(argv or []))
            return cmd_run(ns, out)
        if ns.cmd == "sweep":
            spec = X.SweepSpec(alphas=[float(a) for a in ns.alphas.split(",")], beta=ns.beta, gamma=ns.gamma,
                               length=ns.length, trials=ns.trials, mcs=ns.mcs, seed=ns.seed)
            X.write_sweep_csv(X.run_park_sweep(spec), ns.csv)
            return 0
        if ns.cmd == "bench":
            modes = [X.parse_engine_mode(m) for m in ns.modes.split(",")]
            rows = X.run_bench_matrix([int(s) for s in ns.sizes.split(",")], modes, ns.mcs, ns.runs, ns.warmups, ns.seed)
            X.write_bench_csv(rows, ns.mcs, ns.csv)
            return 0
        if ns.cmd == "tune":
            rows = X.run_tuning_curve(ns.length, [int(m) for m in ns.multipliers.split(",")], ns.mcs, ns.seed)
            X.write_tuning_csv(rows, ns.length, ns.mcs, ns.csv)
            return 0
        return 2
    except (ConfigError, IoError, FormatError, EngineError) as e:
        print("error: %s" % e, file=sys.stderr)
        return EXIT.get(type(e), 2 if isinstance(e, ConfigError) else 5)
