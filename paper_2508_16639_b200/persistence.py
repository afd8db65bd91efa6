"""Checkpoint / CSV formats of the reference, for device runs.

Byte-compatible with include/escg/persistence.hpp + src/persistence.cpp:
  grid.csv       H rows of L comma-separated cells, then the saved MCS      (persistence.cpp:72-123)
  params.csv     key,value rows in CLI-flag order (+ seed when set)         (persistence.cpp:134-205)
  dominance.csv  S x S; Binary as integers, Rated via format_double          (persistence.cpp:207-258)
  densities.csv  mcs,count_0..count_S rows (header when fresh)              (persistence.cpp:295-309)
  output_dir_name(params)                                                    (persistence.cpp:311-320)
  save_checkpoint / load_checkpoint with the same cross-validation           (persistence.cpp:322-351)

The device RNG state is (seed, MCS): params.csv carries the seed and grid.csv the MCS, so a device
checkpoint resumes bit-exactly without a streams.csv (the reference's MT19937 state dump).
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .engine import DensityTrace, DominanceModel, Lattice, Neighbourhood, RunState, SimParams
from .errors import FormatError, IoError
from .experiments import format_double

PARAM_KEYS = ["length", "height", "mcs", "neighbourhood", "printFrequency", "mobility", "species", "flux", "empty",
              "save", "dominance", "resume", "numRandoms", "maxStep"]


def _open_out(path, append=False):
    try:
        return open(path, "a" if append else "w", newline="")
    except OSError:
        raise IoError("cannot open %s for writing" % path)


def _open_in(path):
    try:
        return open(path, "r", newline="")
    except OSError:
        raise IoError("cannot open %s for reading" % path)


def _lines(f):
    """std::getline over the file with strip_cr (persistence.cpp:22-25)."""
    text = f.read()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    return [ln[:-1] if ln.endswith("\r") else ln for ln in lines]


def _split_csv(line):
    """persistence.cpp:13-20 (a trailing comma yields an empty last field)."""
    if line == "":
        return []
    return line.split(",")


_INT_RE = re.compile(r"-?[0-9]+\Z")


def _parse_int(text, what):
    """persistence.cpp:39-45 (std::from_chars into int64): optional '-', ASCII digits only, the whole
    field, in range."""
    if not _INT_RE.match(text) or not (-(1 << 63) <= int(text) < (1 << 63)):
        raise FormatError("invalid integer '%s' for %s" % (text, what))
    return int(text)


def _parse_double(text, what):
    try:
        if text != text.strip() or text == "" or text.lower() in ("inf", "-inf", "nan", "infinity"):
            raise ValueError
        return float(text)
    except ValueError:
        raise FormatError("invalid number '%s' for %s" % (text, what))


def parse_double(text: str, what: str) -> float:
    """persistence.hpp parse_double: FormatError naming `what` on anything but a finite number."""
    return _parse_double(text, what)


def _parse_bool(text, what):
    if text in ("true", "1"):
        return True
    if text in ("false", "0"):
        return False
    raise FormatError("invalid boolean '%s' for %s" % (text, what))


def _bool_str(v):
    return "true" if v else "false"


# ---- grid -------------------------------------------------------------------------------------

def export_grid(lattice: Lattice, mcs: int, path) -> None:
    cells = np.asarray(lattice.cells).reshape(lattice.height, lattice.length)
    with _open_out(path) as out:
        out.write("".join(",".join(map(str, row.tolist())) + "\n" for row in cells))
        out.write("%d\n" % mcs)


def import_grid(path):
    with _open_in(path) as f:
        lines = _lines(f)
    rows, width = [], 0
    mcs, have_mcs = 0, False
    for i, line in enumerate(lines):
        lineno = i + 1
        last = i == len(lines) - 1
        if line == "" and last:
            break
        fields = _split_csv(line)
        if len(fields) == 1 and lineno > 1 and last:
            mcs = _parse_int(fields[0], "saved MCS (line %d)" % lineno)
            have_mcs = True
            break
        if width == 0:
            width = len(fields)
        if len(fields) != width:
            raise FormatError("%s: ragged row at line %d" % (path, lineno))
        row = []
        for fld in fields:
            v = _parse_int(fld, "cell (line %d)" % lineno)
            if v < 0:
                raise FormatError("%s: negative cell at line %d" % (path, lineno))
            row.append(v)
        rows.append(row)
    if not have_mcs:
        raise FormatError("%s: missing saved-MCS trailer line (line %d)" % (path, len(lines)))
    if not rows or width < 2:
        raise FormatError("%s: grid must be at least 2x2" % path)
    if len(rows) < 2:
        raise FormatError("%s: grid must have at least 2 rows" % path)
    return Lattice(width, len(rows), np.array(rows, np.int32).ravel()), mcs


# ---- params -----------------------------------------------------------------------------------

def export_params(p: SimParams, path) -> None:
    with _open_out(path) as out:
        out.write("length,%d\nheight,%d\nmcs,%d\nneighbourhood,%d\nprintFrequency,%d\n" %
                  (p.length, p.height, p.mcs_limit, int(p.neighbourhood), p.print_frequency))
        out.write("mobility,%s\nspecies,%d\nflux,%s\nempty,%s\n" % (format_double(p.mobility), p.species,
                                                                   _bool_str(p.flux), format_double(p.empty_prob)))
        out.write("save,%s\ndominance,%s\nresume,%s\nnumRandoms,%d\nmaxStep,%s\n" %
                  (_bool_str(p.save), _bool_str(p.dominance_import), _bool_str(p.resume), p.num_randoms,
                   _bool_str(p.max_step)))
        if p.seed is not None:
            out.write("seed,%d\n" % p.seed)


def import_params(path) -> SimParams:
    with _open_in(path) as f:
        lines = _lines(f)
    kv = {}
    for i, line in enumerate(lines):
        if line == "":
            continue
        fields = _split_csv(line)
        if len(fields) != 2:
            raise FormatError("%s: expected key,value at line %d" % (path, i + 1))
        if fields[0] in kv:
            raise FormatError("%s: duplicate key '%s'" % (path, fields[0]))
        kv[fields[0]] = fields[1]
    for key in PARAM_KEYS:
        if key not in kv:
            raise FormatError("%s: missing required key '%s'" % (path, key))
    for key in sorted(kv):
        if key != "seed" and key not in PARAM_KEYS:
            raise FormatError("%s: unknown key '%s'" % (path, key))
    p = SimParams()
    p.length = _parse_int(kv["length"], "length")
    p.height = _parse_int(kv["height"], "height")
    p.mcs_limit = _parse_int(kv["mcs"], "mcs")
    nb = _parse_int(kv["neighbourhood"], "neighbourhood")
    if nb not in (4, 8):
        raise FormatError("%s: neighbourhood must be 4 or 8" % path)
    p.neighbourhood = Neighbourhood(nb)
    p.print_frequency = _parse_int(kv["printFrequency"], "printFrequency")
    p.mobility = _parse_double(kv["mobility"], "mobility")
    p.species = _parse_int(kv["species"], "species")
    p.flux = _parse_bool(kv["flux"], "flux")
    p.empty_prob = _parse_double(kv["empty"], "empty")
    p.save = _parse_bool(kv["save"], "save")
    p.dominance_import = _parse_bool(kv["dominance"], "dominance")
    p.resume = _parse_bool(kv["resume"], "resume")
    p.num_randoms = _parse_int(kv["numRandoms"], "numRandoms")
    p.max_step = _parse_bool(kv["maxStep"], "maxStep")
    if "seed" in kv:
        t = kv["seed"]
        if not t.isdigit() or int(t) >= 2 ** 64:
            raise FormatError("%s: invalid seed '%s'" % (path, t))
        p.seed = int(t)
    p.validate()
    return p


# ---- dominance --------------------------------------------------------------------------------

def export_dominance(model: DominanceModel, path) -> None:
    m = model.matrix()
    with _open_out(path) as out:
        for i in range(model.size):
            if model.kind == DominanceModel.Kind.Binary:
                out.write(",".join(str(int(v)) for v in m[i]) + "\n")
            else:
                out.write(",".join(format_double(float(v)) for v in m[i]) + "\n")


def import_dominance(path) -> DominanceModel:
    with _open_in(path) as f:
        lines = _lines(f)
    rows, rated = [], False
    for i, line in enumerate(lines):
        if line == "":
            continue
        row = []
        for fld in _split_csv(line):
            v = _parse_double(fld, "dominance entry (line %d)" % (i + 1))
            if v < 0.0 or v > 1.0:
                raise FormatError("%s: entry out of [0, 1] at line %d" % (path, i + 1))
            if v != 0.0 and v != 1.0:
                rated = True
            row.append(v)
        rows.append(row)
    if not rows:
        raise FormatError("%s: empty dominance matrix" % path)
    for r, row in enumerate(rows):
        if len(row) != len(rows):
            raise FormatError("%s: matrix is not square (row %d)" % (path, r + 1))
    m = DominanceModel(len(rows), DominanceModel.Kind.Rated if rated else DominanceModel.Kind.Binary,
                       np.array(rows, np.float64).ravel())
    m.validate()
    return m


# ---- densities / dir name ---------------------------------------------------------------------

def export_densities(trace: DensityTrace, path, append: bool = False) -> None:
    fresh = not append or not os.path.exists(path)
    with _open_out(path, append=not fresh) as out:
        if fresh and trace.counts:
            out.write("mcs" + "".join(",count_%d" % s for s in range(len(trace.counts[0]))) + "\n")
        for step, row in zip(trace.steps, trace.counts):
            out.write("%d%s\n" % (step, "".join(",%d" % int(c) for c in row)))


def output_dir_name(p: SimParams) -> str:
    return "L%d_H%d_n%d_m%s_flux%d_s%d" % (p.length, p.height, int(p.neighbourhood), format_double(p.mobility),
                                          1 if p.flux else 0, p.species)


# ---- checkpoints ------------------------------------------------------------------------------

@dataclass
class Checkpoint:
    params: SimParams
    lattice: Lattice
    dominance: DominanceModel
    saved_mcs: int = 0
    streams: List = field(default_factory=list)  # MT19937 states of the reference (unused on device)


def save_checkpoint(directory, params: SimParams, lattice: Lattice, model: DominanceModel, mcs: int) -> None:
    try:
        os.makedirs(directory, exist_ok=True)
    except OSError as e:
        raise IoError("cannot create directory %s: %s" % (directory, e))
    export_params(params, os.path.join(directory, "params.csv"))
    export_grid(lattice, mcs, os.path.join(directory, "grid.csv"))
    export_dominance(model, os.path.join(directory, "dominance.csv"))


def load_checkpoint(directory) -> Checkpoint:
    params = import_params(os.path.join(directory, "params.csv"))
    lattice, mcs = import_grid(os.path.join(directory, "grid.csv"))
    dom = import_dominance(os.path.join(directory, "dominance.csv"))
    cp = Checkpoint(params, lattice, dom, mcs)
    if lattice.length != params.length or lattice.height != params.height:
        raise FormatError("%s: grid dimensions do not match params" % directory)
    if dom.size != params.species:
        raise FormatError("%s: dominance size does not match species count" % directory)
    if np.any(np.asarray(lattice.cells) > params.species):
        raise FormatError("%s: grid cell exceeds species count" % directory)
    if mcs < 0 or mcs > params.mcs_limit:
        raise FormatError("%s: saved MCS outside [0, mcs limit]" % directory)
    return cp


def resume_state(cp: Checkpoint) -> RunState:
    """RunState to pass as simulate(..., resume_from=...) (engine.cpp:219-221)."""
    return RunState(lattice=cp.lattice, current_mcs=cp.saved_mcs, model=cp.dominance)
