"""paper_2508_16639_b200 — B200-native ESCG Monte Carlo engine (drop-in for the reference's step path).

The compute path is libescg_b200.so (sm_100a CUDA kernels behind the C ABI in include/escg_dev.h);
this package is the host-side mirror of the reference's C++ API (escg::simulate and friends).
"""
from .engine import (PAPER_SPECIES, ActionRates, DensityTrace, DeviceEngine, DominanceModel, EngineMode, Lattice,
                     Neighbourhood, RunHooks, RunState, RunStatus, SimParams, SimulationResult, action_rates,
                     align_num_randoms, densities, is_save_mcs, make_circulant, make_park8, make_rpsls, make_rpsls_ablated,
                     simulate, stasis, thresholds)
from .errors import ConfigError, EngineError, FormatError, IoError

__all__ = [
    "PAPER_SPECIES", "ActionRates", "DensityTrace", "DeviceEngine", "DominanceModel", "EngineMode", "Lattice",
    "Neighbourhood", "RunHooks", "RunState", "RunStatus", "SimParams", "SimulationResult", "action_rates",
    "align_num_randoms", "densities", "is_save_mcs", "make_circulant", "make_park8", "make_rpsls", "make_rpsls_ablated",
    "simulate", "stasis", "thresholds", "ConfigError", "EngineError", "FormatError", "IoError",
]
