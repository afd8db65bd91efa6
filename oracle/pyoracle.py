"""ctypes bindings for the test oracles.

*** TEST INFRASTRUCTURE ONLY *** — imported by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs, never by the product package.

* ``Oracle``    — oracle/liboracle.so, the C restatement (escg_oracle.c).
* ``Reference`` — oracle/_ref/libescg_ref.so, the unmodified reference engine + ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libescg_ref.so")

_p = np.ctypeslib.ndpointer
_i32 = _p(dtype=np.int32, flags="C_CONTIGUOUS")
_u32 = _p(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64 = _p(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64 = _p(dtype=np.int64, flags="C_CONTIGUOUS")
_f64 = _p(dtype=np.float64, flags="C_CONTIGUOUS")

STATUS = {0: "Completed", 1: "Stasis", 2: "Stopped"}


def build():
    """Build oracle/liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class Oracle:
    """C restatement of the reference hot path."""

    def __init__(self):
        L = self.lib = _load(ORACLE_SO)
        L.orc_murmur_finalize.restype = C.c_uint32
        L.orc_murmur_finalize.argtypes = [C.c_uint32]
        L.orc_seed_mix.restype = C.c_uint32
        L.orc_seed_mix.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_sizeof_mt.restype = C.c_int64
        L.orc_mt_seed.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_mt_extract.restype = C.c_uint32
        L.orc_mt_extract.argtypes = [C.c_void_p]
        L.orc_stream_init.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64]
        L.orc_unit.restype = C.c_float
        L.orc_unit.argtypes = [C.c_uint32]
        L.orc_align_num_randoms.restype = C.c_int64
        L.orc_align_num_randoms.argtypes = [C.c_int64, C.c_int64]
        L.orc_action_rates.argtypes = [C.c_double, C.c_int64, _f64]
        L.orc_neighbor_index.restype = C.c_int64
        L.orc_neighbor_index.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_elementary_step.restype = C.c_int
        L.orc_elementary_step.argtypes = [_i32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64, C.c_double,
                                          C.c_int64, C.c_int, C.c_float]
        L.orc_bucket.restype = C.c_int
        L.orc_bucket.argtypes = [C.c_uint32, C.c_double, C.c_int64]
        L.orc_interaction.restype = C.c_int
        L.orc_interaction.argtypes = [C.c_uint32, C.c_double, C.c_int64, _f64, C.c_int, C.c_int, C.c_int]
        L.orc_check_bucket_thresholds.restype = C.c_int64
        L.orc_check_bucket_thresholds.argtypes = [_u32, C.c_double, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_densities.restype = C.c_int
        L.orc_densities.argtypes = [_i32, C.c_int64, C.c_int, _u64]
        L.orc_is_save_mcs.restype = C.c_int
        L.orc_is_save_mcs.argtypes = [C.c_int64, C.c_int64]
        L.orc_run_serial.restype = C.c_int
        L.orc_run_serial.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64, C.c_double, C.c_double,
                                     C.c_int64, C.c_uint64, C.c_void_p, C.c_int, _i32, _i64, _u64, C.c_int64,
                                     C.POINTER(C.c_int64)]
        L.orc_serial_draws.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _i32, C.c_int64, _u32,
                                       _u32, _u32]
        L.orc_apply_draws.restype = C.c_int
        L.orc_apply_draws.argtypes = [_i32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64, C.c_double, _u32,
                                      _u32, _u32, C.c_int64]
        L.orc_philox.argtypes = [_u32, _u32, _u32]
        L.orc_crs_round.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    _p(dtype=np.intc, flags="C_CONTIGUOUS")]
        L.orc_crs_round_g.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), _p(dtype=np.intc, flags="C_CONTIGUOUS")]
        L.orc_crs_init.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _i32]
        L.orc_crs_run.restype = C.c_int
        L.orc_crs_run.argtypes = [_i32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64, C.c_double, C.c_uint64,
                                  C.c_int64, C.c_int64, C.c_int]
        L.orc_seed32.restype = C.c_uint32
        L.orc_seed32.argtypes = [C.c_uint64]
        L.orc_slice3_table.argtypes = [C.c_int, _u32]
        L.orc_slice3_mask.restype = C.c_uint32
        L.orc_slice3_mask.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, C.c_int]

    # --- RNG -----------------------------------------------------------------------------
    def mt_words(self, seed32, n):
        st = C.create_string_buffer(int(self.lib.orc_sizeof_mt()))
        self.lib.orc_mt_seed(st, seed32)
        return np.array([self.lib.orc_mt_extract(st) for _ in range(n)], dtype=np.uint32)

    def stream_words(self, seed, k, n, burn_in=50000):
        st = C.create_string_buffer(int(self.lib.orc_sizeof_mt()))
        self.lib.orc_stream_init(st, seed, k, burn_in)
        return np.array([self.lib.orc_mt_extract(st) for _ in range(n)], dtype=np.uint32)

    def philox(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.orc_philox(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    # --- model ---------------------------------------------------------------------------
    def action_rates(self, mobility, cells):
        out = np.zeros(4)
        self.lib.orc_action_rates(mobility, cells, out)
        return out

    def neighbor_index(self, i, d, arity, length, height, flux):
        return int(self.lib.orc_neighbor_index(i, d, arity, length, height, int(flux)))

    def densities(self, cells, species):
        counts = np.zeros(species + 1, np.uint64)
        rc = self.lib.orc_densities(np.ascontiguousarray(cells, np.int32), cells.size, species, counts)
        if rc:
            raise RuntimeError("corrupt lattice value")
        return counts

    # --- engines -------------------------------------------------------------------------
    def run_serial(self, length, height, dom, mobility, empty_prob, mcs_limit, seed, arity=4, flux=True,
                   init=None, tracked=0, cap=None):
        species = int(round(np.sqrt(np.asarray(dom).size)))
        dom = np.ascontiguousarray(dom, np.float64).ravel()
        cap = cap or (mcs_limit + 2)
        cells = np.zeros(length * height, np.int32)
        steps = np.zeros(cap, np.int64)
        counts = np.zeros(cap * (species + 1), np.uint64)
        n_rec = C.c_int64(0)
        init_p = None
        if init is not None:
            init = np.ascontiguousarray(init, np.int32)
            init_p = init.ctypes.data
        st = self.lib.orc_run_serial(length, height, species, arity, int(flux), dom, mobility, empty_prob, mcs_limit,
                                     seed, init_p, tracked, cells, steps, counts, cap, C.byref(n_rec))
        if st < 0:
            raise RuntimeError("oracle engine error %d" % st)
        n = min(n_rec.value, cap)
        return dict(status=STATUS[st], cells=cells, steps=steps[:n], counts=counts[: n * (species + 1)].reshape(n, species + 1))

    def serial_draws(self, length, height, species, empty_prob, seed, n_attempts):
        init = np.zeros(length * height, np.int32)
        wc, wd, wa = (np.zeros(n_attempts, np.uint32) for _ in range(3))
        self.lib.orc_serial_draws(length, height, species, empty_prob, seed, init, n_attempts, wc, wd, wa)
        return init, wc, wd, wa

    def apply_draws(self, cells, length, height, dom, mobility, wc, wd, wa, arity=4, flux=True):
        species = int(round(np.sqrt(np.asarray(dom).size)))
        cells = np.ascontiguousarray(cells, np.int32).copy()
        rc = self.lib.orc_apply_draws(cells, length, height, species, arity, int(flux),
                                      np.ascontiguousarray(dom, np.float64).ravel(), mobility, wc, wd, wa, wc.size)
        if rc:
            raise RuntimeError("oracle engine error %d" % rc)
        return cells

    def crs_round(self, seed, mcs):
        oy, ox = C.c_int(0), C.c_int(0)
        perm = np.zeros(4, np.intc)
        self.lib.orc_crs_round(seed, mcs, C.byref(oy), C.byref(ox), perm)
        return oy.value, ox.value, perm.tolist()

    def crs_round_g(self, seed, mcs, ncy, ncx):
        oy, ox = C.c_int(0), C.c_int(0)
        perm = np.zeros(9, np.intc)
        self.lib.orc_crs_round_g(seed, mcs, ncy, ncx, C.byref(oy), C.byref(ox), perm)
        return oy.value, ox.value, perm[:ncy * ncx].tolist()

    def slice3_table(self, K):
        """SLICED3 tables (escg_oracle.c orc_slice3_table): T[1..32], S[0..31], then C[m][g]."""
        out = np.zeros(64 + 31 * 32, np.uint32)
        self.lib.orc_slice3_table(K, out)
        return out

    def slice3_mask(self, seed, item, mcs, phase, attempt, K):
        return int(self.lib.orc_slice3_mask(seed, item, mcs, phase, attempt, K))

    def crs_init(self, length, height, species, empty_prob, seed):
        cells = np.zeros(length * height, np.int32)
        self.lib.orc_crs_init(length, height, species, empty_prob, seed, cells)
        return cells

    def crs_run(self, cells, length, height, dom, mobility, seed, mcs0, n_mcs, arity=4, flux=True, narrow=False):
        """`narrow`: draw format — False/True (WIDE/NARROW) or the engine's draw code
        (DeviceEngine.draw_code(): 0 WIDE, 1 NARROW, 2 | K << 8 SLICED, 3 | K << 8 SLICED3)."""
        species = int(round(np.sqrt(np.asarray(dom).size)))
        cells = np.ascontiguousarray(cells, np.int32).copy()
        rc = self.lib.orc_crs_run(cells, length, height, species, arity, int(flux),
                                  np.ascontiguousarray(dom, np.float64).ravel(), mobility, seed, mcs0, n_mcs,
                                  narrow if isinstance(narrow, int) and not isinstance(narrow, bool) else int(bool(narrow)))
        if rc:
            raise RuntimeError("oracle crs error %d" % rc)
        return cells


class Reference:
    """The unmodified reference engine (oracle/_ref/libescg_ref.so)."""

    available = os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        L = self.lib = C.CDLL(REF_SO)
        L.ref_stream_words.restype = C.c_int
        L.ref_stream_words.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int64, _u32]
        L.ref_mt_raw.argtypes = [C.c_uint32, C.c_int64, _u32]
        L.ref_seed_mix.restype = C.c_uint32
        L.ref_seed_mix.argtypes = [C.c_uint32, C.c_uint32]
        L.ref_align_num_randoms.restype = C.c_int64
        L.ref_align_num_randoms.argtypes = [C.c_int64, C.c_int64]
        L.ref_action_rates.argtypes = [C.c_double, C.c_int64, _f64]
        L.ref_neighbor_index.restype = C.c_int64
        L.ref_neighbor_index.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_init_lattice.restype = C.c_int
        L.ref_init_lattice.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _i32]
        L.ref_elementary_step.restype = C.c_int
        L.ref_elementary_step.argtypes = [_i32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64, C.c_int,
                                          C.c_double, C.c_int64, C.c_int, C.c_float]
        L.ref_simulate.restype = C.c_int
        L.ref_simulate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64, C.c_int,
                                   C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_make_circulant.restype = C.c_int
        L.ref_make_circulant.argtypes = [C.c_int, _p(dtype=np.intc, flags="C_CONTIGUOUS"), C.c_int, _f64]
        L.ref_make_rpsls_ablated.argtypes = [_f64]
        L.ref_make_park8.restype = C.c_int
        L.ref_make_park8.argtypes = [C.c_double, C.c_double, C.c_double, _f64]
        L.ref_validate_dominance.restype = C.c_int
        L.ref_validate_dominance.argtypes = [_f64, C.c_int, C.c_int]
        L.ref_ks_two_sample_pvalue.restype = C.c_double
        L.ref_ks_two_sample_pvalue.argtypes = [_f64, C.c_int64, _f64, C.c_int64]
        L.ref_chi_square_uniform_pvalue.restype = C.c_double
        L.ref_chi_square_uniform_pvalue.argtypes = [_u64, C.c_int64]

    def circulant(self, species, offsets):
        out = np.zeros(species * species)
        rc = self.lib.ref_make_circulant(species, np.asarray(offsets, np.intc), len(offsets), out)
        if rc:
            raise ValueError("ConfigError")
        return out.reshape(species, species)

    def rpsls_ablated(self):
        out = np.zeros(25)
        self.lib.ref_make_rpsls_ablated(out)
        return out.reshape(5, 5)

    def park8(self, alpha, beta=0.75, gamma=1.0):
        out = np.zeros(64)
        if self.lib.ref_make_park8(alpha, beta, gamma, out):
            raise ValueError("ConfigError")
        return out.reshape(8, 8)

    def stream_words(self, seed, n, count=1, k=0):
        out = np.zeros(n, np.uint32)
        self.lib.ref_stream_words(seed, count, k, n, out)
        return out

    def mt_raw(self, seed, n):
        out = np.zeros(n, np.uint32)
        self.lib.ref_mt_raw(seed, n, out)
        return out

    def init_lattice(self, length, height, species, empty_prob, seed):
        out = np.zeros(length * height, np.int32)
        rc = self.lib.ref_init_lattice(length, height, species, empty_prob, seed, out)
        if rc:
            raise RuntimeError("reference error %d" % rc)
        return out

    def simulate(self, length, height, dom, mobility, empty_prob, mcs_limit, seed, mode=0, workers=1, arity=4,
                 flux=True, rated=None, tracked=0, init=None, num_randoms=100000000, cap=None, want_cells=True):
        dom = np.ascontiguousarray(dom, np.float64)
        species = dom.shape[0]
        if rated is None:
            rated = int(np.any((dom != 0) & (dom != 1)))
        cap = cap if cap is not None else mcs_limit + 2
        cells = np.zeros(length * height, np.int32) if want_cells else None
        steps = np.zeros(max(cap, 1), np.int64)
        counts = np.zeros(max(cap, 1) * (species + 1), np.uint64)
        n_rec, status, elapsed = C.c_int64(0), C.c_int(0), C.c_double(0)
        init_p = None
        if init is not None:
            init = np.ascontiguousarray(init, np.int32)
            init_p = init.ctypes.data
        rc = self.lib.ref_simulate(mode, workers, length, height, species, arity, int(flux), dom.ravel(), rated,
                                   mobility, empty_prob, mcs_limit, num_randoms, seed, tracked, init_p,
                                   cells.ctypes.data if cells is not None else None, steps.ctypes.data,
                                   counts.ctypes.data, cap, C.byref(n_rec), C.byref(status), C.byref(elapsed))
        if rc:
            raise RuntimeError("reference error code %d" % rc)
        n = min(n_rec.value, cap)
        return dict(status=STATUS[status.value], cells=cells, steps=steps[:n],
                    counts=counts[: n * (species + 1)].reshape(n, species + 1), n_records=n_rec.value,
                    elapsed_s=elapsed.value)

    def ks(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return float(self.lib.ref_ks_two_sample_pvalue(a, a.size, b, b.size))

    def chi_square_uniform(self, bins):
        """stats.cpp chi_square_uniform_pvalue (the reference's own uniformity test)."""
        b = np.ascontiguousarray(bins, np.uint64)
        return float(self.lib.ref_chi_square_uniform_pvalue(b, b.size))
