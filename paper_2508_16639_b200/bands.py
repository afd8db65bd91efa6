"""Row-band sharding of one lattice over several GPUs.

Band g owns rows [start_g, start_g + rows_g) (multiples of 4) of the global lattice and keeps
12*kmcs halo rows on each side.  Every chunk of kmcs MCS each band pulls its halos from its ring
neighbours (peer copies over NVLink when the bands sit on different GPUs) and runs the block kernel
on its rows.  The draws are a function of the global (seed, MCS, phase, tile), so the banded run is
bit-identical to the single-lattice run for any number of bands (tests/test_gpu_parity.py).

`BandGroup` drives all bands from one process (one GPU or several with peer access).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from ._lib import check, lib
from .engine import DominanceModel, SimParams
from .errors import ConfigError, EngineError


def band_rows(height: int, n_bands: int):
    """Row split of the band engines (engine.cpp create_impl): [(start, rows)] at multiples of 4."""
    u = height // 4
    return [(u * g // n_bands * 4, (u * (g + 1) // n_bands - u * g // n_bands) * 4) for g in range(n_bands)]


class BandGroup:
    def __init__(self, params: SimParams, model: DominanceModel, n_bands: int, devices: Optional[Sequence[int]] = None,
                 kmcs: int = 2):
        if params.seed is None:
            raise ConfigError("a band group needs an explicit seed (every band must share it)")
        self.params, self.model, self.n = params, model, int(n_bands)
        devices = list(devices) if devices is not None else [0] * self.n
        if len(devices) != self.n:
            raise ConfigError("one device per band")
        self._h = []
        try:
            for g in range(self.n):
                h = C.c_void_p()
                check(lib().escg_dev_create_band(C.byref(params.to_c()), np.ascontiguousarray(model.entries, np.float64),
                                                 int(model.size), int(model.kind), int(devices[g]), self.n, g,
                                                 int(kmcs), C.byref(h)))
                self._h.append(h)
        except Exception:
            self.close()
            raise
        self.info = [self._band_info(h) for h in self._h]

    @staticmethod
    def _band_info(h):
        v = [C.c_int32(0) for _ in range(4)]
        check(lib().escg_dev_band_info(h, *[C.byref(x) for x in v]))
        return dict(start=v[0].value, rows=v[1].value, halo=v[2].value, kmcs=v[3].value)

    def close(self):
        for h in self._h:
            if h:
                lib().escg_dev_destroy(h)
        self._h = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_lattice(self):
        for h in self._h:
            check(lib().escg_dev_init_lattice(h))

    def set_lattice(self, cells, mcs: int = 0):
        cells = np.ascontiguousarray(np.asarray(cells).ravel(), np.int32)
        L = self.params.length
        for h, inf in zip(self._h, self.info):
            part = np.ascontiguousarray(cells[inf["start"] * L:(inf["start"] + inf["rows"]) * L])
            check(lib().escg_dev_set_lattice(h, 0, part, int(mcs)))

    def get_lattice(self) -> np.ndarray:
        L = self.params.length
        out = np.zeros(self.params.cells(), np.int32)
        for h, inf in zip(self._h, self.info):
            part = np.zeros(inf["rows"] * L, np.int32)
            m = C.c_int64(0)
            check(lib().escg_dev_get_lattice(h, 0, part.ctypes.data_as(C.c_void_p), C.byref(m)))
            out[inf["start"] * L:(inf["start"] + inf["rows"]) * L] = part
        return out

    def counts(self) -> np.ndarray:
        tot = np.zeros(self.model.size + 1, np.uint64)
        for h in self._h:
            c = np.zeros(self.model.size + 1, np.uint64)
            check(lib().escg_dev_counts(h, 0, c))
            tot += c
        return tot

    def advance(self, n_mcs: int):
        arr = (C.c_void_p * self.n)(*[h.value for h in self._h])
        check(lib().escg_group_advance(arr, self.n, int(n_mcs)))


# ---- one process per GPU ---------------------------------------------------------------------

def exchange_halos(recv_top, send_top, send_bot, recv_bot, rank: int, world: int, group=None) -> None:
    """Ring halo exchange of a band group over torch.distributed point-to-point (NCCL on GPUs, gloo
    on CPU tensors).  Band g's top halo receives the last `halo` rows of band g-1 and its bottom
    halo the first `halo` rows of band g+1 (periodic ring).  Two shifts, each one send + one recv per
    rank, so the pairing is unambiguous for any world size >= 2 (world 2: both neighbours are the
    same rank)."""
    import torch.distributed as dist

    up, down = (rank - 1) % world, (rank + 1) % world
    for sends, recvs in (((send_bot, down), (recv_top, up)), ((send_top, up), (recv_bot, down))):
        ops = [dist.P2POp(dist.isend, sends[0], sends[1], group), dist.P2POp(dist.irecv, recvs[0], recvs[1], group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class _DevView:
    """Zero-copy view of engine-owned device bytes for torch (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3}


class DistributedBand:
    """This rank's band of one lattice sharded by rows over ranks, one process per GPU.

    Each chunk of kmcs MCS: halo rows move between ring neighbours with NCCL send/recv straight
    from/to the engine's device buffers (exchange_halos), then the block kernel runs on the band
    (escg_dev_band_step).  Draws depend only on global coordinates, so the sharded run equals the
    single-lattice run bit for bit.  The engine issues its work on torch's current stream of the
    device (escg_dev_set_stream), so exchange and step are ordered on the device with no host
    synchronisation per chunk (the NCCL requests make that stream wait on their own)."""

    def __init__(self, params: SimParams, model: DominanceModel, rank: int, world: int, device: int = 0, kmcs: int = 2,
                 group=None):
        if params.seed is None:
            raise ConfigError("a band group needs an explicit seed (every band must share it)")
        if world < 2:
            raise ConfigError("a distributed band group needs at least 2 ranks")
        self.params, self.model, self.rank, self.world, self.device, self.group = params, model, rank, world, device, group
        h = C.c_void_p()
        check(lib().escg_dev_create_band(C.byref(params.to_c()), np.ascontiguousarray(model.entries, np.float64),
                                         int(model.size), int(model.kind), int(device), int(world), int(rank),
                                         int(kmcs), C.byref(h)))
        self._h = h
        self.info = BandGroup._band_info(h)
        self._stream = None
        try:
            import torch

            if torch.cuda.is_available():
                self._stream = torch.cuda.current_stream(device)
                check(lib().escg_dev_set_stream(h, C.c_void_p(self._stream.cuda_stream)))
        except ImportError:
            pass
        if self.info["kmcs"] != kmcs:
            raise EngineError("band engine runs %d MCS per chunk, %d requested" % (self.info["kmcs"], kmcs))
        self._check_uniform_chunk()

    def _check_uniform_chunk(self):
        """Every rank must post the same number of halo exchanges per advance: the chunk (kmcs) and
        halo depth have to agree over the group, else ranks pair stale halos and hang."""
        import torch
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized():
            return
        backend = dist.get_backend(self.group)
        dev = torch.device("cuda", self.device) if backend == "nccl" else torch.device("cpu")
        mine = torch.tensor([self.info["kmcs"], self.info["halo"]], dtype=torch.int64, device=dev)
        lo, hi = mine.clone(), mine.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=self.group)
        if not torch.equal(lo, hi):
            raise EngineError("band chunk/halo differ across ranks: min %s max %s" % (lo.tolist(), hi.tolist()))

    def close(self):
        if self._h:
            lib().escg_dev_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def init_lattice(self):
        check(lib().escg_dev_init_lattice(self._h))

    def set_band(self, band_cells, mcs: int = 0):
        """This band's rows (band_rows x L int32) at MCS `mcs`."""
        part = np.ascontiguousarray(np.asarray(band_cells).ravel(), np.int32)
        check(lib().escg_dev_set_lattice(self._h, 0, part, int(mcs)))

    def get_band(self) -> np.ndarray:
        part = np.zeros(self.info["rows"] * self.params.length, np.int32)
        m = C.c_int64(0)
        check(lib().escg_dev_get_lattice(self._h, 0, part.ctypes.data_as(C.c_void_p), C.byref(m)))
        return part

    def counts(self) -> np.ndarray:
        c = np.zeros(self.model.size + 1, np.uint64)
        check(lib().escg_dev_counts(self._h, 0, c))
        return c

    def halo_views(self):
        """(recv_top, send_top, send_bot, recv_bot) as uint8 CUDA tensors over the current buffer."""
        import torch

        p = [C.c_void_p() for _ in range(4)]
        nbytes = C.c_int64(0)
        check(lib().escg_dev_band_rows(self._h, *[C.byref(x) for x in p], C.byref(nbytes)))
        dev = torch.device("cuda", self.device)
        return tuple(torch.as_tensor(_DevView(x.value, nbytes.value), device=dev) for x in p)

    def advance(self, n_mcs: int):
        """Enqueue n_mcs MCS (chunks of kmcs: halo exchange, band step) on the band's stream; returns
        without waiting for the device (synchronize the stream, or read the band, to wait)."""
        import torch

        k = self.info["kmcs"]
        done = 0
        with torch.cuda.stream(self._stream) if self._stream is not None else _nullctx():
            while done < n_mcs:
                chunk = min(k, n_mcs - done)
                exchange_halos(*self.halo_views(), self.rank, self.world, self.group)
                check(lib().escg_dev_band_step(self._h, int(chunk)))
                done += chunk


# ---- multi-part ring: the ring kernel across GPUs -------------------------------------------

def ring_neighbours(part: int, n_parts: int):
    """(part above, part below) of a periodic ring of parts."""
    return (part - 1) % n_parts, (part + 1) % n_parts


def _part_export(h, ipc: bool):
    """(planes0, planes1, inbox, rows, ipc handle bytes or None, inbox byte offset) of a ring part."""
    p0, p1, ib = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rows, off = C.c_int32(0), C.c_int64(0)
    buf = (C.c_ubyte * 192)() if ipc else None
    check(lib().escg_dev_ring_part_export(h, C.byref(p0), C.byref(p1), C.byref(ib), C.byref(rows),
                                          C.cast(buf, C.c_void_p) if ipc else None, C.byref(off)))
    return p0.value, p1.value, ib.value, rows.value, (bytes(buf) if ipc else None), off.value


class RingGroup:
    """One lattice as a multi-part ring driven from one process (escg_ring_group_advance).

    Parts on one device run as ONE cooperative launch over all parts — the single-GPU form of the
    multi-GPU ring: the same kernel, with every cross-part row going through the inbox and plane
    pointers a part on another GPU would use.  Parts on several devices run one launch each with
    peer access.  Draws use global coordinates, so any split equals the single-lattice run bit for
    bit (tests/test_gpu_ring.py)."""

    def __init__(self, params: SimParams, model: DominanceModel, n_parts: int, devices: Optional[Sequence[int]] = None,
                 ctas: int = 0):
        if params.seed is None:
            raise ConfigError("a ring group needs an explicit seed (every part must share it)")
        self.params, self.model, self.n = params, model, int(n_parts)
        devices = list(devices) if devices is not None else [0] * self.n
        if len(devices) != self.n:
            raise ConfigError("one device per part")
        if ctas == 0 and len(set(devices)) == 1:
            # one launch over every part: the parts share the device's SMs
            try:
                import torch

                sms = torch.cuda.get_device_properties(devices[0]).multi_processor_count
            except Exception:
                sms = 148
            ctas = max(1, sms // self.n)
        self._h = []
        try:
            for g in range(self.n):
                h = C.c_void_p()
                check(lib().escg_dev_create_ring_part(C.byref(params.to_c()),
                                                      np.ascontiguousarray(model.entries, np.float64),
                                                      int(model.size), int(model.kind), int(devices[g]), self.n, g,
                                                      int(ctas), C.byref(h)))
                self._h.append(h)
            ex = [_part_export(h, False) for h in self._h]
            for g, h in enumerate(self._h):
                up, dn = ring_neighbours(g, self.n)
                check(lib().escg_dev_ring_part_connect(h, ex[up][0], ex[up][1], ex[up][2], ex[up][3], ex[dn][0],
                                                       ex[dn][1], ex[dn][2], ex[dn][3]))
        except Exception:
            self.close()
            raise
        self.info = [BandGroup._band_info(h) for h in self._h]

    close = BandGroup.close
    __enter__ = BandGroup.__enter__
    __exit__ = BandGroup.__exit__
    __del__ = BandGroup.__del__
    init_lattice = BandGroup.init_lattice
    set_lattice = BandGroup.set_lattice
    get_lattice = BandGroup.get_lattice
    counts = BandGroup.counts

    def describe(self, part: int = 0):
        v = [C.c_int32(0) for _ in range(4)]
        check(lib().escg_dev_describe(self._h[part], *[C.byref(x) for x in v]))
        fmt = C.c_int32(0)
        check(lib().escg_dev_draw_format(self._h[part], C.byref(fmt)))
        return dict(kernel={1: "tile", 2: "block", 3: "ring"}[v[0].value], ctas=v[1].value, threads=v[2].value,
                    smem_bytes=v[3].value, draw_code=fmt.value)

    def advance(self, n_mcs: int):
        arr = (C.c_void_p * self.n)(*[h.value for h in self._h])
        check(lib().escg_ring_group_advance(arr, self.n, int(n_mcs)))

    def last_ms(self) -> float:
        ms, n = C.c_double(0), C.c_int64(0)
        check(lib().escg_dev_last_timing(self._h[0], C.byref(ms), C.byref(n)))
        return ms.value


def exchange_part_info(mine, rank: int, world: int, group=None):
    """All-gather every rank's ring-part export (IPC handles, inbox offset, rows) and return the
    entries of this rank's part above and below."""
    import torch.distributed as dist

    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    up, dn = ring_neighbours(rank, world)
    return allv[up], allv[dn]


class DistributedRing:
    """This rank's part of one lattice as a multi-part ring, one process per GPU.

    The parts' ring kernels exchange boundary rows with each other inside the kernel, every colour
    phase, through tagged system-scope stores into the neighbour part's inbox (CUDA IPC mappings of
    the neighbours' allocations over NVLink): advance() enqueues one launch and returns; nothing on
    the host takes part in the exchange.  Reads and writes of the lattice synchronise every rank."""

    def __init__(self, params: SimParams, model: DominanceModel, rank: int, world: int, device: int = 0, ctas: int = 0,
                 group=None):
        import torch
        import torch.distributed as dist

        if params.seed is None:
            raise ConfigError("a ring needs an explicit seed (every part must share it)")
        if world < 2:
            raise ConfigError("a distributed ring needs at least 2 ranks")
        self.params, self.model, self.rank, self.world, self.device, self.group = params, model, rank, world, device, group
        self._opened = []
        h = C.c_void_p()
        check(lib().escg_dev_create_ring_part(C.byref(params.to_c()), np.ascontiguousarray(model.entries, np.float64),
                                              int(model.size), int(model.kind), int(device), int(world), int(rank),
                                              int(ctas), C.byref(h)))
        self._h = h
        try:
            _, _, _, rows, ipc, off = _part_export(h, True)
            up, dn = exchange_part_info((ipc, off, rows), rank, world, group)
            cache = {}

            def open_part(entry):
                key = entry[0]
                if key not in cache:
                    ptrs = []
                    for k in range(3):
                        p = C.c_void_p()
                        check(lib().escg_ipc_open(int(device), entry[0][64 * k:64 * (k + 1)], C.byref(p)))
                        self._opened.append(p.value)
                        ptrs.append(p.value)
                    cache[key] = (ptrs[0], ptrs[1], ptrs[2] + entry[1], entry[2])
                return cache[key]

            u, d = open_part(up), open_part(dn)
            check(lib().escg_dev_ring_part_connect(h, u[0], u[1], u[2], u[3], d[0], d[1], d[2], d[3]))
        except Exception:
            self.close()
            raise
        self.info = BandGroup._band_info(h)
        self._torch, self._dist = torch, dist
        # the part's launches go on torch's current stream: CUDA events there bracket them
        self._stream = torch.cuda.current_stream(device)
        check(lib().escg_dev_set_stream(h, C.c_void_p(self._stream.cuda_stream)))

    def close(self):
        for p in self._opened:
            lib().escg_ipc_close(int(self.device), p)
        self._opened = []
        if getattr(self, "_h", None):
            try:  # every rank unmapped this part's buffers before they are freed
                import torch.distributed as dist

                if dist.is_available() and dist.is_initialized():
                    dist.barrier(group=self.group)
            except Exception:
                pass
            lib().escg_dev_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _quiesce(self):
        """Every rank's launches done: the neighbours' last rows are in this part's planes."""
        self._torch.cuda.synchronize(self.device)
        self._dist.barrier(group=self.group)

    def init_lattice(self):
        self._quiesce()
        check(lib().escg_dev_init_lattice(self._h))
        self._dist.barrier(group=self.group)

    def set_band(self, band_cells, mcs: int = 0):
        """This part's rows (rows x L int32) at MCS `mcs` (every rank, before the next advance)."""
        self._quiesce()
        part = np.ascontiguousarray(np.asarray(band_cells).ravel(), np.int32)
        check(lib().escg_dev_set_lattice(self._h, 0, part, int(mcs)))
        self._dist.barrier(group=self.group)

    def get_band(self) -> np.ndarray:
        self._quiesce()
        part = np.zeros(self.info["rows"] * self.params.length, np.int32)
        m = C.c_int64(0)
        check(lib().escg_dev_get_lattice(self._h, 0, part.ctypes.data_as(C.c_void_p), C.byref(m)))
        return part

    def counts(self) -> np.ndarray:
        self._quiesce()
        c = np.zeros(self.model.size + 1, np.uint64)
        check(lib().escg_dev_counts(self._h, 0, c))
        return c

    def advance(self, n_mcs: int):
        """Enqueue n_mcs MCS as one ring launch on this rank's GPU; returns without waiting."""
        check(lib().escg_dev_advance(self._h, int(n_mcs)))
