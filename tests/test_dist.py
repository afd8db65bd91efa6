"""CPU, world_size 2 over gloo: the multi-GPU host logic (replica partition, gather, max-over-ranks)
used by bench.py and the sharded ensembles.  The device runner is replaced by the oracle's
coloured-schedule restatement, so results must be identical for world_size 1 and 2."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_runner(seeds):
    """Stand-in for device_replica_runner: L=24 RPS, 15 MCS of the CRS schedule per seed."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Oracle

    o = Oracle()
    D = np.array([[0, 1, 0], [0, 0, 1], [1, 0, 0]], float)
    out = []
    for s in seeds:
        init = o.crs_init(24, 24, 3, 0.1, int(s))
        fin = o.crs_run(init, 24, 24, D, 1e-3, int(s), 0, 15)
        out.append((15, 0, np.bincount(fin, minlength=4).tolist()))
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_16639_b200 import dist as edist

    res = edist.run_sharded(list(range(100, 111)), oracle_runner)
    m = edist.max_over_ranks(float(rank + 1) * 1.5)
    if rank == 0:
        q.put((res, m))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_covers_all():
    from paper_2508_16639_b200.dist import partition

    for total in (0, 1, 7, 11, 1024):
        for world in (1, 2, 3, 8):
            spans = [partition(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


@pytest.mark.timeout(300)
def test_sharded_ensemble_world2_equals_world1():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res2, m = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res1 = oracle_runner(list(range(100, 111)))
    assert [tuple(map(lambda x: tuple(x) if isinstance(x, list) else x, r)) for r in res2] == \
        [tuple(map(lambda x: tuple(x) if isinstance(x, list) else x, r)) for r in res1]
    assert m == 3.0


def _halo_worker(rank, world, port, q, H, L, halo):
    """Each rank holds halo + band + halo rows of a global lattice (as a band engine's buffer does);
    after exchange_halos its halos must equal the global rows above/below the band (periodic)."""
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_16639_b200.bands import band_rows, exchange_halos

    G = np.arange(H * L, dtype=np.int64).reshape(H, L) % 251
    start, rows = band_rows(H, world)[rank]
    buf = torch.full(((rows + 2 * halo) * L,), 255, dtype=torch.uint8)
    buf[halo * L:(halo + rows) * L] = torch.from_numpy(G[start:start + rows].astype(np.uint8).ravel())
    v = buf.view(rows + 2 * halo, L)
    recv_top, send_top = v[:halo].reshape(-1), v[halo:2 * halo].reshape(-1)
    send_bot, recv_bot = v[rows:rows + halo].reshape(-1), v[rows + halo:].reshape(-1)
    exchange_halos(recv_top, send_top, send_bot, recv_bot, rank, world)
    want_top = G[[(start - halo + i) % H for i in range(halo)]].astype(np.uint8)
    want_bot = G[[(start + rows + i) % H for i in range(halo)]].astype(np.uint8)
    ok = np.array_equal(v[:halo].numpy(), want_top) and np.array_equal(v[rows + halo:].numpy(), want_bot)
    ok = ok and np.array_equal(v[halo:halo + rows].numpy(), G[start:start + rows].astype(np.uint8))
    q.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_halo_exchange_gloo(world):
    """The multi-process band group's halo exchange (bands.exchange_halos, the NCCL path's host
    logic) moves exactly the neighbours' edge rows, for world 2 (both neighbours the same rank) and 3."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    H, L, halo = 48, 20, 12
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q, H, L, halo)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert got == {r: True for r in range(world)}


def _ring_worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_16639_b200.bands import band_rows, exchange_part_info

    # what DistributedRing exchanges: (IPC handles, inbox offset, rows) of every rank's part
    start, rows = band_rows(4096, world)[rank]
    mine = (bytes([rank]) * 192, 1000 + rank, rows)
    up, dn = exchange_part_info(mine, rank, world)
    q.put((rank, up, dn))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_part_wiring_over_gloo(world):
    """Each rank of a multi-part ring connects to the part above (rank - 1) and below (rank + 1),
    periodically, with that rank's own handles, inbox offset and row count."""
    from paper_2508_16639_b200.bands import band_rows

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        r, up, dn = q.get(timeout=120)
        got[r] = (up, dn)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows = [r for _, r in band_rows(4096, world)]
    for r in range(world):
        u, d = (r - 1) % world, (r + 1) % world
        assert got[r][0] == (bytes([u]) * 192, 1000 + u, rows[u])
        assert got[r][1] == (bytes([d]) * 192, 1000 + d, rows[d])
