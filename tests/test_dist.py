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
