"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing only.

The ESCG path shards without a data-path collective.  Replicas (independent seeds) are
split in contiguous blocks across ranks, each rank runs its block on its own GPU, and rank 0 gathers
the per-replica outcomes (extinction MCS, final counts).  Draws are a function of (seed, MCS, tile),
so results do not depend on the world size; `tests/test_dist.py` checks this on CPU with gloo.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import torch
import torch.distributed as dist


def partition(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [begin, end) of `total` items owned by `rank` (random_batch.hpp:70-72 rule)."""
    return total * rank // world, total * (rank + 1) // world


def world_info() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def max_over_ranks(x: float) -> float:
    """Max of a host scalar over ranks (multi-GPU timings are max over ranks)."""
    rank, world = world_info()
    if world == 1:
        return float(x)
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(local: list) -> List:
    """Concatenate per-rank lists on rank 0 in rank order (other ranks get [])."""
    rank, world = world_info()
    if world == 1:
        return list(local)
    out = [None] * world if rank == 0 else None
    dist.gather_object(local, out, dst=0)
    if rank != 0:
        return []
    return [x for part in out for x in part]


def run_sharded(tasks: Sequence, runner: Callable[[Sequence], list]) -> List:
    """Run `runner` on this rank's contiguous share of `tasks`; rank 0 returns all results in task order."""
    rank, world = world_info()
    b, e = partition(len(tasks), world, rank)
    local = runner(tasks[b:e]) if e > b else []
    assert len(local) == e - b, "runner must return one result per task"
    return gather_to_rank0(local)


def device_replica_runner(params, model, tracked: int = 0, interval: int = 1, device: int = None):
    """Runner for run_sharded: tasks are seeds; each seed is one replica on this rank's GPU.  Returns
    (stop MCS, status, final counts) per seed — the outcomes the experiments harness consumes."""
    from .engine import DeviceEngine

    def run(seeds):
        dev = torch.cuda.current_device() if device is None else device
        with DeviceEngine(params, model, n_replicas=len(seeds), seeds=list(seeds), device=dev) as eng:
            eng.init_lattice()
            eng.run(params.mcs_limit, interval=interval, tracked=tracked, record_trace=False)
            out = []
            for r in range(len(seeds)):
                m, st, last = eng.replica_result(r)
                out.append((int(m), int(st), [int(c) for c in last]))
            return out

    return run
