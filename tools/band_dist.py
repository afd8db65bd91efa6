"""One lattice sharded by rows over GPUs, one process per GPU (NCCL halo exchange).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/band_dist.py \
        --length 3200 --mcs 100 --kmcs 2 [--check]

Each rank owns one row band (paper_2508_16639_b200.bands.DistributedBand) on cuda:LOCAL_RANK; every
chunk of kmcs MCS the halo rows move with NCCL send/recv straight between the engines' device
buffers.  Prints the whole-lattice attempts/s (max over ranks of the device time).  --check makes
rank 0 also run the single lattice and compare the gathered bands bit for bit.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_16639_b200 as escg  # noqa: E402
from paper_2508_16639_b200.bands import DistributedBand  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, default=3200)
    ap.add_argument("--mcs", type=int, default=100)
    ap.add_argument("--kmcs", type=int, default=2)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = args.length
    p = escg.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10 ** 9)
    model = escg.make_circulant(3, [1])
    with DistributedBand(p, model, rank, world, device=local, kmcs=args.kmcs) as band:
        band.init_lattice()  # global-coordinate init: every band draws its own rows
        band.advance(args.kmcs)  # warm-up
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        band.advance(args.mcs)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        counts = torch.tensor(band.counts().astype(np.int64), device="cuda")
        dist.all_reduce(counts)
        if args.check:
            part = torch.tensor(band.get_band(), device="cuda")
            sizes = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([part.numel()], device="cuda"))
            parts = [torch.zeros(int(s.item()), dtype=part.dtype, device="cuda") for s in sizes]
            dist.all_gather(parts, part)
    if rank == 0:
        print("bands=%d L=%d mcs=%d: %.3e attempts/s (max-over-ranks wall of the advance), counts %s"
              % (world, L, args.mcs, L * L * args.mcs / dt.item(), counts.tolist()), flush=True)
        if args.check:
            got = torch.cat(parts).cpu().numpy()
            with escg.DeviceEngine(p, model, kernel="block", device=local) as eng:
                eng.init_lattice()
                eng.advance(args.kmcs + args.mcs)
                want = eng.get_lattice()
            print("bit-exact vs single lattice:", bool(np.array_equal(got, want)), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
