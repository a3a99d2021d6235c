#!/usr/bin/env python
"""Multi-GPU use of the library: one process per GPU, i-sharded, NCCL all-gather per step.

    torchrun --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 examples/multi_gpu.py [C4] [10]
    python examples/multi_gpu.py C1 10 --loopback 4     # 4 emulated ranks on one GPU

Every rank passes the FULL system (m, x, v); the library copies its own contiguous slice
(nbody_local_range) and exchanges 32-byte j-packets with the other ranks every step
(PAPER.md:140 replicated j data; P:251 multiple accelerators).  Rank 0 creates the NCCL
unique id and the torch process group broadcasts it; energies are collective and global;
results are bit-identical for any number of ranks.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C4")
    ap.add_argument("steps", nargs="?", type=int, default=10)
    ap.add_argument("--loopback", type=int, default=0, help="emulate this many ranks on one GPU")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2509_19294_b200 import binding, inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [binding.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)   # every rank gets rank 0's 128-byte id
        nccl_id = obj[0]

    c = inputs.CONFIGS[a.config]
    m, x, v = inputs.make(a.config)
    kw = dict(world=a.loopback, loopback=True) if a.loopback > 1 else dict(world=world, rank=rank,
                                                                         nccl_id=nccl_id)
    with binding.NBody(m, x, v, eps=c.eps, dt=c.dt, device=local, **kw) as sim:
        ke0, pe0 = sim.energy()                    # collective: every rank calls it
        sim.step(a.steps)                          # predict -> all-gather -> force -> correct
        ke1, pe1 = sim.energy()
        xs, vs = sim.state()                       # this rank's slice [i0, i1)
        sim.sync()
        if rank == 0:
            print(f"{a.config}: N = {c.n}, ranks = {a.loopback or world}, rank 0 owns [{sim.i0}, {sim.i1}); "
                  f"E {ke0 + pe0:.12f} -> {ke1 + pe1:.12f} after {a.steps} steps "
                  f"(relative drift {abs((ke1 + pe1) - (ke0 + pe0)) / abs(ke0 + pe0):.2e})")
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
