"""Probe: torch symmetric memory between 2 processes that share one GPU (gloo group).

    python tools/probe_symm.py
"""
import os

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch.distributed._symmetric_memory as symm

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    buf = symm.empty((world, 4), dtype=torch.float32, device=dev)
    buf.fill_(-1)
    hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
    print(rank, "ptrs", [hex(p) for p in hdl.buffer_ptrs], flush=True)
    # write my row into every peer's buffer through its pointer
    for p in range(world):
        peer = hdl.get_buffer(p, (world, 4), torch.float32)
        peer[rank].fill_(rank + 10)
    hdl.barrier(channel=0)
    torch.cuda.synchronize()
    print(rank, "buf", buf.cpu().tolist(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2,), nprocs=2)
