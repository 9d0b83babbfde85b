"""KV-head-group sharding over NCCL on >= 2 GPUs: every rank runs
decode.Decoder(head_shard=(world, rank)) on the same inputs; the gathered
output (NCCL all-gather, and the projection kernel's peer stores into torch
symmetric memory) must equal the unsharded decoder's on rank 0. Skipped when
fewer than two GPUs are visible (the gloo world-2 test in test_parallel.py
covers the host logic on CPU)."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

needs_two = pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                               reason="needs >= 2 GPUs")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, variant, gather, q):
    import torch.distributed as dist

    from paper_2508_10395_b200 import decode as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        g = 4 if variant == "xq-gqa" else 1
        shape = D.ModelShape("t", 2048, 3, 16, g)
        w, wq = D.synthetic_weights(shape, variant, dev, seed=0)
        gen = torch.Generator(device=dev).manual_seed(1)
        B, n = 4, 700
        dec = D.Decoder(shape, variant, 3, B, 1024, w, wq, device=dev, head_shard=(world, rank),
                        gather=gather)
        dec.fill_synthetic(n, seed=2)
        x = torch.randn(shape.n_layers, B, shape.hidden_dim, generator=gen, device=dev).to(torch.bfloat16)
        out = dec.step(x)
        torch.cuda.synchronize()
        if rank == 0:
            full = D.Decoder(shape, variant, 3, B, 1024, w, wq, device=dev)
            full.fill_synthetic(n, seed=2)
            ref = full.step(x)
            q.put(((out - ref).abs().max() / ref.abs().max()).item())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@needs_two
@pytest.mark.parametrize("variant,gather", [("xq-mha", "nccl"), ("xq-gqa", "nccl"),
                                            ("xq-gqa", "peer")])
def test_head_sharded_decoder_nccl(variant, gather):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, variant, gather, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=5) <= 1e-5
