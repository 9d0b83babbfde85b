"""Host-side multi-GPU logic on CPU: sharding helpers, and a world_size-2 gloo
run where each rank computes the attention of its KV-head shard with the CPU
oracle and HeadGather (the same all_gather_into_tensor the NCCL path uses)
assembles the full output, which must equal the unsharded oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_10395_b200 import parallel as P
from paper_2508_10395_b200.cache import LayerWeights
from paper_2508_10395_b200.errors import ConfigError


def test_batch_shard_partitions():
    for n, world in [(8, 1), (8, 2), (16, 8), (10, 4), (3, 8)]:
        got = [list(P.batch_shard(n, world, r)) for r in range(world)]
        assert sum(got, []) == list(range(n))
        sizes = [len(g) for g in got]
        assert max(sizes) - min(sizes) <= 1


def test_head_shard_and_wq_columns():
    assert P.head_shard(8, 2, 1) == range(4, 8)
    with pytest.raises(ConfigError):
        P.head_shard(8, 3, 0)
    wq = torch.arange(4 * 8 * 128, dtype=torch.float32).view(4, 8 * 128)
    # GQA group 4: kv heads 1..2 serve query heads 4..7 -> columns 512..1024
    got = P.shard_wq(wq, range(1, 2), 4)
    assert torch.equal(got, wq[:, 512:1024])


def test_shard_layer_weights_slices_columns():
    d = 256
    lw = LayerWeights(w_k=torch.randn(d, d), w_v=torch.randn(d, d),
                      u_k=torch.randn(d, 128), u_v=torch.randn(d, 128),
                      fused_k=torch.randn(128, 256), fused_v=torch.randn(128, 256))
    s = P.shard_layer_weights(lw, "xq-gqa", range(1, 2))
    assert torch.equal(s.w_k, lw.w_k[:, 128:256]) and torch.equal(s.fused_v, lw.fused_v[:, 128:])
    assert s.u_k is lw.u_k  # the latent projection stays whole (replicated cache)
    assert s._cache == {} and s._cache is not lw._cache


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, variant, out_q):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
    import xq_oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)  # identical inputs on every rank
        d, hd = 512, 128
        g = 1 if variant == "xq-mha" else 2
        H, n_kv = d // hd, d // hd // g
        n, B = 200, 2
        x = rng.normal(size=(B, n, d))
        w_k = rng.normal(size=(d, n_kv * hd)) / np.sqrt(d)
        w_v = rng.normal(size=(d, n_kv * hd)) / np.sqrt(d)
        q = rng.normal(size=(B, H * hd))
        lw = LayerWeights(w_k=torch.from_numpy(w_k), w_v=torch.from_numpy(w_v))
        kv = P.head_shard(n_kv, world, rank)
        local = P.shard_layer_weights(lw, "xq-mha", kv)
        qcols = slice(kv.start * g * hd, kv.stop * g * hd)
        outs = []
        for b in range(B):
            st = O.XqMhaCache(3, hd, 128)
            st.append(x[b])
            k, v = st.remat(local.w_k.numpy(), local.w_v.numpy())
            qr = O.apply_rope(q[b:b + 1, qcols], [n - 1], hd)
            outs.append(O.attention(qr, k, v, len(kv) * g, g)[0])
        mine = torch.tensor(np.stack(outs), dtype=torch.float32).view(B, len(kv) * g, hd)
        full = P.HeadGather(B, len(kv) * g, world, "cpu")(mine)
        if rank == 0:
            refs = []
            for b in range(B):
                st = O.XqMhaCache(3, hd, 128)
                st.append(x[b])
                k, v = st.remat(w_k, w_v)
                refs.append(O.attention(O.apply_rope(q[b:b + 1], [n - 1], hd), k, v, H, g)[0])
            ref = np.stack(refs).reshape(B, H, hd)
            out_q.put(float(np.max(np.abs(full.numpy() - ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["xq-mha", "gqa-group2"])
def test_head_sharded_attention_gloo_world2(variant):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, variant, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=5) < 1e-5


def test_bench_rank_split():
    """bench.py's per-rank workload: configs[2] (C3) is one global batch of 16 split
    by sequence (16/n per GPU), C4 serves the whole batch per KV-head shard, C2 is
    weak scaling; both arms print the same config dict."""
    import importlib
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    bench = importlib.import_module("bench")
    for world in (1, 2, 4, 8):
        c3 = [bench._split(bench.CONFIGS["c3"], world, r) for r in range(world)]
        assert sum(b for b, _, _ in c3) == 16 and all(t == 16 for _, t, _ in c3)
        assert [s for _, _, s in c3] == [sum(b for b, _, _ in c3[:r]) for r in range(world)]
        c4 = [bench._split(bench.CONFIGS["c4"], world, r) for r in range(world)]
        assert all(b == 32 and t == 32 for b, t, _ in c4)
        c2 = [bench._split(bench.CONFIGS["c2"], world, r) for r in range(world)]
        assert all(b == 8 and t == 8 * world for b, t, _ in c2)
        for name in bench.CONFIGS:
            cfg = bench._config_dict(bench.CONFIGS[name], world)
            assert cfg["global_batch"] == bench._split(bench.CONFIGS[name], world, 0)[1]
