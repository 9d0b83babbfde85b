"""Decode engine (decode.Decoder) on the GPU: a multi-layer step against the
CPU oracle, and KV-head-group shards reassembling the unsharded output."""


import numpy as np
import pytest

from _util import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("kernel_path")]

TOL = 2e-2


def _setup(variant, bits, n_layers=4, d=512, H=4, g=1, B=2, n=300, seed=0):
    import torch

    from paper_2508_10395_b200 import decode as D

    shape = D.ModelShape("tiny", d, n_layers, H, g)
    dev = torch.device("cuda", 0)
    w, wq = D.synthetic_weights(shape, variant, dev, seed=seed)
    gen = torch.Generator(device="cpu").manual_seed(seed + 1)
    xs = torch.randn(n_layers, B, n + 1, d, generator=gen).to(torch.bfloat16)
    return shape, w, wq, xs, dev


def _run(shape, variant, bits, w, wq, xs, dev, head_shard=None):
    import torch

    from paper_2508_10395_b200 import decode as D

    L, B, n1, d = xs.shape
    dec = D.Decoder(shape, variant, bits, B, 512, w, wq, device=dev, head_shard=head_shard)
    dec.gather = None  # single process: shards are concatenated by the test
    for s in range(B):
        for i, c in enumerate(dec.caches):
            c._prefill(s, xs[i, s, :-1].to(dev), dec.weights[i], dec.acc)
    dec.n_tokens[:] = n1 - 1
    dec.lens_dev.fill_(n1 - 1)
    out = torch.empty((L, B, dec.n_heads_local, 128), dtype=torch.float32, device=dev)
    dec.step(xs[:, :, -1].to(dev).contiguous(), attn_out=out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), dec


@pytest.mark.parametrize("variant,bits", [("xq-mha", 3), ("xq-mha", 4), ("fp16", 16)])
def test_decoder_step_matches_oracle(variant, bits):
    import xq_oracle as O

    shape, w, wq, xs, dev = _setup(variant, bits)
    out, dec = _run(shape, variant, bits, w, wq, xs, dev)
    L, B, n1, d = xs.shape
    x = xs.double().numpy()
    for i in range(L):
        wk, wv = w[i].w_k.double().cpu().numpy(), w[i].w_v.double().cpu().numpy()
        wqi = wq[i].double().cpu().numpy()
        for b in range(B):
            if variant == "fp16":
                st = O.Fp16Cache(128)
                st.append(x[i, b], wk, wv)
                k, v = st.remat()
            else:
                st = O.XqMhaCache(dec.policy.bits[i], 128, 128)
                st.append(x[i, b])
                k, v = st.remat(wk, wv)
            q = x[i, b, -1:] @ wqi
            ref = O.attention(O.apply_rope(q, [n1 - 1], 128), k, v, shape.n_heads, 1)[0]
            assert rel_err(out[i, b].reshape(-1), ref) <= TOL, (i, b)


@pytest.mark.parametrize("variant,g", [("xq-mha", 1), ("xq-gqa", 2)])
def test_head_shards_reassemble(variant, g):
    shape, w, wq, xs, dev = _setup(variant, 3, n_layers=2, d=1024, H=8, g=g)
    full, _ = _run(shape, variant, 3, w, wq, xs, dev)
    parts = [_run(shape, variant, 3, w, wq, xs, dev, head_shard=(2, r))[0] for r in range(2)]
    got = np.concatenate(parts, axis=2)
    assert got.shape == full.shape
    assert np.max(np.abs(got - full)) <= 1e-5 * np.max(np.abs(full))


def test_decoder_cl_step_matches_oracle():
    import xq_oracle as O

    shape, w, wq, xs, dev = _setup("xq-cl-mha", 2, n_layers=5, d=256, H=2)
    # residual-stream-like inputs (the regime CL is for): x_i = x_{i-1} + 0.03 noise
    import torch

    base = xs[0].float()
    drift = [base]
    for i in range(1, xs.shape[0]):
        drift.append(drift[-1] + 0.03 * xs[i].float())
    xs = torch.stack(drift).to(torch.bfloat16)
    out, dec = _run(shape, "xq-cl-mha", 2, w, wq, xs, dev)
    L, B, n1, d = xs.shape
    x = xs.double().numpy()
    for b in range(B):
        stack = O.XqClMhaStack(dec.policy.bits, dec.policy.base_layers, 128, 128)
        stack.step([x[i, b, :-1] for i in range(L)])
        weights = [(w[i].w_k.double().cpu().numpy(), w[i].w_v.double().cpu().numpy()) for i in range(L)]
        _, kvs = stack.step([x[i, b, -1] for i in range(L)], weights)
        for i in range(L):
            q = x[i, b, -1:] @ wq[i].double().cpu().numpy()
            ref = O.attention(O.apply_rope(q, [n1 - 1], 128), kvs[i][0], kvs[i][1], shape.n_heads, 1)[0]
            assert rel_err(out[i, b].reshape(-1), ref) <= TOL, (i, b)


def test_decoder_cl_gqa_step_matches_oracle():
    """xq-cl-gqa through the decode engine: 5 layers (base 3), 8 query heads on 2 KV
    heads, the shared K|V subspace from the SVD of [W_k | W_v]; against the oracle
    (the reference's float64 algorithm) on the same inputs."""
    import torch

    import xq_oracle as O

    shape, w, wq, xs, dev = _setup("xq-cl-gqa", 3, n_layers=5, d=1024, H=8, g=4, n=260)
    base = xs[0].float()
    drift = [base]
    for i in range(1, xs.shape[0]):
        drift.append(drift[-1] + 0.03 * xs[i].float())
    xs = torch.stack(drift).to(torch.bfloat16)
    out, dec = _run(shape, "xq-cl-gqa", 3, w, wq, xs, dev)
    L, B, n1, d = xs.shape
    x = xs.double().numpy()
    subs = [(w[i].u_kv.double().cpu().numpy(), w[i].fused_kv.double().cpu().numpy()) for i in range(L)]
    for b in range(B):
        stack = O.XqClGqaStack(dec.policy.bits, dec.policy.base_layers, 128, 128)
        stack.step([x[i, b, :-1] for i in range(L)], subs)
        o = stack.step([x[i, b, -1] for i in range(L)], subs)
        for i in range(L):
            q = x[i, b, -1:] @ wq[i].double().cpu().numpy()
            ref = O.attention(O.apply_rope(q, [n1 - 1], 128), o[i][1], o[i][2], shape.n_heads, 4)[0]
            assert rel_err(out[i, b].reshape(-1), ref) <= TOL, (i, b)


class _LocalPeers:
    """Stand-in for parallel.PeerHeadGather with every rank's decoder in this process:
    the "peer" buffers are ordinary device tensors. The fused kernel's peer stores and
    the decoder's plumbing run exactly as over NVLink. Only the pointers come from
    elsewhere, and the barrier is a no-op because the ranks run in stream order."""

    peer = True

    def __init__(self, bufs, rank):
        self.bufs, self.rank = bufs, rank  # bufs[rank][parity]: [world, B, H_local, 128]

    def out_ptrs(self, layer):
        slot = self.bufs[0][0][0].numel() * 4
        return [b[layer % 2].data_ptr() + self.rank * slot for b in self.bufs]

    def finish(self, layer):
        from paper_2508_10395_b200 import parallel as P

        return P.gathered_view(self.bufs[self.rank][layer % 2])

    def __call__(self, local, layer=0):
        for b in self.bufs:
            b[layer % 2][self.rank].copy_(local)
        return self.finish(layer)


@pytest.mark.parametrize("variant,g", [("xq-mha", 1), ("xq-gqa", 2)])
def test_peer_store_gather(variant, g, kernel_path):
    """KV-head-group sharding with the gather done by the projection kernel's peer
    stores (xq_decode_attend_absorbed_peers): every rank's buffer holds the unsharded
    output, and attn_out keeps the local heads."""
    import torch

    from paper_2508_10395_b200 import decode as D

    world = 2
    shape, w, wq, xs, dev = _setup(variant, 3, n_layers=3, d=1024, H=8, g=g)
    full, _ = _run(shape, variant, 3, w, wq, xs, dev)
    L, B, n1, d = xs.shape
    h_loc = shape.n_heads // world
    bufs = [[torch.full((world, B, h_loc, 128), float("nan"), device=dev) for _ in range(2)]
            for _ in range(world)]
    locals_ = []
    for r in range(world):
        dec = D.Decoder(shape, variant, 3, B, 512, w, wq, device=dev, head_shard=(world, r))
        dec.gather = _LocalPeers(bufs, r)
        for s in range(B):
            for i, c in enumerate(dec.caches):
                c._prefill(s, xs[i, s, :-1].to(dev), dec.weights[i], dec.acc)
        dec.n_tokens[:] = n1 - 1
        dec.lens_dev.fill_(n1 - 1)
        out = torch.empty((L, B, h_loc, 128), dtype=torch.float32, device=dev)
        last = dec.step(xs[:, :, -1].to(dev).contiguous(), attn_out=out)
        torch.cuda.synchronize()
        locals_.append(out.cpu().numpy())
        assert last.shape == (B, shape.n_heads, 128)
        if kernel_path == "absorbed":  # the absorbed kernel did the peer stores
            assert all(c.peer_stored for c in dec.caches)
    scale = np.max(np.abs(full))
    np.testing.assert_allclose(np.concatenate(locals_, axis=2), full, atol=1e-5 * scale, rtol=0)
    for r in range(world):  # the last two layers' buffers (parity L-1, L-2) on every rank
        for i in (L - 1, L - 2):
            from paper_2508_10395_b200 import parallel as P

            got = P.gathered_view(bufs[r][i % 2]).cpu().numpy()
            np.testing.assert_allclose(got, full[i], atol=1e-5 * scale, rtol=0)
