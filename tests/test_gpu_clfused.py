"""XQuant-CL accumulate fused into the delta layer's decode kernel
(xq_decode_attend_absorbed_cl, XQ_A_F16_ACC).

The delta layer's ``acc += deq(deltas)`` (cache.py:472-481, Accumulator.add
cache.py:139-146) runs in the first K pass of the fused kernel instead of a
separate xq_cl_accumulate launch. It computes the same fp16 values with the
same arithmetic and feeds the same operand to the same MMAs, so the fused and
the two-launch paths must agree BIT FOR BIT, both in the accumulator rows they
leave behind and in the attention output. Covered: 2/3/4/8-bit deltas, one K
pass (4 KV heads: the V side is the first reader of the written-back rows) and
several passes (odd passes walk the chunks backwards), ragged lengths across
slots, a tile straddling the arena end, and a multi-layer decode step of the
engine against the CPU oracle.
"""

import numpy as np
import pytest

from _util import rel_err

pytestmark = pytest.mark.gpu


def _stack(d, H, bits, B, n, seed, L_max=1152):
    """Three layers (base, seeding base, delta) of xq-cl-mha with the fp16
    accumulator, prefilled with n[b] tokens per slot and one decode append."""
    import torch

    from paper_2508_10395_b200 import cache as M

    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(seed)
    policy = M.LayerPolicy([bits] * 3, base_layers=2, high_precision_prefix=2)
    caches = [M.make_cache("xq-cl-mha", i, policy, 128, n_slots=B, max_len=L_max, hidden_dim=d,
                           n_heads=H, device=dev) for i in range(3)]
    for c in caches:
        c.absorb = True  # the absorbed kernel whatever the size (the fused path needs it)
    ws = [M.LayerWeights(w_k=(torch.randn(d, d, generator=g) / d**0.5).to(torch.bfloat16).to(dev),
                         w_v=(torch.randn(d, d, generator=g) / d**0.5).to(torch.bfloat16).to(dev))
          for _ in range(3)]
    acc = M.Accumulator(B, L_max, d, dev, precision="fp16")
    xs = torch.randn(3, B, max(n) + 1, d, generator=g).to(torch.bfloat16)
    for s in range(B):
        for i, c in enumerate(caches):
            c.prefill(xs[i, s, :n[s]].to(dev), ws[i], acc, slot=s)
    # ragged: every slot appends one token at its own length
    for i, c in enumerate(caches):
        rows = torch.stack([xs[i, s, n[s]] for s in range(B)]).to(dev)
        c.decode_append(rows, ws[i], acc)
    q = torch.randn(B, H, 128, generator=g).to(dev)
    return caches, ws, acc, q


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("d,H", [(512, 4), (1024, 8)])
def test_fused_accumulate_bit_identical(bits, d, H):
    import torch

    n = [700, 299, 1100]  # the last tile of the last slot runs past the 1152-row arena
    outs, accs = [], []
    for fused in (True, False):
        caches, ws, acc, q = _stack(d, H, bits, len(n), n, seed=bits * 10 + H)
        delta = caches[2]
        assert acc.pending is not None and acc.pending[0] is delta
        if not fused:
            acc.settle()  # the two-launch path: xq_cl_accumulate, then the F16-row kernel
        out = delta.decode_attend(q, ws[2], acc)
        assert delta.fused_accumulate == fused
        assert acc.pending is None
        torch.cuda.synchronize()
        outs.append(out.cpu())
        accs.append([acc.x16[s, :n[s] + 1].cpu() for s in range(len(n))])
    assert torch.equal(outs[0], outs[1]), float((outs[0] - outs[1]).abs().max())
    for a, b in zip(accs[0], accs[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("d,H", [(512, 4), (1024, 8)])
def test_fused_accumulate_many_tiles_per_cluster(d, H):
    """More 256-token tiles than CTA pairs: every CTA pair runs several tiles, so the
    first-pass stage loads of one tile follow the previous tile's later passes."""
    import torch

    n = [3000, 2900, 2999, 1500, 2048, 2100]
    n = n + [x - 7 for x in n]  # 118 tiles for 74 CTA pairs
    outs, accs = [], []
    for fused in (True, False):
        caches, ws, acc, q = _stack(d, H, 3, len(n), n, seed=5, L_max=3072)
        if not fused:
            acc.settle()
        out = caches[2].decode_attend(q, ws[2], acc)
        torch.cuda.synchronize()
        outs.append(out.cpu())
        accs.append([acc.x16[s, :n[s] + 1].cpu() for s in range(len(n))])
    assert torch.equal(outs[0], outs[1]), float((outs[0] - outs[1]).abs().max())
    for a, b in zip(accs[0], accs[1]):
        assert torch.equal(a, b)


def test_settle_before_other_readers():
    """A deferred accumulate is applied before rematerialize / the next layer's update."""
    import torch

    n = [300, 260]
    caches, ws, acc, q = _stack(512, 4, 3, 2, n, seed=7)
    delta = caches[2]
    k, v = delta.rematerialize(ws[2], np.arange(n[0] + 1), acc, slot=0)  # settles
    assert acc.pending is None
    caches2, ws2, acc2, _ = _stack(512, 4, 3, 2, n, seed=7)
    acc2.settle()
    k2, v2 = caches2[2].rematerialize(ws2[2], np.arange(n[0] + 1), acc2, slot=0)
    assert torch.equal(k, k2) and torch.equal(v, v2)


def test_engine_step_with_fused_accumulate_matches_oracle():
    """Decoder.step on an 8-layer xq-cl-mha stack (fused delta layers, 2 K passes)
    against the oracle (the reference's float64 algorithm) on the same inputs."""
    import torch
    import xq_oracle as O

    from paper_2508_10395_b200 import decode as D

    d, H, n_layers, B, n = 1024, 8, 8, 2, 600
    shape = D.ModelShape("tiny", d, n_layers, H, 1)
    dev = torch.device("cuda", 0)
    w, wq = D.synthetic_weights(shape, "xq-cl-mha", dev, seed=3)
    gen = torch.Generator(device="cpu").manual_seed(4)
    # residual-stream-like inputs (the regime CL is for): x_i = x_{i-1} + 0.03 noise
    drift = [torch.randn(B, n + 1, d, generator=gen)]
    for _ in range(1, n_layers):
        drift.append(drift[-1] + 0.03 * torch.randn(B, n + 1, d, generator=gen))
    xs = torch.stack(drift).to(torch.bfloat16)
    dec = D.Decoder(shape, "xq-cl-mha", 2, B, 1024, w, wq, device=dev)
    for c in dec.caches:
        c.absorb = True
    for s in range(B):
        for i, c in enumerate(dec.caches):
            c._prefill(s, xs[i, s, :-1].to(dev), dec.weights[i], dec.acc)
    dec.n_tokens[:] = n
    dec.lens_dev.fill_(n)
    out = torch.empty((n_layers, B, H, 128), dtype=torch.float32, device=dev)
    dec.step(xs[:, :, -1].to(dev).contiguous(), attn_out=out)
    torch.cuda.synchronize()
    fused = [c.fused_accumulate for c in dec.caches[dec.policy.base_layers:]]
    assert all(fused), fused
    out = out.cpu().numpy()
    x = xs.double().numpy()
    weights = [(w[i].w_k.double().cpu().numpy(), w[i].w_v.double().cpu().numpy())
               for i in range(n_layers)]
    for b in range(B):
        stack = O.XqClMhaStack(dec.policy.bits, dec.policy.base_layers, 128, 128)
        stack.step([x[i, b, :-1] for i in range(n_layers)], keep=False)
        _, kvs = stack.step([x[i, b, -1] for i in range(n_layers)], weights, keep=False)
        for i in range(n_layers):
            q = x[i, b, -1:] @ wq[i].double().cpu().numpy()
            ref = O.attention(O.apply_rope(q, [n], 128), kvs[i][0], kvs[i][1], H, 1)[0]
            err = rel_err(out[i, b].reshape(-1), ref)
            assert err <= 2e-2, (i, b, err)
