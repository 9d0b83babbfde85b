"""Quantization groups of 32 and 64 channels in the fused decode kernel.

The reference's group_size is a parameter (quant.py:37-55, cache.py:620-630; 128 by
default, which every benchmark config uses). The fused kernel's per-token producers
take groups of 32, 64 or 128 channels (one or two (scale, zp) per 64-channel chunk);
per-channel streams (the xq-gqa K latent) keep 128-token groups, one per CTA tile.
Checked against the oracle (the reference's float64 algorithm), through the XQuant-CL
fused accumulate (bit-identical to the two-launch path), and through the
reference-signature make_cache against the reference's own run.
"""

import os
import sys

import numpy as np
import pytest

from _util import ROOT, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [32, 64])
@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_xq_mha_group_sizes_match_oracle(G, bits):
    import torch
    import xq_oracle as O

    from paper_2508_10395_b200 import cache as M

    dev = torch.device("cuda", 0)
    d, H, B, n = 512, 4, 2, 300
    g = torch.Generator(device="cpu").manual_seed(bits * 7 + G)
    wk = (torch.randn(d, d, generator=g) / d**0.5).to(torch.bfloat16)
    wv = (torch.randn(d, d, generator=g) / d**0.5).to(torch.bfloat16)
    w = M.LayerWeights(w_k=wk.to(dev), w_v=wv.to(dev))
    st = M.make_cache("xq-mha", 0, M.LayerPolicy.uniform(bits, 1), 128, G, n_slots=B, max_len=512,
                      hidden_dim=d, n_heads=H, device=dev)
    x = torch.randn(B, n + 1, d, generator=g).to(torch.bfloat16)
    st.prefill(x[:, :n].to(dev), w)
    st.decode_append(x[:, n].to(dev), w)
    q = torch.randn(B, H, 128, generator=g)
    out = st.decode_attend(q.to(dev), w).cpu().numpy()
    for s in range(B):
        cache = O.XqMhaCache(bits, 128, G)
        cache.append(x[s].double().numpy())
        kk, vv = cache.remat(wk.double().numpy(), wv.double().numpy())
        qr = O.apply_rope(q[s].double().numpy().reshape(1, -1), [n], 128)
        ref = O.attention(qr, kk, vv, H, 1)[0]
        err = rel_err(out[s].reshape(-1), ref)
        assert err <= 2e-2, (G, bits, s, err)


@pytest.mark.parametrize("G", [32, 64])
def test_cl_fused_accumulate_group_sizes(G):
    """The in-kernel accumulate reads one (scale, zp) per G channels: bit-identical to
    the standalone xq_cl_accumulate for the same groups."""
    import torch

    from paper_2508_10395_b200 import cache as M

    dev = torch.device("cuda", 0)
    d, H, B = 1024, 8, 3
    n = [700, 299, 1000]
    outs, accs = [], []
    for fused in (True, False):
        g = torch.Generator(device="cpu").manual_seed(G)
        policy = M.LayerPolicy([3] * 3, base_layers=2, high_precision_prefix=2)
        caches = [M.make_cache("xq-cl-mha", i, policy, 128, G, n_slots=B, max_len=1024,
                               hidden_dim=d, n_heads=H, device=dev) for i in range(3)]
        ws = [M.LayerWeights(w_k=(torch.randn(d, d, generator=g) / d**0.5).to(torch.bfloat16).to(dev),
                             w_v=(torch.randn(d, d, generator=g) / d**0.5).to(torch.bfloat16).to(dev))
              for _ in range(3)]
        acc = M.Accumulator(B, 1024, d, dev, precision="fp16")
        xs = torch.randn(3, B, max(n) + 1, d, generator=g).to(torch.bfloat16)
        for s in range(B):
            for i, c in enumerate(caches):
                c.prefill(xs[i, s, :n[s]].to(dev), ws[i], acc, slot=s)
        for i, c in enumerate(caches):
            c.decode_append(torch.stack([xs[i, s, n[s]] for s in range(B)]).to(dev), ws[i], acc)
        q = torch.randn(B, H, 128, generator=g).to(dev)
        if not fused:
            acc.settle()
        out = caches[2].decode_attend(q, ws[2], acc)
        assert caches[2].fused_accumulate == fused
        torch.cuda.synchronize()
        outs.append(out.cpu())
        accs.append([acc.x16[s, :n[s] + 1].cpu() for s in range(B)])
    assert torch.equal(outs[0], outs[1])
    assert all(torch.equal(a, b) for a, b in zip(*accs))


def test_reference_cache_group_size_64():
    """The reference-signature make_cache with group_size=64 against the reference's
    own xq-mha cache with the same groups (codes bit-exact, K/V to the fp16 params)."""
    REF = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(REF, "xcache")):
        pytest.skip("oracle/_ref (the reference package) is not built")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from xcache import cache as R
    from xcache.linalg import RngState, gen_weights

    from paper_2508_10395_b200 import cache as M

    d = 512
    rng = RngState(3)
    lw = R.LayerWeights(gamma_attn=np.ones(d), gamma_mlp=np.ones(d), w_q=gen_weights(rng, d, d),
                        w_k=gen_weights(rng, d, d), w_v=gen_weights(rng, d, d),
                        w_o=gen_weights(rng, d, d), w_up=gen_weights(rng, d, 2 * d),
                        w_down=gen_weights(rng, 2 * d, d))
    x = gen_weights(RngState(4), 200, d) * np.sqrt(d)
    pol = R.LayerPolicy.uniform(3, 1)
    ours, theirs = M.make_cache("xq-mha", 0, pol, 128, 64), R.make_cache("xq-mha", 0, pol, 128, 64)
    for mod, st in ((M, ours), (R, theirs)):
        mod.prefill(st, x[:-1], lw)
        mod.decode_append(st, x[-1], lw)
    k, v = M.rematerialize(ours, lw, np.arange(200))
    rk, rv = R.rematerialize(theirs, lw, np.arange(200))
    assert rel_err(k, rk) <= 2e-3 and rel_err(v, rv) <= 2e-3
