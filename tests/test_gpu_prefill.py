"""Prefill path on the GPU: bulk quantization of the prompt
(``prefill``), K/V rebuilt from the cache just written, causal attention over
all prompt positions (``_Session.prefill``, model.py:205-221) -- against the
CPU oracle on the same inputs, every variant."""

import math

import numpy as np
import pytest

from _util import rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _bf16(t):
    import torch

    return t.to(torch.bfloat16)


def _q_rot(q, n):
    import xq_oracle as O

    return O.apply_rope(q, np.arange(n), 128)


@pytest.mark.parametrize("variant,bits", [("xq-mha", 3), ("xq-mha", 4), ("fp16", 16), ("kvq", 4),
                                          ("xq-mha", 16)])
def test_prefill_mha_against_oracle(variant, bits):
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import cache as M

    d, H = 512, 4
    g = torch.Generator().manual_seed(bits)
    pol = M.LayerPolicy.uniform(bits, 1)
    st = M.make_cache(variant, 0, pol, 128, 128, n_slots=2, max_len=512, hidden_dim=d, n_heads=H)
    w = M.LayerWeights(w_k=_bf16(torch.randn(d, d, generator=g) / math.sqrt(d)).cuda(),
                       w_v=_bf16(torch.randn(d, d, generator=g) / math.sqrt(d)).cuda())
    wk, wv = w.w_k.double().cpu().numpy(), w.w_v.double().cpu().numpy()
    for slot, n in ((1, 300), (0, 130)):
        x = _bf16(torch.randn(n, d, generator=g))
        q = torch.randn(n, d, generator=g)
        ctx = st.prefill_attend(x.cuda(), q.cuda(), w, slot=slot).cpu().numpy().reshape(n, -1)
        xs = x.double().numpy()
        if variant == "fp16" or bits == 16:
            ref_st = O.Fp16Cache(128)
            ref_st.append(xs, wk, wv)
            k, v = ref_st.remat()
        elif variant == "kvq":
            ref_st = O.KvqCache(bits, 128, 128)
            ref_st.prefill(xs @ wk, xs @ wv)
            k, v = ref_st.remat()
        else:
            ref_st = O.XqMhaCache(bits, 128, 128)
            ref_st.append(xs)
            k, v = ref_st.remat(wk, wv)
        ref = O.attention(_q_rot(q.double().numpy(), n), k, v, H, 1)
        assert rel_err(ctx, ref) <= TOL, (variant, slot)
        assert int(st.n_tokens[slot]) == n


def test_prefill_gqa_against_oracle():
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import cache as M

    d, H, gq = 1024, 8, 4
    r = d // gq
    gen = torch.Generator().manual_seed(3)
    st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, 128, n_slots=1, max_len=512,
                      hidden_dim=d, n_heads=H, kv_group=gq)
    uk = torch.linalg.qr(torch.randn(d, r, generator=gen, dtype=torch.float64))[0]
    uv = torch.linalg.qr(torch.randn(d, r, generator=gen, dtype=torch.float64))[0]
    fk = torch.randn(r, r, generator=gen) / math.sqrt(r)
    fv = torch.randn(r, r, generator=gen) / math.sqrt(r)
    w = M.LayerWeights(u_k=uk.float().cuda(), u_v=uv.float().cuda(), fused_k=fk.cuda(), fused_v=fv.cuda())
    n = 300  # 2 flushed K-latent groups + 44 residual rows
    x = _bf16(torch.randn(n, d, generator=gen))
    q = torch.randn(n, d, generator=gen)
    ctx = st.prefill_attend(x.cuda(), q.cuda(), w).cpu().numpy().reshape(n, -1)
    xs = x.double().numpy()
    ref_st = O.XqGqaCache(3, 128, 128)
    ref_st.prefill(xs @ uk.float().double().numpy(), xs @ uv.float().double().numpy())
    k, v = ref_st.remat(fk.double().numpy(), fv.double().numpy())
    ref = O.attention(_q_rot(q.double().numpy(), n), k, v, H, gq)
    assert rel_err(ctx, ref) <= TOL


@pytest.mark.parametrize("variant", ["xq-cl-mha", "xq-cl-gqa"])
def test_prefill_cross_layer_against_oracle(variant):
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import cache as M
    from paper_2508_10395_b200 import decode as D

    gq = 1 if variant == "xq-cl-mha" else 4
    d, H, L, n = 1024, 8, 4, 260
    shape = D.ModelShape("tiny", d, L, H, gq)
    ws, _ = D.synthetic_weights(shape, variant, torch.device("cuda"), seed=5)
    pol = M.LayerPolicy.for_bits(3, L)
    sts = [M.make_cache(variant, i, pol, 128, 128, n_slots=1, max_len=384, hidden_dim=d,
                        n_heads=H, kv_group=gq) for i in range(L)]
    acc = M.Accumulator(1, 384, d)
    gen = torch.Generator().manual_seed(9)
    base = torch.randn(n, d, generator=gen)
    xs, qs, ctxs = [], [], []
    for i in range(L):
        base = base + 0.03 * torch.randn(n, d, generator=gen)
        xs.append(_bf16(base))
        qs.append(torch.randn(n, d, generator=gen))
        ctxs.append(sts[i].prefill_attend(xs[i].cuda(), qs[i].cuda(), ws[i], acc).cpu().numpy())
    xd = [x.double().numpy() for x in xs]
    if variant == "xq-cl-mha":
        stack = O.XqClMhaStack(pol.bits, pol.base_layers, 128, 128)
        _, kvs = stack.step(xd, [(w.w_k.double().cpu().numpy(), w.w_v.double().cpu().numpy()) for w in ws])
    else:
        stack = O.XqClGqaStack(pol.bits, pol.base_layers, 128, 128)
        o = stack.step(xd, [(w.u_kv.double().cpu().numpy(), w.fused_kv.double().cpu().numpy()) for w in ws])
        kvs = [(e[1], e[2]) for e in o]
    for i in range(L):
        ref = O.attention(_q_rot(qs[i].double().numpy(), n), kvs[i][0], kvs[i][1], H, gq)
        assert rel_err(ctxs[i].reshape(n, -1), ref) <= TOL, i
