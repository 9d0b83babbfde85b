"""kvq, the quantized-KV decode baseline (QuantizedKvCache, cache.py:326-360;
SURVEY 8(f) row 3), on the GPU against the reference's golden-pinned oracle:
codes of both streams, remat K/V and decode attention across flushes."""

import math

import numpy as np
import pytest

from _util import rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.mark.parametrize("bits,g", [(3, 1), (4, 1), (2, 4)])
def test_kvq_decode_against_oracle(bits, g):
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import cache as M

    d, H = 1024, 8
    kvw = d // g
    gen = torch.Generator().manual_seed(bits + g)
    st = M.make_cache("kvq", 0, M.LayerPolicy.uniform(bits, 1), 128, 128, n_slots=2, max_len=512,
                      hidden_dim=d, n_heads=H, kv_group=g)
    w = M.LayerWeights(w_k=(torch.randn(d, kvw, generator=gen) / math.sqrt(d)).to(torch.bfloat16).cuda(),
                       w_v=(torch.randn(d, kvw, generator=gen) / math.sqrt(d)).to(torch.bfloat16).cuda())
    lens = [250, 120]
    xs = [torch.randn(n + 12, d, generator=gen).to(torch.bfloat16) for n in lens]
    for s, n in enumerate(lens):
        st.prefill(xs[s][:n].cuda(), w, slot=s)
    wk = w.w_k.double().cpu().numpy()
    wv = w.w_v.double().cpu().numpy()
    orc = [O.KvqCache(bits, 128, 128) for _ in lens]
    for s, n in enumerate(lens):
        # K/V projected like the GPU (fp32 GEMM) so the codes compare stage-wise
        xb = xs[s][:n].cuda().float()
        orc[s].prefill((xb @ w.w_k.float()).double().cpu().numpy(),
                       (xb @ w.w_v.float()).double().cpu().numpy())
    for t in range(12):  # crosses the 256-token K flush of slot 0
        xt = torch.stack([xs[s][lens[s] + t] for s in range(2)]).cuda()
        st.decode_append(xt, w)
        kk, vv = xt.float() @ w.w_k.float(), xt.float() @ w.w_v.float()
        for s in range(2):
            orc[s].push(kk[s].double().cpu().numpy(), vv[s].double().cpu().numpy())
        q = torch.randn(2, H, 128, generator=gen)
        out = st.decode_attend(q.cuda(), w).cpu().numpy()
        for s in range(2):
            n = lens[s] + t + 1
            k, v = orc[s].remat()
            ref = O.attention(O.apply_rope(q[s].double().numpy().reshape(1, -1), [n - 1], 128), k, v, H, g)[0]
            assert rel_err(out[s].reshape(-1), ref) <= TOL, (t, s)
    # codes of slot 0 (flushed K groups, quantized V rows) vs the oracle, stage-wise
    ks, vs = st.k_stream, st.v_stream
    nk = int(ks.n_flushed[0])
    got = ks.codes[:nk].cpu().numpy()
    un = np.stack([O.unpack_codes(got[r].view(np.uint64), bits, kvw) for r in range(nk)])
    assert np.mean(un != orc[0].k.codes[:nk]) <= 1e-3
    kk, vv = st.rematerialize(w, np.arange(lens[0] + 12))
    k, v = orc[0].remat()
    assert rel_err(kk.cpu().numpy(), k) <= TOL
    assert rel_err(vv.cpu().numpy(), v) <= TOL


def test_kvq_against_reference_golden():
    """The reference's own kvq run (tests/golden, make_golden.py): 4 query heads on
    2 KV heads, 3-bit, prefill 250 + 12 decode steps through the K flush."""
    import torch

    from _util import golden, torch_bf16
    from paper_2508_10395_b200 import cache as M

    z = golden("backends")
    x = torch_bf16(z["kvq_x"])
    q = torch_bf16(z["kvq_q"]).float()
    w = M.LayerWeights(w_k=torch_bf16(z["kvq_wk"]), w_v=torch_bf16(z["kvq_wv"]))
    st = M.make_cache("kvq", 0, M.LayerPolicy.uniform(3, 1), 128, 128, n_slots=1, max_len=384,
                      hidden_dim=512, n_heads=4, kv_group=2)
    st.prefill(x[:250], w)
    errs = []
    for t in range(12):
        st.decode_append(x[250 + t][None], w)
        out = st.decode_attend(q[t][None], w)
        errs.append(rel_err(out.reshape(-1).cpu().numpy(), z["kvq_attn"][t]))
    assert max(errs) <= TOL, errs
    kk, vv = st.rematerialize(w, np.arange(262))
    assert rel_err(kk.cpu().numpy(), z["kvq_k"]) <= TOL
    assert rel_err(vv.cpu().numpy(), z["kvq_v"]) <= TOL
    assert int(st.v_stream.n_flushed[0]) == 250 and int(st.k_stream.n_flushed[0]) == 256
