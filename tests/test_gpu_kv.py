"""fp16-KV decode baseline (FullPrecisionCache, cache.py:302-323) with grouped query
heads. GROUP > 1 runs the mma.sync kernel `k_kv_decode_gqa`. It is checked against the
float64 oracle attention (model.py:150-182) over the cache's own bf16 K/V, with ragged
sequences, single-token sequences and chunk boundaries inside a sequence."""

import math

import numpy as np
import pytest

from _util import rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("tpc", [None, 1])
def test_fp16_kv_gqa_against_oracle(g, tpc):
    import torch

    import xq_oracle as O
    from paper_2508_10395_b200 import cache as M

    d, H = 1024, 8
    kvw = H // g * 128
    gen = torch.Generator().manual_seed(7 * g + (tpc or 0))
    lens = [700, 1, 37, 300]
    st = M.make_cache("fp16", 0, M.LayerPolicy.uniform(16, 1), 128, n_slots=len(lens), max_len=1024,
                      hidden_dim=d, n_heads=H, kv_group=g)
    w = M.LayerWeights(w_k=(torch.randn(d, kvw, generator=gen) / math.sqrt(d)).to(torch.bfloat16).cuda(),
                       w_v=(torch.randn(d, kvw, generator=gen) / math.sqrt(d)).to(torch.bfloat16).cuda())
    for s, n in enumerate(lens):
        x = torch.randn(n, d, generator=gen).to(torch.bfloat16).cuda()
        st.prefill(x, w, slot=s)
    q = torch.randn(len(lens), H, 128, generator=gen) * 2.0
    out = st.decode_attend(q.cuda(), w, tiles_per_chunk=tpc).cpu().numpy()
    for s, n in enumerate(lens):
        kk, vv = st.rematerialize(w, np.arange(n), slot=s)
        qr = O.apply_rope(q[s].reshape(1, -1).double().numpy(), [n - 1], 128)
        ref = O.attention(qr, kk.double().cpu().numpy(), vv.double().cpu().numpy(), H, g)[0]
        assert rel_err(out[s].reshape(-1), ref) <= TOL, (s, n)
