import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests"); sys.path.insert(0, ROOT + "/oracle")
from _util import golden, rel_err, torch_bf16, bf16f
import xq_oracle as O
from paper_2508_10395_b200 import cache as M
z = golden("backends")
xs = torch_bf16(z["clg_x"])
bits = [int(b) for b in z["clg_bits"]]
pol = M.LayerPolicy(bits, base_layers=3, high_precision_prefix=3)
ws = [M.LayerWeights(u_kv=torch.from_numpy(z["clg_u"][i]).cuda(), fused_kv=torch_bf16(z["clg_fused"][i])) for i in range(5)]
kw = dict(n_slots=1, max_len=384, hidden_dim=1024, n_heads=8, kv_group=4)
fus = bf16f(z["clg_fused"]); xsd = bf16f(z["clg_x"])
n_pre = 250
for i in [1, 2]:
    st = M.make_cache("xq-cl-gqa", i, pol, 128, 128, **kw)
    acc = M.Accumulator(1, 384, 1024)
    acc.seeded = True
    u = z["clg_u"][i].astype(np.float64)
    lat = xsd[i, :n_pre] @ u
    oc = O.Stream(bits[i], O.PER_CHANNEL, 512, 128, True)
    oc.bulk(lat)
    if i == 2:
        st.stream.channel_bulk(0, xs[i, :n_pre].float() @ ws[i].f32("u_kv"))
        st.n_tokens[0] = n_pre
        r1 = st.stream.channel_reconstruct(0, n_pre).cpu().numpy()
        print("layer", i, "bulk only: recon rel", rel_err(r1, oc.reconstruct()))
        st2 = M.make_cache("xq-cl-gqa", i, pol, 128, 128, **kw)
        st2._prefill(0, xs[i, :n_pre], ws[i], acc)
        r2 = st2.stream.channel_reconstruct(0, n_pre).cpu().numpy()
        print("layer", i, "_prefill: recon rel", rel_err(r2, oc.reconstruct()))
        p = st2.stream.params[0].float().cpu().numpy()  # [2, 512] (permuted)
        print("scales gpu[:8]", p[0, :8], "oracle", oc.scales[0, :8])
    else:
        st._prefill(0, xs[i, :n_pre], ws[i], acc)
        r = st.stream.channel_reconstruct(0, n_pre).cpu().numpy()
        print("layer", i, "recon rel", rel_err(r, oc.reconstruct()))
st = M.make_cache("xq-cl-gqa", 2, pol, 128, 128, **kw)
lat_g = xs[2, :n_pre].float() @ ws[2].f32("u_kv")
st.stream.channel_bulk(0, lat_g)
r = st.stream.channel_reconstruct(0, n_pre).cpu().numpy()
oc = O.Stream(bits[2], O.PER_CHANNEL, 512, 128, True)
oc.bulk(xsd[2, :n_pre] @ z["clg_u"][2].astype(np.float64))
orc = oc.reconstruct()
d = np.abs(r - orc)
i, j = np.unravel_index(np.argmax(d), d.shape)
print("flushed part rel", rel_err(r[:128], orc[:128]), "resid part rel", rel_err(r[128:], orc[128:]))
print("worst at row", i, "col", j, "gpu", r[i, j], "oracle", orc[i, j], "lat", lat_g[i, j].item())
rows = np.nonzero(d.max(axis=1) > 1e-2)[0]; cols = np.nonzero(d.max(axis=0) > 1e-2)[0]
print("bad rows", rows[:20], len(rows), "bad cols", cols[:20], len(cols))
