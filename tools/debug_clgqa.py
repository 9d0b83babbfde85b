"""Per-layer diagnostics of the xq-cl-gqa backend against the reference golden vectors."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from _util import golden, rel_err, torch_bf16  # noqa: E402
import xq_oracle as O  # noqa: E402
from paper_2508_10395_b200 import cache as M  # noqa: E402

z = golden("backends")
xs = torch_bf16(z["clg_x"])
q = torch_bf16(z["clg_q"]).float()
bits = [int(b) for b in z["clg_bits"]]
pol = M.LayerPolicy(bits, base_layers=int(z["clg_base"]), high_precision_prefix=3)
ws = [M.LayerWeights(u_kv=torch.from_numpy(z["clg_u"][i]).cuda(), fused_kv=torch_bf16(z["clg_fused"][i]))
      for i in range(5)]
kw = dict(n_slots=1, max_len=384, hidden_dim=1024, n_heads=8, kv_group=4)
sts = [M.make_cache("xq-cl-gqa", i, pol, 128, 128, **kw) for i in range(5)]
acc = M.Accumulator(1, 384, 1024)
n_pre, n_dec = 250, 8
# oracle in lock-step, fed the GPU's inputs
ost = O.XqClGqaStack(bits, 3, 128, 128)
subs = [(z["clg_u"][i].astype(np.float64), xs.new_tensor(0) if False else None) for i in range(5)]
from _util import bf16f  # noqa: E402
fus = bf16f(z["clg_fused"])
subs = [(z["clg_u"][i].astype(np.float64), fus[i]) for i in range(5)]
xsd = bf16f(z["clg_x"])
for i in range(5):
    sts[i].prefill(xs[i, :n_pre], ws[i], acc)
ost.step([x[:n_pre] for x in xsd], subs)
for t in range(n_dec):
    outs = []
    for i in range(5):
        sts[i].decode_append(xs[i, n_pre + t][None], ws[i], acc)
        outs.append(sts[i].decode_attend(q[i][None], ws[i], acc).reshape(-1).cpu().numpy())
    o = ost.step([x[n_pre + t] for x in xsd], subs)
n = n_pre + n_dec
for i in range(5):
    k, v = sts[i].rematerialize(ws[i], np.arange(n), acc)
    k, v = k.cpu().numpy(), v.cpu().numpy()
    ref = O.attention(O.apply_rope(bf16f(z["clg_q"])[i:i + 1], [n - 1], 128), o[i][1], o[i][2], 8, 4)[0]
    print(f"layer {i}: fused vs golden {rel_err(outs[i], z['clg_attn'][i]):.2e}  fused vs oracle {rel_err(outs[i], ref):.2e}"
          f"  K {rel_err(k, o[i][1]):.2e}  V {rel_err(v, o[i][2]):.2e}"
          + (f"  acc {rel_err(acc.x_hat[0, :n].cpu().numpy(), o[i][3]):.2e}" if o[i][3] is not None else ""))
print("acc vs golden", rel_err(acc.x_hat[0, :n].cpu().numpy(), z["clg_acc_last"]))
for i in range(5):
    s = sts[i].stream
    nfl = int(s.n_flushed[0])
    got = s.codes[:nfl].cpu().numpy()
    un = np.stack([O.unpack_codes(got[r].view(np.uint64), bits[i], 512) for r in range(nfl)])
    oc = ost.streams[i].codes
    ob = ost.streams[i].buf
    res = s.resid[0, :n - nfl].cpu().numpy()
    print(f"layer {i}: nfl {nfl} oracle rows {oc.shape[0]} code mismatch frac {np.mean(un != oc[:nfl]):.2e}"
          f"  resid rel {rel_err(res, ob):.2e}  golden codes eq {np.array_equal(oc, z[f'clg_codes{i}'])}")
for i in range(5):
    rec = sts[i].stream.channel_reconstruct(0, n).cpu().numpy()
    orc = ost.streams[i].reconstruct()
    kvo = orc @ fus[i]
    k, v = sts[i].rematerialize(ws[i], np.arange(n), acc) if i < 3 else (None, None)
    msg = ""
    if k is not None:
        kpre = O.apply_rope(kvo[:, :256], np.arange(n), 128)
        msg = f"  K(f32 remat) vs oracle-from-own-stream {rel_err(k.cpu().numpy(), kpre):.2e}"
    print(f"layer {i}: recon rel {rel_err(rec, orc):.2e} max|d| {np.abs(rec - orc).max():.3e}{msg}")
