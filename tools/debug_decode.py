"""Dump the fused kernel's raw accumulator for a small xq-mha case (debug)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_10395_b200 import _native as N  # noqa: E402
from paper_2508_10395_b200 import cache as M  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = sys.argv[2] if len(sys.argv) > 2 else "codes"
d, H, n = 256, 2, 300
g = torch.Generator().manual_seed(0)
x = torch.randn(n, d, generator=g).to(torch.bfloat16).cuda()
wk = (torch.randn(d, d, generator=g) / 16).to(torch.bfloat16).cuda()
wv = (torch.randn(d, d, generator=g) / 16).to(torch.bfloat16).cuda()
q = torch.randn(1, H, 128, generator=g).cuda()
w = M.LayerWeights(w_k=wk, w_v=wv)
pol = M.LayerPolicy.uniform(16 if mode == "f16" else bits, 1)
st = M.make_cache("xq-mha", 0, pol, 128, n_slots=1, max_len=512, hidden_dim=d, n_heads=H)
st.prefill(x, w)
n_tiles = 3
dbg = torch.zeros((1, H, n_tiles, 128, 256), dtype=torch.float32, device="cuda")
N.call("xq_debug_set_acc_dump", N.ptr(dbg), n_tiles)
out = st.decode_attend(q, w)
torch.cuda.synchronize()
N.call("xq_debug_set_acc_dump", None, 0)
if mode == "f16":
    xh = st.x16[:n].float()
else:
    xh = torch.empty((n, d), dtype=torch.float32, device="cuda")
    s = st.stream
    N.call("xq_dequant_rows", N.ptr(s.codes), s.row_bytes, N.ptr(s.params), 0, bits, 128, d, 0, n,
           N.ptr(xh), N.stream_of())
kk, vv = st.rematerialize(w, np.arange(n))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez(os.path.join(ROOT, "gpurun_out", f"dbg_{mode}_{bits}.npz"), acc=dbg.cpu().numpy(),
         xh=xh.cpu().numpy(), wk=wk.float().cpu().numpy(), wv=wv.float().cpu().numpy(),
         out=out.cpu().numpy(), q=q.cpu().numpy(), k=kk.cpu().numpy(), v=vv.cpu().numpy(),
         arr=w._cache[next(k for k in w._cache if k[0] == "mha")].float().cpu().numpy())
ref = (xh @ wk.float())
print("tile0 K err", (dbg[0, 0, 0, :, :128] - ref[:128, :128]).abs().max().item(), ref.abs().max().item())
