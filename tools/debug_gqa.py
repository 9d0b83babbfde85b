"""Dump the fused kernel's raw accumulator for a small xq-gqa case (debug)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_10395_b200 import _native as N  # noqa: E402
from paper_2508_10395_b200 import cache as M  # noqa: E402

n_pre = int(sys.argv[1]) if len(sys.argv) > 1 else 256
d, H, g = 1024, 8, 4
r = d // g
n = n_pre
gen = torch.Generator().manual_seed(0)
x = torch.randn(n, d, generator=gen).to(torch.bfloat16).cuda()
uk = torch.linalg.qr(torch.randn(d, r, generator=gen))[0].to(torch.bfloat16).cuda()
uv = torch.linalg.qr(torch.randn(d, r, generator=gen))[0].to(torch.bfloat16).cuda()
fk = (torch.randn(r, r, generator=gen) / 16).to(torch.bfloat16).cuda()
fv = (torch.randn(r, r, generator=gen) / 16).to(torch.bfloat16).cuda()
q = torch.randn(1, H, 128, generator=gen).cuda()
w = M.LayerWeights(u_k=uk, u_v=uv, fused_k=fk, fused_v=fv)
st = M.make_cache("xq-gqa", 0, M.LayerPolicy.uniform(3, 1), 128, n_slots=1, max_len=512,
                  hidden_dim=d, n_heads=H, kv_group=g)
st.prefill(x, w)
n_tiles = (n + 127) // 128
dbg = torch.zeros((1, 2, n_tiles, 128, 256), dtype=torch.float32, device="cuda")
N.call("xq_debug_set_acc_dump", N.ptr(dbg), n_tiles)
out = st.decode_attend(q, w)
torch.cuda.synchronize()
N.call("xq_debug_set_acc_dump", None, 0)
ks, vs = st.k_stream, st.v_stream
nf = int(ks.n_flushed[0])
lk = torch.empty((n, r), dtype=torch.float32, device="cuda")
lv = torch.empty((n, r), dtype=torch.float32, device="cuda")
if nf:
    N.call("xq_dequant_rows", N.ptr(ks.codes), ks.row_bytes, N.ptr(ks.params), 1, 3, 128, r, 0, nf,
           N.ptr(lk), N.stream_of())
lk[nf:] = ks.resid[0, : n - nf]
N.call("xq_dequant_rows", N.ptr(vs.codes), vs.row_bytes, N.ptr(vs.params), 0, 3, 128, r, 0, n,
       N.ptr(lv), N.stream_of())
kk, vv = st.rematerialize(w, np.arange(n))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez(os.path.join(ROOT, "gpurun_out", f"dbg_gqa_{n}.npz"), acc=dbg.cpu().numpy(),
         lk=lk.cpu().numpy(), lv=lv.cpu().numpy(), fk=fk.float().cpu().numpy(),
         fv=fv.float().cpu().numpy(), out=out.cpu().numpy(), q=q.cpu().numpy(),
         k=kk.cpu().numpy(), v=vv.cpu().numpy(), nf=nf)
refk = lk @ fk.float()
print("nf", nf, "tile0 K err", (dbg[0, 0, 0, :, :128] - refk[:128, :128]).abs().max().item(),
      refk.abs().max().item())
