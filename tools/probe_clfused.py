"""Fused XQuant-CL accumulate (xq_decode_attend_absorbed_cl) vs the two-launch path
on one shape (debug tool): python tools/probe_clfused.py d H B n bits"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from test_gpu_clfused import _stack  # noqa: E402

d, H, B, n, bits = (int(a) for a in sys.argv[1:6])
L_max = -(-(n + 8) // 128) * 128
outs, accs = [], []
for fused in (True, False):
    caches, ws, acc, q = _stack(d, H, bits, B, [n - 3 * s for s in range(B)], seed=1, L_max=L_max)
    if not fused:
        acc.settle()
    out = caches[2].decode_attend(q, ws[2], acc)
    torch.cuda.synchronize()
    outs.append(out.cpu())
    accs.append(acc.x16.cpu())
print(f"d={d} H={H} B={B} n={n} bits={bits}: out max diff {float((outs[0]-outs[1]).abs().max()):.3e} "
      f"acc equal {torch.equal(accs[0], accs[1])}", flush=True)
