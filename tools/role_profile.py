"""Per-role barrier wait fractions of the absorbed kernel.

    bash tools/build_role_profile.sh   # here (cross-compiles)
    python tools/role_profile.py [--config c2] [--layers 4]   # on the GPU box

Runs one decode step of the config with the role-profiling library and prints,
for each role, the fraction of the kernel's cycles it spent blocked on each
barrier (averaged over the warps of that role).
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("XQ_LIB", os.path.join(ROOT, "paper_2508_10395_b200", "libxquant_prof.so"))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_10395_b200 import _native as N  # noqa: E402
from paper_2508_10395_b200 import decode as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--layers", type=int, default=4)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
dev = torch.device("cuda", 0)
shape = D.SHAPES[cfg["shape"]]
B, ctx = cfg["batch"], cfg["ctx"]
L_max = -(-(ctx + 8) // 128) * 128
w, wq = D.synthetic_weights(shape, cfg["variant"], dev, layers=args.layers)
dec = D.Decoder(shape, cfg["variant"], cfg["bits"], B, L_max, w, wq, device=dev)
dec.fill_synthetic(ctx)
xs = [torch.randn(args.layers, B, shape.hidden_dim, device=dev).to(torch.bfloat16) for _ in range(2)]
dec.step(xs[0])
torch.cuda.synchronize()
buf = (C.c_uint64 * 16)()
N.call("xq_debug_role_profile", C.cast(buf, C.c_void_p), 1)
dec.step(xs[1])
torch.cuda.synchronize()
N.call("xq_debug_role_profile", C.cast(buf, C.c_void_p), 1)
v = list(buf)
n_cta = 148
total = v[11] / n_cta  # cycles per CTA
names = [("W-TMA", "empty", 0, n_cta), ("MMA", "tempty", 1, n_cta // 2), ("MMA", "full(K)", 2, n_cta // 2),
         ("MMA", "pready", 3, n_cta // 2), ("MMA", "full(V)", 4, n_cta // 2),
         ("codes-TMA", "cempty", 5, n_cta), ("producer", "cfull", 6, 8 * n_cta),
         ("producer", "empty", 7, 8 * n_cta), ("epilogue", "tfull(K)", 8, 4 * n_cta),
         ("epilogue", "xfull", 9, 4 * n_cta), ("epilogue", "tfull(V)", 10, 4 * n_cta),
         ("epilogue", "[busy K]", 12, 4 * n_cta), ("epilogue", "[busy X]", 13, 4 * n_cta),
         ("epilogue", "[busy V]", 14, 4 * n_cta), ("epilogue", "[setup]", 15, 4 * n_cta)]
print(f"{args.config}: {args.layers} layers, cycles per CTA (sum over launches) {total:.3e}")
for role, bar, c, nw in names:
    print(f"  {role:10s} waits on {bar:9s}: {100 * v[c] / nw / total:5.1f}% of its time")
