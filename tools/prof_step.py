"""One C2 decode step (or a few layers of it) inside an NVTX range 'step', for ncu.

    ncu --nvtx --nvtx-include "step/" ... python tools/prof_step.py [--layers N] [--config c2]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_10395_b200 import decode as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--variant", default=None)
ap.add_argument("--tpc", type=int, default=None)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
if args.variant:
    cfg["variant"] = args.variant
dev = torch.device("cuda", 0)
shape = D.SHAPES[cfg["shape"]]
n_layers = args.layers or cfg.get("layers", shape.n_layers)
B, ctx = cfg["batch"], cfg["ctx"]
L_max = -(-(ctx + 8) // 128) * 128
w, wq = D.synthetic_weights(shape, cfg["variant"], dev, layers=n_layers)
dec = D.Decoder(shape, cfg["variant"], cfg["bits"], B, L_max, w, wq, device=dev, tiles_per_chunk=args.tpc)
dec.fill_synthetic(ctx)
xs = [torch.randn(n_layers, B, shape.hidden_dim, device=dev).to(torch.bfloat16) for _ in range(2)]
dec.step(xs[0])
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
dec.step(xs[1])
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done", cfg["variant"], n_layers, "layers")
