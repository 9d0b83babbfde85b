"""Host-side cost of one decode step (the launch-bound small configurations, e.g. C1):
wall time per step with the GPU queue kept full vs the device time, then the Python
profile of the same steps.

    python tools/prof_host.py --config c1 [--variant fp16] [--steps 300]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_10395_b200 import decode as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--variant", default=None)
ap.add_argument("--steps", type=int, default=300)
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
variant = a.variant or cfg["variant"]
dev = torch.device("cuda", 0)
shape = D.SHAPES[cfg["shape"]]
n_layers = cfg.get("layers", shape.n_layers)
B, ctx = cfg["batch"], cfg["ctx"]
L_max = -(-(ctx + 3 * a.steps + 16) // 128) * 128
w, wq = D.synthetic_weights(shape, variant, dev, layers=n_layers)
dec = D.Decoder(shape, variant, cfg["bits"], B, L_max, w, wq, device=dev)
dec.fill_synthetic(ctx)
x = torch.randn(n_layers, B, shape.hidden_dim, device=dev).to(torch.bfloat16)
for _ in range(10):
    dec.step(x)
torch.cuda.synchronize()

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(a.steps):
    dec.step(x)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / a.steps * 1e6
dev_us = e0.elapsed_time(e1) / a.steps * 1e3
# device time with the host out of the way: one step at a time, synchronised, events
# around the step only
evs = []
for _ in range(50):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record()
    dec.step(x)
    s1.record()
    evs.append((s0, s1))
torch.cuda.synchronize()
print(f"{a.config} {variant}: wall {wall:.1f} us/step, device span {dev_us:.1f} us/step, "
      f"isolated step {sum(p.elapsed_time(q) for p, q in evs) / len(evs) * 1e3:.1f} us (incl. host issue)")

pr = cProfile.Profile()
pr.enable()
for _ in range(a.steps):
    dec.step(x)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(25)
