import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2508_10395_b200 import decode as D
cfg = dict(bench.CONFIGS["c1"])
dev = torch.device("cuda", 0)
shape = D.SHAPES[cfg["shape"]]
n_layers = cfg.get("layers", shape.n_layers)
B, ctx = cfg["batch"], cfg["ctx"]
L_max = -(-(ctx + 300) // 128) * 128
w, wq = D.synthetic_weights(shape, cfg["variant"], dev, layers=n_layers)
dec = D.Decoder(shape, cfg["variant"], cfg["bits"], B, L_max, w, wq, device=dev)
dec.fill_synthetic(ctx)
xs = [torch.randn(n_layers, B, shape.hidden_dim, device=dev).to(torch.bfloat16) for _ in range(4)]
for k in range(20): dec.step(xs[k % 4])
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(100): dec.step(xs[k % 4])
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"CPU issue time per step {1e3*(t1-t0)/100:.3f} ms, wall per step {1e3*(t2-t0)/100:.3f} ms")
pr = cProfile.Profile(); pr.enable()
for k in range(100): dec.step(xs[k % 4])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
