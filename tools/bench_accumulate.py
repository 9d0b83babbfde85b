"""Time `xq_cl_accumulate` alone at the C3 shape (B=16, 32K, d=4096, 2-bit, G=128).

    python tools/bench_accumulate.py [--bits 2] [--fp32]

Prints the kernel's CUDA-event time and its algorithmic HBM rate: per element, the
accumulator in and out (2+2 B for fp16 storage, 4+4+2 B for fp32 + the fp16 copy),
bits/8 B of codes and 4/G B of (scale, zp).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_10395_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=2)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--G", type=int, default=128)
ap.add_argument("--fp32", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
B, L, d, bits, G = args.batch, args.ctx, args.d, args.bits, args.G
row_bytes = -(-d * bits // 64) * 8
codes = torch.randint(0, 255, (B * L, row_bytes), dtype=torch.uint8, device=dev)
params = (torch.rand(B * L, d // G, 2, device=dev) * 0.01).to(torch.float16)
lens = torch.full((B,), L, dtype=torch.int32, device=dev)
x16 = torch.zeros(B * L, d, dtype=torch.float16, device=dev)
acc = torch.zeros(B * L, d, dtype=torch.float32, device=dev) if args.fp32 else None
s = torch.cuda.current_stream().cuda_stream


def run():
    N.call("xq_cl_accumulate", 0, N.ptr(codes), row_bytes, N.ptr(params), bits, G, d, N.ptr(lens), B, L, L,
           N.ptr(acc), N.ptr(x16), s)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
per_elem = (10.0 if args.fp32 else 4.0) + bits / 8 + 4.0 / G
gb = B * L * d * per_elem / 1e9
print(f"xq_cl_accumulate B={B} L={L} d={d} bits={bits} {'fp32' if args.fp32 else 'fp16'}: "
      f"{ms:.3f} ms, {gb:.2f} GB algorithmic, {gb / ms:.2f} TB/s")
