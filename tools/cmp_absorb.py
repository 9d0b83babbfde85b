"""Compare the V-absorbed fused decode with the unabsorbed kernel (and timing).

Usage (GPU box): python tools/cmp_absorb.py [--time]
Prints, per case, rel err (max|a-b|/max|b|) of absorbed vs unabsorbed output.
"""

import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_10395_b200 import cache as M  # noqa: E402


def rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def build(variant, bits, d, H, g, n_slots, lens, seed=0):
    dev = torch.device("cuda")
    gen = torch.Generator(device="cpu").manual_seed(seed)
    L = max(lens) + 128
    L = -(-L // 128) * 128
    width = d // g
    pol = M.LayerPolicy.uniform(bits, 1)
    st = M.make_cache(variant, 0, pol, 128, n_slots=n_slots, max_len=L, hidden_dim=d, n_heads=H,
                      kv_group=g, device=dev)
    wk = (torch.randn(d, width, generator=gen) / d ** 0.5).to(torch.bfloat16).to(dev)
    wv = (torch.randn(d, width, generator=gen) / d ** 0.5).to(torch.bfloat16).to(dev)
    if variant == "xq-gqa":
        uk, _ = torch.linalg.qr(torch.randn(d, width, generator=gen, dtype=torch.float64))
        uv, _ = torch.linalg.qr(torch.randn(d, width, generator=gen, dtype=torch.float64))
        fk = (torch.randn(width, width, generator=gen) / width ** 0.5).to(dev)
        fv = (torch.randn(width, width, generator=gen) / width ** 0.5).to(dev)
        w = M.LayerWeights(u_k=uk.float().to(dev), u_v=uv.float().to(dev), fused_k=fk, fused_v=fv)
    else:
        w = M.LayerWeights(w_k=wk, w_v=wv)
    for s, n in enumerate(lens):
        x = torch.randn(n - 1, d, generator=gen).to(torch.bfloat16).to(dev)
        st.prefill(x, w, slot=s) if n > 1 else None
    # decode_append needs every slot to take one token; slots with 1 token start empty
    xt = torch.randn(n_slots, d, generator=gen).to(torch.bfloat16).to(dev)
    if any(n == 1 for n in lens):
        raise SystemExit("lens must be >= 2")
    st.decode_append(xt, w)
    q = torch.randn(n_slots, H, 128, generator=gen).to(dev)
    return st, w, q


def run(st, w, q, absorb, reps=0, acc=None):
    st.absorb = absorb
    out = st.decode_attend(q, w, acc)
    torch.cuda.synchronize()
    ms = None
    if reps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            st.decode_attend(q, w, acc)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    return out, ms


CASES = [
    ("xq-mha", 3, 512, 4, 1, 1, [300]),
    ("xq-mha", 4, 512, 4, 1, 3, [2, 257, 700]),
    ("xq-mha", 2, 1024, 8, 1, 2, [1000, 513]),
    ("xq-mha", 8, 512, 4, 1, 2, [129, 384]),
    ("xq-mha", 3, 4096, 32, 1, 2, [3000, 1200]),
    ("xq-gqa", 3, 1024, 8, 4, 2, [400, 1000]),
    ("xq-gqa", 4, 4096, 32, 4, 2, [2000, 777]),
]


def main():
    timing = "--time" in sys.argv
    worst = 0.0
    for variant, bits, d, H, g, ns, lens in CASES:
        st, w, q = build(variant, bits, d, H, g, ns, lens)
        a, ta = run(st, w, q, True, 5 if timing else 0)
        b, tb = run(st, w, q, False, 5 if timing else 0)
        e = rel(a, b)
        worst = max(worst, e)
        extra = f"  absorbed {ta:.3f} ms  unabsorbed {tb:.3f} ms" if timing else ""
        print(f"{variant:8s} bits={bits} d={d} H={H} g={g} lens={lens}: rel {e:.2e}{extra}", flush=True)
    # CL delta layer (fp16 accumulator rows as A)
    dev = torch.device("cuda")
    d, H, ns, n = 1024, 8, 2, 600
    pol = M.LayerPolicy.uniform(2, 4)
    gen = torch.Generator(device="cpu").manual_seed(3)
    acc = M.Accumulator(ns, 1024, d, device=dev)
    ws = []
    sts = []
    for li in range(4):
        st = M.make_cache("xq-cl-mha", li, pol, 128, n_slots=ns, max_len=1024, hidden_dim=d,
                          n_heads=H, device=dev)
        w = M.LayerWeights(w_k=(torch.randn(d, d, generator=gen) / d ** 0.5).to(torch.bfloat16).to(dev),
                           w_v=(torch.randn(d, d, generator=gen) / d ** 0.5).to(torch.bfloat16).to(dev))
        x = torch.randn(ns, n, d, generator=gen).to(torch.bfloat16).to(dev)
        st.prefill(x, w, acc)
        ws.append(w)
        sts.append(st)
    q = torch.randn(ns, H, 128, generator=gen).to(dev)
    a, _ = run(sts[3], ws[3], q, True, acc=acc)
    b, _ = run(sts[3], ws[3], q, False, acc=acc)
    e = rel(a, b)
    worst = max(worst, e)
    print(f"xq-cl-mha delta layer d={d} n={n}: rel {e:.2e}", flush=True)
    print(f"worst {worst:.2e}")
    assert worst < 2e-2


if __name__ == "__main__":
    main()
