"""A/B of two library builds on the kvq decode kernel: the same seeded caches (ragged
lengths, a few decode steps so residual rows are live) attended by XQ_LIB's build;
saves the outputs and prints the per-launch time.

    XQ_LIB=paper_2508_10395_b200/libxquant_old.so python tools/kvq_ab.py --tag old
    python tools/kvq_ab.py --tag new --against old
"""
import argparse
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_10395_b200 import cache as M  # noqa: E402

CASES = [  # (bits, kv_group, d, n_heads, lens)
    (3, 1, 4096, 32, [8000, 5003]),
    (4, 1, 4096, 32, [8000, 777]),
    (3, 4, 4096, 32, [8000, 5003]),
    (2, 4, 4096, 32, [4099, 300]),
    (8, 2, 2048, 16, [2000, 129]),
]


def run(bits, g, d, H, lens, seed=0, reps=20):
    kvw = d // g
    gen = torch.Generator().manual_seed(seed + 10 * bits + g)
    L = (max(lens) + 8 + 127) // 128 * 128
    st = M.make_cache("kvq", 0, M.LayerPolicy.uniform(bits, 1), 128, 128, n_slots=len(lens),
                      max_len=L, hidden_dim=d, n_heads=H, kv_group=g)
    w = M.LayerWeights(w_k=(torch.randn(d, kvw, generator=gen) / math.sqrt(d)).to(torch.bfloat16).cuda(),
                       w_v=(torch.randn(d, kvw, generator=gen) / math.sqrt(d)).to(torch.bfloat16).cuda())
    for s, n in enumerate(lens):
        st.prefill(torch.randn(n, d, generator=gen).to(torch.bfloat16).cuda(), w, slot=s)
    for _ in range(5):
        st.decode_append(torch.randn(len(lens), d, generator=gen).to(torch.bfloat16).cuda(), w)
    q = torch.randn(len(lens), H, 128, generator=gen).cuda()
    out = st.decode_attend(q, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        st.decode_attend(q, w)
    e1.record()
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), e0.elapsed_time(e1) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--against")
    a = ap.parse_args()
    os.makedirs("gpurun_out", exist_ok=True)
    for i, (bits, g, d, H, lens) in enumerate(CASES):
        out, us = run(bits, g, d, H, lens)
        np.save(f"gpurun_out/kvq_ab_{a.tag}_{i}.npy", out)
        line = f"{a.tag} bits={bits} g={g} d={d} lens={lens} attend_us={us:.1f}"
        if a.against:
            ref = np.load(f"gpurun_out/kvq_ab_{a.against}_{i}.npy")
            rel = float(np.abs(out - ref).max() / np.abs(ref).max())
            line += f" max_rel_vs_{a.against}={rel:.2e}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
