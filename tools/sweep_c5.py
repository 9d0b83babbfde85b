"""C5: long-context sweep, Llama-2-13B shape, XQuant-CL 3-bit vs fp16 KV decode.

BASELINE.json config 5 is 8K-128K context at batch 1-64 on 8 B200s. The deployment
is batch-sharded (sequences are independent, no collective in the decode loop), so
each GPU runs the same per-GPU shard; this sweep measures those shards on one B200
(bench.py --config c5 --ctx C --batch B) and reports whole-job numbers for 8 GPUs as
8x the shard (weak scaling, no communication to add).

    python tools/sweep_c5.py [--out profiles/r01_c5_sweep]      # on the GPU box
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
POINTS = [(8192, 1), (8192, 8), (32768, 1), (32768, 8), (131072, 1), (131072, 8)]


def run(ctx, batch, steps):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5", "--ctx", str(ctx),
           "--batch", str(batch), "--steps", str(steps), "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    for line in reversed(r.stdout.splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise RuntimeError(r.stderr[-2000:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_c5_sweep"))
    args = ap.parse_args()
    rows = []
    for ctx, b in POINTS:
        steps = 3 if ctx * b >= 131072 * 8 else 5
        d = run(ctx, b, steps)
        f = d.get("fp16_kv") or {}
        row = {"ctx": ctx, "batch_per_gpu": b, "batch_8gpu": 8 * b,
               "xq_tok_s_gpu": d["value"], "xq_e2e_tok_s_gpu": d["e2e"]["value"],
               "xq_ms_step": d["ms_per_step"], "kernel_frac": d["roofline"]["frac"],
               "fp16_tok_s_gpu": f.get("value"), "fp16_note": f.get("note"),
               "xq_arena_gb": d["compression"]["arena_bytes_measured"] / 1e9,
               "fp16_kv_gb_same_capacity": d["compression"]["fp16_kv_bytes_same_capacity"] / 1e9,
               "compression": d["compression"]["factor"], "clocks": d["clocks"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
    with open(args.out + ".json", "w") as fh:
        json.dump(rows, fh, indent=1)
    lines = ["# C5 sweep: Llama-2-13B shape, XQuant-CL 3-bit (layers 0-2 4-bit) vs fp16 KV, one B200 shard",
             "# whole-job 8-GPU tokens/s = 8 x the per-GPU value (batch-sharded, no collective)",
             "| ctx | batch/GPU (8-GPU batch) | XQuant-CL tok/s/GPU | e2e | fp16-KV tok/s/GPU | kernel frac | XQ arena GB | fp16 KV GB |",
             "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        f16 = f"{r['fp16_tok_s_gpu']:.1f}" if r["fp16_tok_s_gpu"] else "does not fit"
        lines.append(f"| {r['ctx'] // 1024}K | {r['batch_per_gpu']} ({r['batch_8gpu']}) | "
                     f"{r['xq_tok_s_gpu']:.2f} | {r['xq_e2e_tok_s_gpu']:.2f} | {f16} | "
                     f"{r['kernel_frac']:.2f} | {r['xq_arena_gb']:.1f} | {r['fp16_kv_gb_same_capacity']:.1f} |")
    with open(args.out + ".md", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
