#!/usr/bin/env bash
# Profiles committed under profiles/ (run on the GPU box via gpurun):
#  1. launch list of the bench command's timed region (NVTX range "bench_timed": per-launch
#     device time, cold, serialised)
#  2. ncu --set full of the dominant kernel (one 3-bit layer launch of the C2 step)
set -u
OUT=${1:-gpurun_out}
CFG=${2:-c2}
mkdir -p "$OUT"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "bench_timed/" \
  --log-file "$OUT/launches_bench_$CFG.csv" \
  python bench.py --config "$CFG" --steps 2 --warmup 1 --no-fp16 --no-cpu-baseline > "$OUT/launches_bench_$CFG.log" 2>&1
tail -c 300 "$OUT/launches_bench_$CFG.log"
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" \
  -k regex:k_decode_a -s 3 -c 1 -o "$OUT/decode_full_$CFG" \
  python tools/prof_step.py --config "$CFG" --layers 4 > "$OUT/decode_full_$CFG.log" 2>&1
tail -2 "$OUT/decode_full_$CFG.log"
