#!/usr/bin/env bash
# Profiles committed under profiles/ (run on the GPU box via gpurun):
#  1. launch list of the bench command itself (per-launch device time, cold, serialised)
#  2. ncu --set full of the dominant kernel (one 3-bit layer launch of the C2 step)
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches_bench.csv" \
  python bench.py --steps 2 --warmup 1 --no-fp16 --no-cpu-baseline > "$OUT/launches_bench.log" 2>&1
tail -c 300 "$OUT/launches_bench.log"
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" \
  -k regex:k_decode_attend -s 3 -c 1 -o "$OUT/decode_full" \
  python tools/prof_step.py --layers 4 > "$OUT/decode_full.log" 2>&1
tail -2 "$OUT/decode_full.log"
