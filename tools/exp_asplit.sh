# Sweep of the evict-first share of each fp16-row A sweep (XQ_A_SPLIT16, in 16ths) on the C3 delta layer
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "cl or accum or absorb" > gpurun_out/asplit_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/asplit_tests.log; tail -2 gpurun_out/asplit_tests.log
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second
for sp in 2 4 6 8 10 12; do
  XQ_A_SPLIT16=$sp timeout 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "step/" -k regex:k_decode_absorbed -s 3 -c 1 --csv python tools/prof_step.py --config c3 --layers 4 > gpurun_out/asplit_ncu_$sp.csv 2>/dev/null
  grep -E '"(dram|lts|gpu__time|gpc)' gpurun_out/asplit_ncu_$sp.csv | awk -F'","' -v h=$sp '{gsub(/"/,"",$NF); print "split="h" "$(NF-2)" "$NF}'
done
