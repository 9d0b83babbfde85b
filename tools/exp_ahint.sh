# A/B of the fp16-row A-operand L2 hint policy (XQ_A_HINT) on the C3 delta layer
set -u
mkdir -p gpurun_out
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second
for h in 0 1 2; do
  XQ_A_HINT=$h timeout 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "step/" -k regex:k_decode_absorbed -s 3 -c 1 --csv python tools/prof_step.py --config c3 --layers 4 > gpurun_out/ahint_ncu_$h.csv 2>/dev/null
  grep -E '"(dram|lts|gpu__time|gpc)' gpurun_out/ahint_ncu_$h.csv | awk -F'","' -v h=$h '{gsub(/"/,"",$NF); print "hint="h" "$(NF-2)" "$NF}'
done
for h in 0 1 0 1; do
  XQ_A_HINT=$h python bench.py --config c3 --no-cpu-baseline --steps 5 > gpurun_out/ahint_bench_$h.log 2>&1
  tail -1 gpurun_out/ahint_bench_$h.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hint=$h', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
