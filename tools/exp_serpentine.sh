set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/serp_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/serp_tests.log; tail -2 gpurun_out/serp_tests.log
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for lib in fwd main; do
  if [ $lib = fwd ]; then export XQ_LIB=$PWD/paper_2508_10395_b200/libxquant_fwd.so; else unset XQ_LIB; fi
  timeout 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "step/" -k regex:k_decode_absorbed -s 3 -c 2 --csv python tools/prof_step.py --config c3 --layers 5 > gpurun_out/serp_ncu_$lib.csv 2>/dev/null
  grep -E '"(dram|lts|gpu__time|gpc|sm__pipe)' gpurun_out/serp_ncu_$lib.csv | awk -F'","' -v l=$lib '{print l" "$(NF-2)" "$(NF-1)" "$NF}'
done
for lib in fwd main fwd main; do
  if [ $lib = fwd ]; then export XQ_LIB=$PWD/paper_2508_10395_b200/libxquant_fwd.so; else unset XQ_LIB; fi
  python bench.py --config c3 --no-cpu-baseline --steps 5 > gpurun_out/serp_bench_$lib.log 2>&1
  tail -1 gpurun_out/serp_bench_$lib.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
done
