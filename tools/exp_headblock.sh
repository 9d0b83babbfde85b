M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for hb in 32 16 8 4; do
  XQ_HEAD_BLOCK=$hb timeout 300 ncu --metrics $M --clock-control none --nvtx --nvtx-include "step/" -k regex:k_decode_attend -s 3 -c 1 --csv python tools/prof_step.py --layers 4 2>/dev/null | grep -E '"(dram|lts|gpu__time|sm__pipe)' | awk -F'","' -v h=$hb '{print "hb="h" "$(NF-2)" "$(NF-1)" "$NF}'
  XQ_HEAD_BLOCK=$hb timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fp16 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hb=$hb bench', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
