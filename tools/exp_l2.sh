M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for cfg in "1 4" "0 4" "2 4" "1 1" "0 1" "1 16"; do
  set -- $cfg
  XQ_W_HINT=$1 timeout 300 ncu --metrics $M --clock-control none --nvtx --nvtx-include "step/" -k regex:k_decode_attend -s 3 -c 1 --csv python tools/prof_step.py --layers 4 --tpc $2 2>/dev/null | grep -E '"(dram|lts|gpu__time|sm__pipe)' | awk -F'","' -v h=$1 -v t=$2 '{print "hint="h" tpc="t" "$(NF-2)" "$(NF-1)" "$NF}'
done
