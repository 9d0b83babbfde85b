#!/usr/bin/env bash
# A/B timing of library variants on one box (tools/build_variant.sh): prints the fused
# kernel's per-launch time and SM clock for each (variant, config).
#   bash tools/exp_ab.sh "c4 c2" "'' noconv noscore ''"
set -u
CFGS=$1; shift
for v in "$@"; do
  for c in $CFGS; do
    lib=paper_2508_10395_b200/libxquant${v:+_$v}.so
    XQ_LIB=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fp16 \
      --no-prefill 2>/dev/null | python -c "import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
r=d['roofline']; print('${v:-default}', '$c', round(d['value'],2), 'launch_us', round(r['launch_us']), 'frac', round(r['frac'],3), 'MHz', d['clocks']['sm_mhz'], 'cyc_M', round(r['launch_us']*d['clocks']['sm_mhz']/1e6, 3))"
  done
done
