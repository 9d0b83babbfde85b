#!/usr/bin/env bash
# On the GPU box, after `XQ_LIB=<old build> python tools/kvq_ab.py --tag old`: the current
# build against it (tools/kvq_ab.py), the kvq GPU tests, and the C2 / C4 kvq bench legs.
python tools/kvq_ab.py --tag new --against old > gpurun_out/kvq_ab2.txt 2>&1
python -m pytest tests/test_gpu_kvq.py tests/test_gpu_compat.py tests/test_gpu_sixteen.py tests/test_gpu_prefill.py -q -x -k kvq 2>&1 | tail -3 >> gpurun_out/kvq_ab2.txt
for c in c2 c4; do python bench.py --config $c --kvq --steps 3 --warmup 3 --no-cpu-baseline --no-fp16 --no-prefill 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith(\"{\")][-1]); k=d[\"kvq\"]; print(\"$c\", round(d[\"value\"],2), \"kvq\", round(k[\"value\"],1), round(k[\"hbm_gbs_achieved\"]), d[\"clocks\"][\"sm_mhz\"])" >> gpurun_out/kvq_ab2.txt; done
cat gpurun_out/kvq_ab2.txt
