#!/usr/bin/env bash
# On the GPU box: ncu --set full of one kvq decode launch (prof_step.py), exported to csv.
#   bash tools/kvq_profile.sh c2
mkdir -p gpurun_out/kvqprof2
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:k_kvq_decode -c 1 -o gpurun_out/kvqprof2/kvq python tools/prof_step.py --variant kvq --config ${1:-c2} --layers 4 > gpurun_out/kvqprof2/log.txt 2>&1
ncu -i gpurun_out/kvqprof2/kvq.ncu-rep --page details --csv > gpurun_out/kvqprof2/details.csv
ncu -i gpurun_out/kvqprof2/kvq.ncu-rep --page raw --csv > gpurun_out/kvqprof2/raw.csv
ncu -i gpurun_out/kvqprof2/kvq.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/kvqprof2/src.csv
rm gpurun_out/kvqprof2/kvq.ncu-rep
