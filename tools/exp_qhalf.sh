# A/B of fp16 q in the pipelined (GQA) absorbed kernel epilogue on C4. The XQ_Q_F16 variant measured slower and was
# reverted from csrc; this harness is kept for the record (it needs that patch to build libxquant_qh.so).
set -u
mkdir -p gpurun_out
XQ_LIB=$PWD/paper_2508_10395_b200/libxquant_qh.so python -m pytest tests -m gpu -x -q > gpurun_out/qh_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/qh_tests.log; tail -3 gpurun_out/qh_tests.log
for v in main qh main qh; do
  if [ $v = main ]; then unset XQ_LIB; else export XQ_LIB=$PWD/paper_2508_10395_b200/libxquant_qh.so; fi
  python bench.py --config c4 --no-cpu-baseline --no-fp16 --steps 5 > gpurun_out/qh_bench_$v.log 2>&1
  tail -1 gpurun_out/qh_bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
