mkdir -p gpurun_out
: > gpurun_out/ab3.jsonl
python tools/ab_rgcn.py >> gpurun_out/ab3.jsonl 2>/dev/null
for v in ab/*/; do
  export STRATA_B200_LIB=$v/libstrata_b200.so
  python tools/ab_rgcn.py >> gpurun_out/ab3.jsonl 2>/dev/null
  python tools/ab_rgcn.py >> gpurun_out/ab3.jsonl 2>/dev/null
done
unset STRATA_B200_LIB
python tools/ab_rgcn.py >> gpurun_out/ab3.jsonl 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_tc.py -q -k "rgms" 2>&1 | tail -1
cat gpurun_out/ab3.jsonl
