mkdir -p gpurun_out
: > gpurun_out/ab5.jsonl
for v in default ab/nopad default ab/nopad; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  python tools/ab_rgcn.py >> gpurun_out/ab5.jsonl 2>/dev/null
done
unset STRATA_B200_LIB
timeout 900 python -m pytest tests/test_gpu_tc.py -q -k "rgms" 2>&1 | tail -1
cat gpurun_out/ab5.jsonl
