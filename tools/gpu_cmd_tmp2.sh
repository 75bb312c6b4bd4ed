mkdir -p gpurun_out
: > gpurun_out/ab10.jsonl
for v in default ab/sv2m4 ab/sv2k2 default ab/sv2m4 ab/sv2k2; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  python tools/ab_rgcn.py >> gpurun_out/ab10.jsonl 2>/dev/null
done
for v in ab/sv2m4 ab/sv2k2; do
  export STRATA_B200_LIB=$v/libstrata_b200.so
  timeout 900 python -m pytest tests/test_gpu_tc.py -q -k rgms 2>&1 | tail -1 | sed "s|^|$v: |"
done
cat gpurun_out/ab10.jsonl
