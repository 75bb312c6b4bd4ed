mkdir -p gpurun_out
: > gpurun_out/ab4.jsonl
for v in default ab/y64; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  python tools/ab_spmm.py >> gpurun_out/ab4.jsonl 2>/dev/null
  timeout 900 python -m pytest tests/test_gpu_sddmm.py tests/test_gpu_c2.py tests/test_gpu_shard.py -q 2>&1 | tail -1 | sed "s|^|$v: |" >> gpurun_out/ab4_tests.log
done
cat gpurun_out/ab4.jsonl gpurun_out/ab4_tests.log
