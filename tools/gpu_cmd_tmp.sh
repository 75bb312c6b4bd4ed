mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for v in default ab/st4 ab/epi ab/st4epi ab/minb5; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  python tools/ab_spmm.py >> gpurun_out/ab.jsonl 2>/dev/null
  python tools/ab_rgcn.py >> gpurun_out/ab.jsonl 2>/dev/null
  timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gnn_layer.py tests/test_gpu_tc.py -q -k "gemm or gnn or rgms" 2>&1 | tail -1 | sed "s|^|$v: |" >> gpurun_out/ab_tests.log
done
cat gpurun_out/ab.jsonl gpurun_out/ab_tests.log
