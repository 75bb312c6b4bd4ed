mkdir -p gpurun_out
: > gpurun_out/ab7.jsonl
for v in default ab/epi32 default ab/epi32; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  python tools/ab_spmm.py >> gpurun_out/ab7.jsonl 2>/dev/null
done
export STRATA_B200_LIB=ab/epi32/libstrata_b200.so
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gnn_layer.py -q 2>&1 | tail -1
unset STRATA_B200_LIB
timeout 900 python -m pytest tests/test_gpu_cpp.py -q 2>&1 | tail -3
cat gpurun_out/ab7.jsonl
