mkdir -p gpurun_out
: > gpurun_out/ab8.jsonl
for v in default ab2/v64 ab2/v128 default ab2/v64 ab2/v128; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  python tools/ab_spmm.py >> gpurun_out/ab8.jsonl 2>/dev/null
done
for v in default ab2/v64 ab2/v128; do
  if [ "$v" = default ]; then unset STRATA_B200_LIB; else export STRATA_B200_LIB=$v/libstrata_b200.so; fi
  timeout 900 python -m pytest tests/test_gpu_hyb.py tests/test_gpu_peer.py tests/test_gpu_shard.py -q 2>&1 | tail -1 | sed "s|^|$v: |"
done
cat gpurun_out/ab8.jsonl
