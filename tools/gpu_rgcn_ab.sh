#!/bin/bash
# RGCN/BSR: tensor-core GPU tests with the in-tree library and every ab/*/ variant, then A/B timing.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
for v in ab/*/; do
  [ -d "$v" ] || continue
  STRATA_B200_LIB=$v/libstrata_b200.so timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "golden or random" >> gpurun_out/pytest_tc.log 2>&1; echo "$v rc=$?" >> gpurun_out/pytest_tc.log
done
bash tools/gpu_ab_rgcn.sh
