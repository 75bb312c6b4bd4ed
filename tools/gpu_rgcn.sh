#!/bin/bash
# RGCN (C4) round: GPU tests for the tensor-core paths, launch list, full captures of both passes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python tools/ab_rgcn.py > gpurun_out/ab_rgcn.json 2> gpurun_out/ab_rgcn.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_rgcn.csv python tools/prof_workloads.py rgcn 3 > gpurun_out/ncu_l_rgcn.log 2>&1
for k in rgms_edge_gemm_kernel rgms_row_sum_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/prof_$k -f python tools/prof_workloads.py rgcn 2 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
