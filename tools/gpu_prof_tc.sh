#!/bin/bash
# Launch list + full capture for the tensor-core workloads (RGCN C4, BSR C3).
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_rgcn.csv python tools/prof_workloads.py rgcn 2 > gpurun_out/ncu_l_rgcn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rgms_tc_kernel -s 1 -c 1 \
  -o gpurun_out/prof_rgcn2 -f python tools/prof_workloads.py rgcn 2 > gpurun_out/ncu_rgcn2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bsr_spmm_tc_kernel -s 2 -c 1 \
  -o gpurun_out/prof_bsr2 -f python tools/prof_workloads.py bsr 4 > gpurun_out/ncu_bsr2.log 2>&1
