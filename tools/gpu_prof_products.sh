#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_hyb_kernel -s 2 -c 1 \
  -o gpurun_out/prof_products_new -f python tools/prof_workloads.py products 3 > gpurun_out/ncu_pn.log 2>&1
STRATA_B200_LIB=ab/mb2/libstrata_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_hyb_kernel -s 2 -c 1 \
  -o gpurun_out/prof_products_mb2 -f python tools/prof_workloads.py products 3 > gpurun_out/ncu_pm.log 2>&1
