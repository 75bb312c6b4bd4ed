#!/bin/bash
# ncu captures (one kernel each) for the workloads in tools/prof_workloads.py.
# usage: WORKLOADS="reddit_spmm bsr" bash tools/gpu_prof.sh
mkdir -p gpurun_out
for w in ${WORKLOADS:-products reddit_spmm reddit_sddmm bsr bsr12 rgcn rgcn_sum srbcrs attention}; do
  run=$w
  case $w in
    products|reddit_spmm) k=spmm_hyb_kernel ;;
    reddit_sddmm) k=sddmm_kernel ;;
    bsr|bsr12) k=bsr_spmm_tc_kernel ;;
    rgcn) k=rgms_edge_gemm_kernel ;;
    rgcn_sum) k=rgms_row_sum_kernel; run=rgcn ;;
    srbcrs) k=srbcrs_spmm_tc_kernel ;;
    attention) k=attn_kernel ;;
    bsr12_sddmm) k=bsr_sddmm_tc_kernel ;;
    dbsr) k=bsr_spmm_tc_kernel ;;
    gnn) k=gemm_tf32 ;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$w -f python tools/prof_workloads.py $run 4 > gpurun_out/ncu_$w.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$w.csv python tools/prof_workloads.py $run 3 > /dev/null 2>&1
done
ls -la gpurun_out
