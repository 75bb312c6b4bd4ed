#!/bin/bash
# GEMM / GNN / SpMM / SDDMM parity on the GPU, then A/B timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gnn_layer.py tests/test_gpu_sddmm.py tests/test_gpu_hyb.py -q ${PYTEST_ARGS} > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 600 bash tools/gpu_ab_only.sh
