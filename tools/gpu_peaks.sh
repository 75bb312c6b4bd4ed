#!/bin/bash
# Measured L2 read bandwidth and pinned host<->device copy rates (tools/peaks.cu) -> profiles/peaks.json
# Run on the GPU box: gpurun -- bash tools/gpu_peaks.sh ; then copy gpurun_out/peaks.json to profiles/.
set -e
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/strata_peaks tools/peaks.cu
/tmp/strata_peaks | tee gpurun_out/peaks.json
