#!/bin/bash
# hyb SpMM / SDDMM: GPU parity tests with the in-tree library, then A/B timing vs ab/*/ builds.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hyb.py tests/test_gpu_sddmm.py -x -q > gpurun_out/pytest_hyb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hyb.log
bash tools/gpu_ab_only.sh
