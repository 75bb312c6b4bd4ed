#!/bin/bash
# Full GPU suite (no -x: every failure listed), then A/B timing of the in-tree library vs ab/*/.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_ab_only.sh
