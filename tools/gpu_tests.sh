#!/bin/bash
# Selected GPU tests: TESTS="tests/test_gpu_mtx.py ..." (default: the whole -m gpu suite).
mkdir -p gpurun_out
timeout ${TMO:-1500} python -m pytest ${TESTS:-tests} -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
tail -30 gpurun_out/pytest_sel.log
