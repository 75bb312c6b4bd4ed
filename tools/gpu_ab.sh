#!/bin/bash
# GPU tests + A/B timing of library variants under ab/*/ + bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/ab_spmm.py > gpurun_out/ab.jsonl 2>&1
for v in ab/*/; do STRATA_B200_LIB=$v/libstrata_b200.so python tools/ab_spmm.py >> gpurun_out/ab.jsonl 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
