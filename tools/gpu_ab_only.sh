#!/bin/bash
# A/B timing only: the in-tree library and every ab/*/ variant (tools/ab_spmm.py).
mkdir -p gpurun_out
python tools/ab_spmm.py > gpurun_out/ab.jsonl 2>&1
for v in ab/*/; do STRATA_B200_LIB=$v/libstrata_b200.so python tools/ab_spmm.py >> gpurun_out/ab.jsonl 2>&1; done
