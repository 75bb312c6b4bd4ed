#!/bin/bash
# A/B timing of RGCN/BSR library variants under ab/*/ (tools/ab_rgcn.py).
mkdir -p gpurun_out
python tools/ab_rgcn.py > gpurun_out/ab_rgcn.jsonl 2>/dev/null
for v in ab/*/; do [ -d "$v" ] || continue; STRATA_B200_LIB=$v/libstrata_b200.so python tools/ab_rgcn.py >> gpurun_out/ab_rgcn.jsonl 2>/dev/null; done
