#!/bin/bash
mkdir -p gpurun_out
cd tools
python ab_rgcn.py > ../gpurun_out/ab_tc.jsonl 2>&1
for v in ../ab/*/; do STRATA_B200_LIB=$v/libstrata_b200.so python ab_rgcn.py >> ../gpurun_out/ab_tc.jsonl 2>&1; done
