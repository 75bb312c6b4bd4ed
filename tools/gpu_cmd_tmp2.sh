python tools/ab_rgcn_scale.py > gpurun_out/ab_rgcn_scale.jsonl 2>&1
STRATA_B200_LIB=ab/tl2/libstrata_b200.so python tools/ab_rgcn_scale.py >> gpurun_out/ab_rgcn_scale.jsonl 2>&1
STRATA_B200_LIB=ab/tl2/libstrata_b200.so timeout 600 python -m pytest tests/test_gpu_tc.py -q -k rgms > gpurun_out/tl2_tests.log 2>&1; tail -3 gpurun_out/tl2_tests.log
cat gpurun_out/ab_rgcn_scale.jsonl
