mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/pytest_att.log 2>&1; echo rc=$? >> gpurun_out/pytest_att.log
for i in 1 2; do python tools/ab_attention.py; for v in ab/*/; do STRATA_B200_LIB=$v/libstrata_b200.so python tools/ab_attention.py; done; done > gpurun_out/ab_att.jsonl 2>&1
