for i in 1 2; do python tools/ab_attention.py; for v in ab/*/; do STRATA_B200_LIB=$v/libstrata_b200.so python tools/ab_attention.py; done; done
STRATA_B200_LIB=ab/av4/libstrata_b200.so timeout 300 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -n1
