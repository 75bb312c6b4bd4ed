for pool in 0 1; do STRATA_HYB_POOL=$pool timeout 600 python tools/time_decompose.py > gpurun_out/time_decompose_$pool.json 2>&1; echo pool=$pool; cat gpurun_out/time_decompose_$pool.json; done
SAN_ONLY="hyb bsr" bash tools/gpu_sanitize.sh
