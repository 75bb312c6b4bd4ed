REF=1 bash tools/gpu_round.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_bench.log 2>&1
WORKLOADS="reddit_spmm" bash tools/gpu_prof.sh > /dev/null 2>&1
SAN_ONLY="hyb sddmm" bash tools/gpu_sanitize.sh > /dev/null 2>&1
ls gpurun_out
