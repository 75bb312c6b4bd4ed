#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize.py (small configs of
# every mbarrier / TMA / tcgen05 pipeline and the gather kernels); summaries to gpurun_out/.
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $SAN_ONLY \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -5 gpurun_out/sanitize_$tool.log
done
