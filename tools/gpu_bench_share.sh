#!/bin/bash
# N = 2 bench code path on a one-GPU box (both ranks on cuda:0, gloo group): the p2p mode
# (NCCL refuses two ranks on one device; the nccl reassembly is covered at world 1 by the tests).
mkdir -p gpurun_out
for mode in p2p; do
  STRATA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
    --no-cpu-baseline --no-extra --allgather $mode > gpurun_out/bench_share_$mode.json 2> gpurun_out/bench_share_$mode.err
done
