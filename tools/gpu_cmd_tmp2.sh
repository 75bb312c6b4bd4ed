mkdir -p gpurun_out
bash tools/gpu_ab_attention.sh
tail -2 gpurun_out/pytest_att.log; cat gpurun_out/ab_att.jsonl
