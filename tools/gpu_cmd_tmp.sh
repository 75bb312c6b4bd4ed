for i in 1 2; do
python tools/ab_spmm.py
for v in ab/*/; do STRATA_B200_LIB=$v/libstrata_b200.so python tools/ab_spmm.py; done
done > gpurun_out/ab.jsonl 2>&1
python - <<'P'
import json
for l in open('gpurun_out/ab.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['lib'], d['C5_spmm_ms'], d['C2_spmm_ms'], d['C1_spmm_ms'], d['C2_sddmm_ms'])
P
