"""A/B timing of the fused attention step at C2 (STRATA_B200_LIB=... for variants)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2207_04606_b200 as S  # noqa: E402
from ab_spmm import timeit  # noqa: E402

dev = torch.device("cuda:0")
m = S.generate_matrix("powerlaw", 232965, 232965, 0, 0, 0, 567.5267, 1)
plan = S.AttentionPlan(m.to_device(dev))
Q = torch.randn(m.rows, 64, device=dev) * 0.1
K = torch.randn(m.cols, 64, device=dev) * 0.1
V = torch.randn(m.cols, 64, device=dev)
Z = torch.empty((m.rows, 64), device=dev)
print(json.dumps({"lib": os.environ.get("STRATA_B200_LIB", "default"),
                  "attn_ms": round(timeit(lambda: plan(Q, K, V, Z), 5), 3)}))
