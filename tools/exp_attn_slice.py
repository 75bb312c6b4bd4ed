"""Experiment: fused attention time per edge when the gathered K/V columns span half the
graph (L2 working set halved) vs the whole C2 graph."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2207_04606_b200 as S  # noqa: E402
from ab_spmm import timeit  # noqa: E402

dev = torch.device("cuda:0")
m = S.generate_matrix("powerlaw", 232965, 232965, 0, 0, 0, 567.5267, 1)
Q = torch.randn(m.rows, 64, device=dev) * 0.1
K = torch.randn(m.cols, 64, device=dev) * 0.1
V = torch.randn(m.cols, 64, device=dev)
Z = torch.empty((m.rows, 64), device=dev)
plan = S.AttentionPlan(m.to_device(dev))
full = timeit(lambda: plan(Q, K, V, Z), 5)
out = {"full_ms": round(full, 3), "nnz": m.nnz}
rows = np.repeat(np.arange(m.rows), np.diff(m.indptr))
for parts in (2, 3):
    ms = []
    for p in range(parts):
        lo, hi = m.cols * p // parts, m.cols * (p + 1) // parts
        keep = (m.indices >= lo) & (m.indices < hi)
        ip = np.zeros(m.rows + 1, np.int64)
        np.add.at(ip, rows[keep] + 1, 1)
        ip = np.cumsum(ip).astype(np.int32)
        sub = S.CsrMatrix(m.rows, m.cols, ip, m.indices[keep].copy(), m.values[keep].copy())
        pl = S.AttentionPlan(sub.to_device(dev))
        ms.append(timeit(lambda: pl(Q, K, V, Z), 5))
        del pl
    out[f"slices{parts}_ms"] = [round(x, 3) for x in ms]
    out[f"slices{parts}_sum_ms"] = round(sum(ms), 3)
print(out)
