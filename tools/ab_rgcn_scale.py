"""RGCN timing at C4 and at scaled-down AM-shaped graphs (T small enough to stay in L2):
per-edge cost vs graph size, for A/B library builds (STRATA_B200_LIB=...)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402
from ab_spmm import timeit  # noqa: E402

dev = torch.device("cuda:0")
out = {"lib": os.environ.get("STRATA_B200_LIB", "default")}
for div in (1, 4, 8, 16):
    n = 1885136 // div
    g = S.generate_matrix("powerlaw", n, n, 0, 0, 0, 3.0051, 1)
    rel = S.split_relations(g, 133, 1).to_device(dev)
    plan = S.RgmsPlan(rel)
    X = torch.randint(-3, 4, (g.cols, 32), device=dev).to(torch.bfloat16)
    W = torch.randint(-3, 4, (133, 32, 32), device=dev).to(torch.bfloat16)
    Y = torch.empty((g.rows, 32), device=dev)
    ms = timeit(lambda: plan.run(X, W, Y), 20)
    out[f"c4_div{div}"] = {"ms": round(ms, 4), "ns_per_edge": round(ms * 1e6 / g.nnz, 4),
                           "t_mb": round(plan.message_rows * 128 / 1e6, 1)}
print(json.dumps(out))
