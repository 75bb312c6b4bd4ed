"""Time the C3 BSR and C4 RGCN calls (CUDA events).  STRATA_B200_LIB=... for A/B builds."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402
from ab_spmm import timeit  # noqa: E402

dev = torch.device("cuda:0")
g = S.generate_matrix("powerlaw", 1885136, 1885136, 0, 0, 0, 3.0051, 1)
rel = S.split_relations(g, 133, 1).to_device(dev)
plan = S.RgmsPlan(rel)
X = torch.randint(-3, 4, (g.cols, 32), device=dev).to(torch.bfloat16)
W = torch.randint(-3, 4, (133, 32, 32), device=dev).to(torch.bfloat16)
Y = torch.empty((g.rows, 32), device=dev)
out = {"lib": os.environ.get("STRATA_B200_LIB", "default"),
       "rgcn_ms": round(timeit(lambda: plan.run(X, W, Y)), 4),
       "rgcn_oneshot_ms": round(timeit(lambda: S.rgms(rel, X, W, Y), 3), 4)}
m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
bs = S.csr_to_bsr(m.to_device(dev), 32)
Xb = torch.randint(-3, 4, (4096, 64), device=dev).to(torch.bfloat16)
Yb = torch.empty((4096, 64), device=dev)
out["bsr_us"] = round(timeit(lambda: S.bsr_spmm(bs, Xb, Yb), 50) * 1e3, 2)
print(json.dumps(out))
