"""Time device decompose_hyb (C5 / C2 / C4 shapes), csr_to_bsr (C3) and the RGMS plan (C4):
wall clock around the call with the CSR already resident, first (cold) and second call."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402

dev = torch.device("cuda:0")
out = {}


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for name, n, avg in [("C5", 2449029, 25.3), ("C2", 232965, 567.5267)]:
    m = S.generate_matrix("powerlaw", n, n, 0, 0, 0, avg, 1)
    dm = m.to_device(dev)
    k = S.hyb_auto_k(m)
    h1, t1 = wall(lambda: S.decompose_hyb(dm, 1, k))
    h2, t2 = wall(lambda: S.decompose_hyb(dm, 1, k))  # second handle alive beside the first
    del h1, h2
    torch.cuda.synchronize()
    h3, t3 = wall(lambda: S.decompose_hyb(dm, 1, k))  # rebuilt after release: pooled memory
    out[name + "_decompose_ms"] = [round(t1, 1), round(t2, 1), round(t3, 1)]
    del h3
m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
dm = m.to_device(dev)
_, t1 = wall(lambda: S.csr_to_bsr(dm, 32))
_, t2 = wall(lambda: S.csr_to_bsr(dm, 32))
out["C3_csr_to_bsr_ms"] = [round(t1, 2), round(t2, 2)]
g = S.generate_matrix("powerlaw", 1885136, 1885136, 0, 0, 0, 3.0051, 1)
rel = S.split_relations(g, 133, 1).to_device(dev)
_, t1 = wall(lambda: S.RgmsPlan(rel))
_, t2 = wall(lambda: S.RgmsPlan(rel))
out["C4_rgms_plan_ms"] = [round(t1, 1), round(t2, 1)]
print(json.dumps(out))

# device build_csr (COO -> CSR) at the C5 shape, triplets shuffled
import numpy as np  # noqa: E402
m = S.generate_matrix("powerlaw", 2449029, 2449029, 0, 0, 0, 25.3, 1)
rows = np.repeat(np.arange(m.rows, dtype=np.int32), np.diff(m.indptr))
perm = np.random.default_rng(0).permutation(m.nnz)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
r, c, v = t(rows[perm]), t(m.indices[perm]), t(m.values[perm])
_, t1 = wall(lambda: S.build_csr_device(m.rows, m.cols, r, c, v))
_, t2 = wall(lambda: S.build_csr_device(m.rows, m.cols, r, c, v))
print(json.dumps({"C5_build_csr_device_ms": [round(t1, 1), round(t2, 1)]}))
