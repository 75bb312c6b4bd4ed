"""Development: real-valued SDDMM error vs the F64 pipeline over seeds (tests' parity metric)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402
from oracle import port  # noqa: E402

cuda = torch.device("cuda:0")
m = S.generate_matrix("powerlaw", 3000, 3000, 0, 0, 0, 2.0, 9)
dm = m.to_device(cuda)


def err(a, b):
    return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1)).max())


for seed in range(8):
    torch.manual_seed(seed)
    X = torch.randn(m.rows, 64, device=cuda)
    Yd = torch.randn(64, m.cols, device=cuda)
    got = S.sddmm(dm, X, Yd).cpu().numpy()
    x, yd = X.cpu().numpy(), Yd.cpu().numpy()
    want = port.sddmm_csr_f64(m.rows, m.cols, m.indptr, m.indices, m.values, x, yd)
    ref32 = port.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values, x, yd)
    print(os.environ.get("STRATA_B200_LIB", "default"), seed, "ours", err(got, want), "ref32", err(ref32, want))
