"""Small invocations of every mbarrier / TMA / tcgen05 pipeline (and the gather kernels) for
compute-sanitizer (racecheck, synccheck, memcheck): tools/gpu_sanitize.sh runs this script under
each tool and keeps the summaries in profiles/.  Each call is checked against the oracle so a
sanitizer run is also a correctness run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402
from oracle import port  # noqa: E402

dev = torch.device("cuda:0")
only = set(sys.argv[1:])


def want(name):
    return not only or name in only


if want("hyb"):  # spmm_hyb_kernel (cp.async staging) + split-run fix-up, c = 1 and c = 2
    m = S.generate_matrix("powerlaw", 3000, 2800, 0, 0, 0, 12.0, 4)
    for c in (1, 2):
        h = S.decompose_hyb(m.to_device(dev), c, 2)
        X = torch.from_numpy(S.dense_int((m.cols, 32), 1)).to(dev)
        Y = S.spmm(h, X).cpu().numpy()
        assert np.array_equal(Y, port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.cpu().numpy()))
    print("hyb ok")

if want("sddmm"):
    m = S.generate_matrix("powerlaw", 2000, 2100, 0, 0, 0, 10.0, 5)
    for d in (32, 64, 128):  # 4-, 8- and 16-lane 256-bit variants
        Xs = torch.from_numpy(S.dense_int((m.rows, d), 2)).to(dev)
        Yd = torch.from_numpy(S.dense_int((d, m.cols), 3)).to(dev)
        B = S.sddmm(m.to_device(dev), Xs, Yd).cpu().numpy()
        assert np.array_equal(B, port.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values,
                                                       Xs.cpu().numpy(), Yd.cpu().numpy()))
    print("sddmm ok")

if want("bsr"):  # tcgen05 + TMA BSR SpMM (PDL launch) and the block-sparse SDDMM
    mb = S.generate_matrix("blocksparse", 512, 512, 0.15, 0, 32, 0, 1)
    bs = S.csr_to_bsr(mb.to_device(dev), 32)
    jp, ji, bv = port.csr_to_bsr(mb.rows, mb.cols, mb.indptr, mb.indices, mb.values, 32)
    Xb = S.dense_int((512, 64), 4)
    Yb = S.bsr_spmm(bs, torch.from_numpy(Xb).to(dev).to(torch.bfloat16)).cpu().numpy()
    assert np.array_equal(Yb, port.bsr_spmm_refnum(16, 32, jp, ji, bv, Xb))
    Q = torch.from_numpy(S.dense_int((512, 64), 5)).to(dev).to(torch.bfloat16)
    K = torch.from_numpy(S.dense_int((512, 64), 6)).to(dev).to(torch.bfloat16)
    S.bsr_sddmm(bs, Q, K)
    torch.cuda.synchronize()
    print("bsr ok")

if want("srbcrs"):  # tcgen05 + TMA gather4
    m = S.generate_matrix("powerlaw", 512, 512, 0, 0, 0, 16.0, 2)
    sr = S.csr_to_srbcrs(m.to_device(dev), 8, 32)
    X = S.dense_int((512, 64), 7)
    Y = S.srbcrs_spmm(sr, torch.from_numpy(X).to(dev).to(torch.bfloat16)).cpu().numpy()
    assert np.array_equal(Y, port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X))
    print("srbcrs ok")

if want("rgms"):  # warp-specialised tcgen05 pass 1 + row sums
    rel = S.split_relations(S.generate_matrix("powerlaw", 3000, 3000, 0, 0, 0, 3.0, 2), 5, 1)
    Xr = S.dense_int((rel.cols, 32), 5)
    Wr = S.dense_int((5, 32, 32), 6)
    Yr = S.RgmsPlan(rel.to_device(dev)).run(torch.from_numpy(Xr).to(dev).to(torch.bfloat16),
                                            torch.from_numpy(Wr).to(dev).to(torch.bfloat16))
    torch.cuda.synchronize()
    print("rgms ok", float(Yr.abs().sum()))

if want("gemm"):  # tcgen05 kind::tf32 3xTF32 GEMM of the GNN layer
    Y = torch.from_numpy(S.dense_int((600, 128), 8)).to(dev)
    W = torch.from_numpy(S.dense_int((128, 64), 9)).to(dev)
    Z = S.gemm(Y, W)
    assert torch.equal(Z.double(), Y.double() @ W.double())
    print("gemm ok")

if want("attention"):
    m = S.generate_matrix("powerlaw", 1500, 1500, 0, 0, 0, 20.0, 3)
    dm = m.to_device(dev)
    plan = S.AttentionPlan(dm)
    Q, K, V = (torch.randn(1500, 64, device=dev) * 0.1 for _ in range(3))
    plan(Q, K, V)
    torch.cuda.synchronize()
    print("attention ok")

if want("mtx"):
    text = b"%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n1 1 2.5\n2 1 -1e-310\n4 2 3e-3\n3 3 7\n"
    mm = S.read_matrix_market(text)
    assert mm.ntriplets == 6
    print("mtx ok")
