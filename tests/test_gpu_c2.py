"""BASELINE configs[1] at full size: the Reddit-shaped power-law graph (232,965 nodes,
avg degree 567.5267, seed 1 -> 114,615,895 non-zeros, d = 64).

This is the config with fully dense 232,965-non-zero hub rows — 456 bucket-9 segments each, the
deepest split-run / fix-up path of the hyb SpMM — and the only SDDMM at scale.  Everything is
checked against the pinned oracle (oracle/strata_oracle.c) on the reference's own integer
operands, where the reference's F32 results are exact, so equality is bitwise:
  * device decompose_hyb (storage.cpp:271-334) for c = 1 (auto k = 9) and c = 2: every part's
    I / J / value arrays and the padding ratio (bucket rows 98,853 / 71,892 /
    207,044, padding 16.38 %);
  * hyb SpMM d = 64 (kernels.cpp:85-108) for c = 1 and c = 2;
  * SDDMM d = 64 (kernels.cpp:110-136) with Y in the reference's [d][n] layout.
"""
import numpy as np
import pytest

import paper_2207_04606_b200 as S
from oracle import port

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

C2 = dict(kind="powerlaw", n=232965, avg=567.5267, seed=1, d=64)


@pytest.fixture(scope="module")
def reddit():
    m = S.generate_matrix(C2["kind"], C2["n"], C2["n"], 0, 0, 0, C2["avg"], C2["seed"])
    return m


def test_c2_graph_shape(reddit):
    m = reddit
    assert m.nnz == 114615895
    lens = np.diff(m.indptr)
    assert lens.min() == 78 and lens.max() == 232965  # dense hub rows
    assert S.hyb_auto_k(m) == 9


@pytest.mark.parametrize("c", [1, 2])
def test_c2_decompose_bitexact(cuda, reddit, c):
    m = reddit
    k = S.hyb_auto_k(m)
    h = S.decompose_hyb(m.to_device(cuda), c, k)
    parts, pr = port.hyb_decompose(m.rows, m.cols, m.indptr, m.indices, m.values, c, k)
    assert h.padding_ratio == pr
    if c == 1:
        assert [P.nrows for P in h.parts] == [98853, 71892, 207044]  # buckets 7, 8, 9
        assert [P.bucket for P in h.parts] == [7, 8, 9]
        assert abs(pr - 0.1638) < 5e-4
        assert sum(P.nrows * P.width for P in h.parts) == 137064064
    assert len(h.parts) == len(parts)
    for i, R in enumerate(parts):
        P = h.parts[i]
        assert (P.partition, P.bucket, P.nrows, P.nnz, P.col_lo, P.col_hi) == \
            (R["partition"], R["bucket"], R["nrows"], R["nnz"], R["col_lo"], R["col_hi"])
        a = h.part_arrays(i)
        pre = f"hyb_p{P.partition}_b{P.bucket}_"
        assert np.array_equal(a[pre + "I_indices"], R["I_indices"]), i
        assert np.array_equal(a[pre + "J_indices"], R["J_indices"]), i
        assert np.array_equal(a["values"].view(np.uint32), R["values"].view(np.uint32)), i


@pytest.mark.parametrize("c", [1, 2])
def test_c2_hyb_spmm_bitwise(cuda, reddit, c):
    import torch
    m = reddit
    d = C2["d"]
    h = S.decompose_hyb(m.to_device(cuda), c, S.hyb_auto_k(m))
    sched = h.schedule_info()
    if c == 1:
        assert sched["crossing_runs"] > 0  # hub rows split across chunks: the fix-up path runs
    X = S.dense_int((m.cols, d), 7)  # tune.cpp:108-111 operand
    got = S.spmm(h, torch.from_numpy(X).to(cuda)).cpu().numpy()
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    assert np.array_equal(got, want)


def test_c2_sddmm_bitwise(cuda, reddit):
    import torch
    m = reddit
    d = C2["d"]
    X = S.dense_int((m.rows, d), 3)
    Yd = S.dense_int((d, m.cols), 4)  # [d][n], kernels.cpp:122
    got = S.sddmm(m.to_device(cuda), torch.from_numpy(X).to(cuda),
                  torch.from_numpy(Yd).to(cuda)).cpu().numpy()
    want = port.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values, X, Yd)
    assert np.array_equal(got, want)
