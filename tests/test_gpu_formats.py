"""GPU: DBSR and SR-BCRS (storage.cpp:336-440) — device conversions bit-exact against the
reference library's arrays (golden.npz, made by tests/golden/make_golden.py), and their tcgen05
SpMM bitwise equal to the reference pipeline ("dbsr:b=32", "srbcrs:t=8,g=32") on integer
operands, plus larger cases against the oracle and real-valued tolerance."""
import os

import numpy as np
import pytest
import torch

import paper_2207_04606_b200 as S
from oracle import port

from test_gpu_hyb import close_ref_metric

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")
NAMES = ("example", "bs128", "pl")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def _csr(G, name):
    meta = G[f"fmt/{name}/csr"]
    rows, cols = int(meta[0]), int(meta[1])
    return S.CsrMatrix(rows, cols, meta[2:].astype(np.int32), G[f"fmt/{name}/indices"],
                       G[f"fmt/{name}/values"])


def bf16(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(torch.bfloat16)


@pytest.mark.parametrize("name", NAMES)
def test_dbsr_arrays_golden(cuda, G, name):
    m = _csr(G, name)
    for b in (2, 32):
        key = f"dbsr/{name}_b{b}"
        db = S.csr_to_dbsr(m.to_device(cuda), b)
        a = db.arrays("")
        assert np.array_equal(a["IO_indices"], G[key + "/IO_indices"]), key
        assert np.array_equal(a["JO_indptr"], G[key + "/JO_indptr"]), key
        assert np.array_equal(a["JO_indices"], G[key + "/JO_indices"]), key
        assert np.array_equal(a["values"], G[key + "/values"]), key
        rows, cols, pad = (int(x) for x in G[key + "/shape"])
        assert (db.mb * b, db.nb * b, db.pad_slots) == (rows, cols, pad)


@pytest.mark.parametrize("name", NAMES)
def test_srbcrs_arrays_golden(cuda, G, name):
    m = _csr(G, name)
    for t, g in ((2, 2), (3, 5), (8, 32)):
        key = f"srbcrs/{name}_t{t}_g{g}"
        sr = S.csr_to_srbcrs(m.to_device(cuda), t, g)
        a = sr.arrays("")
        assert np.array_equal(a["G_indptr"], G[key + "/G_indptr"]), key
        assert np.array_equal(a["JT_indices"], G[key + "/JT_indices"]), key
        assert np.array_equal(a["values"], G[key + "/values"]), key
        rows, cols, pad = (int(x) for x in G[key + "/shape"])
        assert (sr.mb * t, sr.pad_slots) == (rows, pad)


@pytest.mark.parametrize("name", NAMES)
def test_dbsr_srbcrs_spmm_golden(cuda, G, name):
    m = _csr(G, name)
    dm = m.to_device(cuda)
    X = G[f"fmtspmm/{name}/dbsr/X"]
    Y = S.dbsr_spmm(S.csr_to_dbsr(dm, 32), bf16(X, cuda)).cpu().numpy()
    assert np.array_equal(Y, G[f"fmtspmm/{name}/dbsr/Y"])
    X = G[f"fmtspmm/{name}/srbcrs/X"]
    Y = S.srbcrs_spmm(S.csr_to_srbcrs(dm, 8, 32), bf16(X, cuda)).cpu().numpy()
    assert np.array_equal(Y, G[f"fmtspmm/{name}/srbcrs/Y"])


@pytest.mark.parametrize("d", [64, 128, 256, 512])
def test_srbcrs_spmm_feature_sizes(cuda, d):
    """Pruned-weight shape: power-law rows, SR-BCRS(8, 32); integer operands bitwise vs the
    CSR oracle, real-valued within 1e-2 of F64; rows beyond the matrix (t-padding) are zero."""
    m = S.generate_matrix("powerlaw", 5003, 4000, 0, 0, 0, 24.0, 7)
    sr = S.csr_to_srbcrs(m.to_device(cuda), 8, 32)
    X = S.dense_int((m.cols, d), 12)
    Y = S.srbcrs_spmm(sr, bf16(X, cuda)).cpu().numpy()
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    assert Y.shape == (sr.mb * 8, d)
    assert np.array_equal(Y[:m.rows], want) and not Y[m.rows:].any()
    Xr = torch.randn(m.cols, d, device=cuda).to(torch.bfloat16)
    Yr = S.srbcrs_spmm(sr, Xr).cpu().numpy()[:m.rows]
    dense = np.zeros((m.rows, m.cols))
    rows_of = np.repeat(np.arange(m.rows), np.diff(m.indptr))
    dense[rows_of, m.indices] = m.values
    assert close_ref_metric(Yr, dense @ Xr.float().cpu().numpy().astype(np.float64), 1e-2)


def test_dbsr_spmm_sparse_block_rows(cuda):
    """Pruned weights with most block rows empty: DBSR stores only the non-empty ones; the
    SpMM equals BSR's and zero-fills the rest."""
    m = S.generate_matrix("blocksparse", 2048, 1024, 0.02, 0, 32, 0, 9)
    dm = m.to_device(cuda)
    db = S.csr_to_dbsr(dm, 32)
    assert db.nstored < db.mb
    X = bf16(S.dense_int((1024, 128), 13), cuda)
    Yd = S.dbsr_spmm(db, X, torch.full((2048, 128), 7.0, device=cuda))
    Yb = S.bsr_spmm(S.csr_to_bsr(dm, 32), X)
    assert torch.equal(Yd, Yb)
    with pytest.raises(S.StrataError):
        S.srbcrs_spmm(S.csr_to_srbcrs(dm, 4, 32), X)
