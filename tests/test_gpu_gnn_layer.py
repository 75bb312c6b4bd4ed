"""GPU parity: GNN layer step Z = A @ X @ W (strata_gnn_layer_f32).

Both associations are exercised (d_out < d_in: transform first; d_out >= d_in: aggregate
first).  Integer operands (the reference's A in 1..9, X and W in [-3, 3]) keep every partial
sum exact in f32, so the result must equal the f64 product bitwise; real-valued operands are
held to the north_star's fp32 bar, |x - y| <= 1e-5 * max(|x|, |y|, 1) against f64.
"""
import numpy as np
import pytest

import paper_2207_04606_b200 as S

pytestmark = pytest.mark.gpu
TOL = 1e-5


def dense_f64(m):
    A = np.zeros((m.rows, m.cols))
    for i in range(m.rows):
        A[i, m.indices[m.indptr[i]:m.indptr[i + 1]]] = m.values[m.indptr[i]:m.indptr[i + 1]]
    return A


@pytest.mark.parametrize("d_in,d_out", [(64, 32), (32, 64), (128, 128), (64, 16)])
@pytest.mark.parametrize("c", [1, 2])
def test_gnn_layer_integer_exact(d_in, d_out, c):
    import torch
    dev = torch.device("cuda:0")
    m = S.generate_matrix("powerlaw", 1500, 1300, 0, 0, 0, 12.0, 3)
    h = S.decompose_hyb(m.to_device(dev), c, S.hyb_auto_k(m))
    X = S.dense_int((m.cols, d_in), 11).astype(np.float32)
    W = S.dense_int((d_in, d_out), 12).astype(np.float32)
    Z = S.gnn_layer(h, torch.from_numpy(X).to(dev), torch.from_numpy(W).to(dev)).cpu().numpy()
    want = dense_f64(m) @ X.astype(np.float64) @ W.astype(np.float64)
    assert np.array_equal(Z.astype(np.float64), want)


def test_gnn_layer_real_valued():
    import torch
    dev = torch.device("cuda:0")
    m = S.generate_matrix("powerlaw", 2000, 2000, 0, 0, 0, 20.0, 4)
    rng = np.random.default_rng(5)
    vals = rng.standard_normal(m.nnz).astype(np.float32)
    mr = S.CsrMatrix(m.rows, m.cols, m.indptr, m.indices, vals)
    h = S.decompose_hyb(mr.to_device(dev), 1, S.hyb_auto_k(mr))
    for d_in, d_out in [(128, 32), (32, 128)]:
        X = rng.standard_normal((m.cols, d_in)).astype(np.float32)
        W = (rng.standard_normal((d_in, d_out)) / np.sqrt(d_in)).astype(np.float32)
        Z = S.gnn_layer(h, torch.from_numpy(X).to(dev), torch.from_numpy(W).to(dev)).cpu().numpy()
        want = dense_f64(mr) @ X.astype(np.float64) @ W.astype(np.float64)
        err = np.max(np.abs(Z - want) / np.maximum(np.maximum(np.abs(Z), np.abs(want)), 1.0))
        assert err <= TOL, err


def test_gnn_layer_shape_error():
    import torch
    dev = torch.device("cuda:0")
    m = S.generate_matrix("powerlaw", 100, 100, 0, 0, 0, 4.0, 1)
    h = S.decompose_hyb(m.to_device(dev), 1, S.hyb_auto_k(m))
    with pytest.raises(S.StrataError):
        S.gnn_layer(h, torch.zeros((100, 16), device=dev), torch.zeros((8, 4), device=dev))
