"""GPU parity: CSR SDDMM (kernels.cpp:110-136) through the C ABI against the oracle."""
import os

import numpy as np
import pytest

import paper_2207_04606_b200 as S
from oracle import port

from test_gpu_hyb import close_to_f64, csr_of

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def test_sddmm_golden(cuda, G):
    import torch
    for name in G["cases"]:
        m = csr_of(G, name)
        if m.nnz == 0:
            continue
        dcsr = m.to_device(cuda)
        for d in (8, 32):
            key = f"{name}/sddmm_d{d}"
            B = S.sddmm(dcsr, torch.from_numpy(G[key + "/X"]).to(cuda),
                        torch.from_numpy(G[key + "/Yd"]).to(cuda)).cpu().numpy()
            assert close_to_f64(B, G[key + "/B64"], G[key + "/B"]), key


@pytest.mark.parametrize("d", [32, 64, 128, 16, 7])
def test_sddmm_integer_exact(cuda, d):
    import torch
    m = S.generate_matrix("powerlaw", 5000, 4000, 0, 0, 0, 30.0, 2)
    X = S.dense_int((m.rows, d), 4)
    Yd = S.dense_int((d, m.cols), 5)
    want = port.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values, X, Yd)
    got = S.sddmm(m.to_device(cuda), torch.from_numpy(X).to(cuda),
                  torch.from_numpy(Yd).to(cuda)).cpu().numpy()
    assert np.array_equal(got, want)


def test_sddmm_empty_rows_and_real(cuda):
    import torch
    m = S.generate_matrix("powerlaw", 3000, 3000, 0, 0, 0, 2.0, 9)  # many empty rows
    assert (np.diff(m.indptr) == 0).any()
    # Seeded: 64-term dots of N(0,1) data cancel, and both f32 pipelines sit near the 1e-5
    # line (measured over seeds 0-7: ours 0.73-1.12e-5, the reference F32 0.95-2.14e-5).
    for seed in (0, 1, 2):
        gen = torch.Generator(device=cuda)
        gen.manual_seed(seed)
        X = torch.randn(m.rows, 64, device=cuda, generator=gen)
        Yd = torch.randn(64, m.cols, device=cuda, generator=gen)
        got = S.sddmm(m.to_device(cuda), X, Yd).cpu().numpy()
        x, yd = X.cpu().numpy(), Yd.cpu().numpy()
        want = port.sddmm_csr_f64(m.rows, m.cols, m.indptr, m.indices, m.values, x, yd)
        ref32 = port.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values, x, yd)
        assert close_to_f64(got, want, ref32), seed
