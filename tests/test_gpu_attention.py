"""GPU: fused SDDMM -> edge softmax -> SpMM (strata_attn_csr_f32) against an f64 restatement
of the three composed steps (the reference's SDDMM nest, a row softmax over the stored
entries, the reference's SpMM nest).  Tolerance: |z - z64| <= 2e-5 * max(|z|, |z64|, 1)
(the driver.cpp:124-144 metric at twice the f32 SpMM bar: exp and the online rescaling add a
few ulp per edge)."""
import numpy as np
import pytest
import torch

import paper_2207_04606_b200 as S

from test_gpu_hyb import close_ref_metric

pytestmark = pytest.mark.gpu


def attention_f64(m, Q, K, V):
    Q, K, V = (x.astype(np.float64) for x in (Q, K, V))
    Z = np.zeros((m.rows, V.shape[1]))
    for i in range(m.rows):
        q0, q1 = int(m.indptr[i]), int(m.indptr[i + 1])
        if q1 == q0:
            continue
        cols = m.indices[q0:q1]
        s = m.values[q0:q1].astype(np.float64) * (K[cols] @ Q[i])
        w = np.exp(s - s.max())
        Z[i] = (w / w.sum()) @ V[cols]
    return Z


@pytest.mark.parametrize("d,avg", [(64, 12.0), (32, 40.0), (128, 6.0)])
def test_attention_power_law_with_hub_rows(cuda, d, avg):
    g0 = S.generate_matrix("powerlaw", 3000, 2500, 0, 0, 0, avg, 4)  # hub rows > 256 edges
    # empty every 7th row (the generator's rows all have >= 1 entry at these densities)
    lens = np.diff(g0.indptr)
    keep = np.repeat(np.arange(g0.rows) % 7 != 0, lens)
    lens = np.where(np.arange(g0.rows) % 7 != 0, lens, 0)
    m = S.CsrMatrix(g0.rows, g0.cols, np.r_[0, np.cumsum(lens)].astype(np.int32),
                    g0.indices[keep], g0.values[keep])
    assert np.diff(m.indptr).max() > 256 and (np.diff(m.indptr) == 0).any()
    g = torch.Generator(device=cuda)
    g.manual_seed(d)
    Q = torch.randn(m.rows, d, device=cuda, generator=g) * 0.3
    K = torch.randn(m.cols, d, device=cuda, generator=g) * 0.3
    V = torch.randn(m.cols, d, device=cuda, generator=g)
    plan = S.AttentionPlan(m.to_device(cuda))
    Z = plan(Q, K, V).cpu().numpy()
    want = attention_f64(m, Q.cpu().numpy(), K.cpu().numpy(), V.cpu().numpy())
    assert close_ref_metric(Z, want, 2e-5)
    assert not Z[np.diff(m.indptr) == 0].any()
    Z2 = plan(Q, K, V).cpu().numpy()
    assert np.array_equal(Z, Z2)  # deterministic


@pytest.mark.parametrize("d", [64, 128])
def test_attention_16_byte_aligned_operands(cuda, d):
    """K at a 16-byte-only aligned address takes the 128-bit path; same result within the bar
    and the 256-bit path's result on aligned copies."""
    m = S.generate_matrix("powerlaw", 2000, 1800, 0, 0, 0, 30.0, 5)
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    Q = torch.randn(m.rows, d, device=cuda, generator=g) * 0.3
    K = torch.randn(m.cols, d, device=cuda, generator=g) * 0.3
    V = torch.randn(m.cols, d, device=cuda, generator=g)
    buf = torch.empty(m.cols * d + 4, device=cuda)
    K16 = buf[4: 4 + m.cols * d].view(m.cols, d)
    K16.copy_(K)
    plan = S.AttentionPlan(m.to_device(cuda))
    Za = plan(Q, K, V).cpu().numpy()
    Zu = plan(Q, K16, V).cpu().numpy()
    want = attention_f64(m, Q.cpu().numpy(), K.cpu().numpy(), V.cpu().numpy())
    assert close_ref_metric(Za, want, 2e-5) and close_ref_metric(Zu, want, 2e-5)


def test_attention_usage_errors(cuda):
    m = S.generate_matrix("powerlaw", 100, 100, 0, 0, 0, 4.0, 1)
    plan = S.AttentionPlan(m.to_device(cuda))
    x = torch.zeros(100, 48, device=cuda)
    with pytest.raises(S.StrataError) as e:
        plan(x, x, x)
    assert e.value.kind == "Usage"
