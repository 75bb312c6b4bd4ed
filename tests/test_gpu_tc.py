"""GPU parity: device csr_to_bsr / csr_to_ell (bit-exact) and the tcgen05 tensor-core kernels
(BSR SpMM, RGMS gather-GEMM-scatter) through the C ABI.

Bars (BASELINE.json north_star): format arrays bit-exact; bf16 tensor-core results equal to the
f32 reference on the reference's integer operands (exact in bf16, f32 accumulation) and within
1e-2 relative (driver.cpp:124-144 metric) of the F64 oracle on real-valued operands."""
import os

import numpy as np
import pytest

import paper_2207_04606_b200 as S
from oracle import port

from test_gpu_hyb import close_ref_metric, ref_metric_err

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def bf16(t):
    import torch
    return t.to(torch.bfloat16)


def test_bsr_arrays_golden(cuda, G):
    keys = sorted({k.rsplit("/", 1)[0] for k in G.files if k.startswith("bsr/")})
    for key in keys:
        rows, cols, prow, pcol, pad = (int(x) for x in G[key + "/shape"])
        b = int(key.rsplit("_b", 1)[1])
        m = S.CsrMatrix(rows, cols, G[key + "/csr_indptr"], G[key + "/csr_indices"],
                        G[key + "/csr_values"])
        bs = S.csr_to_bsr(m.to_device(cuda), b)
        a = bs.arrays()
        assert (bs.mb * b, bs.nb * b, bs.pad_slots) == (prow, pcol, pad), key
        assert np.array_equal(a["bsr_JO_indptr"], G[key + "/JO_indptr"]), key
        assert np.array_equal(a["bsr_JO_indices"], G[key + "/JO_indices"]), key
        assert np.array_equal(a["values"], G[key + "/values"]), key


def test_bsr_spmm_golden(cuda, G):
    import torch
    for key in ("bsr/bs128_b32", "bsr/pl_b32_b32"):
        rows, cols, prow, pcol, pad = (int(x) for x in G[key + "/shape"])
        m = S.CsrMatrix(rows, cols, G[key + "/csr_indptr"], G[key + "/csr_indices"],
                        G[key + "/csr_values"])
        bs = S.csr_to_bsr(m.to_device(cuda), 32)
        X = torch.from_numpy(G[key + "/X"]).to(cuda)
        Y = S.bsr_spmm(bs, bf16(X)).cpu().numpy()
        assert np.array_equal(Y, G[key + "/Y"]), key


@pytest.mark.parametrize("d", [64, 128, 256])
def test_bsr_spmm_c3_shape(cuda, d):
    """C3: block-sparse 4096^2 mask, b = 32, density 0.1, seed 1 (1,589 blocks)."""
    import torch
    m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
    bs = S.csr_to_bsr(m.to_device(cuda), 32)
    assert bs.nblocks == 1589 and bs.pad_slots == 0
    jp, ji, bv = port.csr_to_bsr(m.rows, m.cols, m.indptr, m.indices, m.values, 32)
    a = bs.arrays()
    assert np.array_equal(a["bsr_JO_indptr"], jp) and np.array_equal(a["bsr_JO_indices"], ji)
    assert np.array_equal(a["values"], bv)
    X = S.dense_int((4096, d), 3)
    want = port.bsr_spmm_refnum(128, 32, jp, ji, bv, X)
    Y = S.bsr_spmm(bs, bf16(torch.from_numpy(X).to(cuda))).cpu().numpy()
    assert np.array_equal(Y, want)
    # real-valued operands: bf16 inputs, f32 accumulate vs the F64 product of the same inputs
    Xr = torch.randn(4096, d, device=cuda).to(torch.bfloat16)
    Yr = S.bsr_spmm(bs, Xr).cpu().numpy()
    Xr64 = Xr.float().cpu().numpy().astype(np.float64)
    dense = np.zeros((4096, 4096))
    for br in range(128):
        for q in range(jp[br], jp[br + 1]):
            dense[br * 32:(br + 1) * 32, ji[q] * 32:(ji[q] + 1) * 32] = bv[q * 1024:(q + 1) * 1024].reshape(32, 32)
    assert close_ref_metric(Yr, dense @ Xr64, 1e-2)


def test_bsr_spmm_pdl_producer_consumer(cuda):
    """The BSR SpMM is launched with programmatic dependent launch; its inputs are read only
    after griddepcontrol.wait.  Chain producer kernels (X written by torch on the same stream)
    and back-to-back SpMMs whose output feeds the next X, without host syncs, and check every
    result against the oracle chain."""
    import torch
    m = S.generate_matrix("blocksparse", 1024, 1024, 0.2, 0, 32, 0, 2)
    bs = S.csr_to_bsr(m.to_device(cuda), 32)
    jp, ji, bv = port.csr_to_bsr(m.rows, m.cols, m.indptr, m.indices, m.values, 32)
    X0 = S.dense_int((1024, 64), 9)
    Xd = bf16(torch.from_numpy(X0).to(cuda))
    outs = []
    for i in range(6):
        Xd = (Xd.float() + i).remainder(5).sub(2).to(torch.bfloat16)  # producer kernels
        Y = S.bsr_spmm(bs, Xd)                                       # consumer (PDL launch)
        outs.append((Xd, Y))
        Xd = Y.remainder(7).sub(3).to(torch.bfloat16)                 # next X from Y
    torch.cuda.synchronize()
    for Xi, Yi in outs:
        want = port.bsr_spmm_refnum(32, 32, jp, ji, bv, Xi.float().cpu().numpy())
        assert np.array_equal(Yi.cpu().numpy(), want)


@pytest.mark.parametrize("heads,d", [(12, 64), (3, 128), (2, 512)])
def test_bsr_spmm_batched_heads(cuda, heads, d):
    """Multi-head batched SpMM: 12 heads on the C3 mask, per-head block values
    and features; each head bitwise equal to the oracle on integer operands, and the
    single-head call through the batched entry equal to strata_bsr_spmm_bf16."""
    import torch
    m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
    bs = S.csr_to_bsr(m.to_device(cuda), 32)
    jp, ji, _ = port.csr_to_bsr(m.rows, m.cols, m.indptr, m.indices, m.values, 32)
    rng = np.random.default_rng(heads * 1000 + d)
    vals = rng.integers(1, 10, (heads, bs.nblocks, 32, 32)).astype(np.float32)
    X = rng.integers(-3, 4, (heads, 4096, d)).astype(np.float32)
    Y = S.bsr_spmm_batched(bs, bf16(torch.from_numpy(vals).to(cuda)),
                           bf16(torch.from_numpy(X).to(cuda))).cpu().numpy()
    for h in range(heads):
        want = port.bsr_spmm_refnum(128, 32, jp, ji, vals[h].reshape(-1), X[h])
        assert np.array_equal(Y[h], want), h
    one = S.bsr_spmm(bs, bf16(torch.from_numpy(X[0]).to(cuda))).cpu().numpy()
    own = bs.arrays()["values"].reshape(1, bs.nblocks, 32, 32)
    Y1 = S.bsr_spmm_batched(bs, bf16(torch.from_numpy(own).to(cuda)),
                            bf16(torch.from_numpy(X[:1]).to(cuda))).cpu().numpy()
    assert np.array_equal(Y1[0], one)


@pytest.mark.parametrize("heads,d,shape", [(1, 64, (4096, 4096, 0.1)), (12, 64, (1024, 2048, 0.2)),
                                           (3, 128, (512, 768, 0.3))])
def test_bsr_sddmm_heads(cuda, heads, d, shape):
    """Block-sparse SDDMM on tcgen05 (four key blocks per MMA): S = A (.) Q K^T on the stored
    blocks, every head bitwise equal to an f64 restatement on integer operands (exact in bf16
    and f32); partial last groups of a block row and empty block rows included."""
    import torch
    n, mcols, dens = shape
    m = S.generate_matrix("blocksparse", n, mcols, dens, 0, 32, 0, 2)
    bs = S.csr_to_bsr(m.to_device(cuda), 32)
    a = bs.arrays()
    jp, ji = a["bsr_JO_indptr"], a["bsr_JO_indices"]
    A = a["values"].reshape(-1, 32, 32).astype(np.float64)
    rng = np.random.default_rng(heads * 7 + d)
    Q = rng.integers(-3, 4, (heads, bs.mb * 32, d)).astype(np.float32)
    K = rng.integers(-3, 4, (heads, bs.nb * 32, d)).astype(np.float32)
    Sg = S.bsr_sddmm(bs, bf16(torch.from_numpy(Q).to(cuda)), bf16(torch.from_numpy(K).to(cuda)))
    Sg = Sg.cpu().numpy()
    for h in range(heads):
        for br in range(bs.mb):
            qt = Q[h, br * 32:(br + 1) * 32].astype(np.float64)
            for q in range(jp[br], jp[br + 1]):
                kt = K[h, ji[q] * 32:(ji[q] + 1) * 32].astype(np.float64)
                assert np.array_equal(Sg[h, q], (A[q] * (qt @ kt.T)).astype(np.float32)), (h, br, q)


def test_bsr_empty_block_rows(cuda):
    import torch
    m = S.generate_matrix("blocksparse", 512, 256, 0.05, 0, 32, 0, 4)
    bs = S.csr_to_bsr(m.to_device(cuda), 32)
    jp, ji, bv = port.csr_to_bsr(m.rows, m.cols, m.indptr, m.indices, m.values, 32)
    assert (np.diff(jp) == 0).any()
    X = S.dense_int((256, 64), 1)
    Y = S.bsr_spmm(bs, bf16(torch.from_numpy(X).to(cuda)), torch.full((512, 64), 9.0, device=cuda))
    assert np.array_equal(Y.cpu().numpy(), port.bsr_spmm_refnum(16, 32, jp, ji, bv, X))


def test_ell_golden_and_capacity(cuda, G):
    for name in ("example", "pl"):
        meta = G[f"ell/{name}/csr"]
        rows, cols, w = (int(x) for x in meta[:3])
        m = S.CsrMatrix(rows, cols, meta[3:].astype(np.int32), G[f"ell/{name}/indices"],
                        G[f"ell/{name}/values"])
        J, V = S.csr_to_ell(m.to_device(cuda), w)
        assert np.array_equal(J.cpu().numpy(), G[f"ell/{name}/J"])
        assert np.array_equal(V.cpu().numpy(), G[f"ell/{name}/V"])
    # test_storage.cpp:95-100: w = 2 on the example fails naming row 2 (Capacity)
    ex = S.CsrMatrix(4, 4, np.array([0, 2, 3, 7, 7], np.int32),
                     np.array([0, 2, 3, 0, 1, 2, 3], np.int32), np.arange(1, 8, dtype=np.float32))
    with pytest.raises(S.StrataError) as e:
        S.csr_to_ell(ex.to_device(cuda), 2)
    assert e.value.kind == "Capacity" and "row 2" in str(e.value)


def test_rgms_golden(cuda, G):
    import torch
    R, m, n = (int(x) for x in G["rgms/shape"])
    rel = S.RelSparse.from_reference_arrays(R, m, n, G["rgms/I_indptr"], G["rgms/I_indices"],
                                            G["rgms/J_indptr"], G["rgms/J_indices"], G["rgms/A"])
    drel = rel.to_device(cuda)
    for fmt in ("csr", "hyb"):
        X = bf16(torch.from_numpy(G[f"rgms/{fmt}/X"]).to(cuda))
        W = bf16(torch.from_numpy(G[f"rgms/{fmt}/W"]).to(cuda))
        Y = S.rgms(drel, X, W).cpu().numpy()
        assert np.array_equal(Y, G[f"rgms/{fmt}/Y"]), fmt


def _relation_csrs(R, m, n, I_indptr, I_indices, J_indptr, J_indices, A):
    """Per-relation CsrMatrix slices of a reference RelSparse (kernels.cpp:19-62)."""
    out = []
    for r in range(R):
        counts = np.zeros(m, np.int64)
        cols, vals = [], []
        for a in range(I_indptr[r], I_indptr[r + 1]):
            i = I_indices[a]
            counts[i] = J_indptr[a + 1] - J_indptr[a]
            cols.append(J_indices[J_indptr[a]:J_indptr[a + 1]])
            vals.append(A[J_indptr[a]:J_indptr[a + 1]])
        indptr = np.r_[0, np.cumsum(counts)].astype(np.int32)
        ix = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
        vv = np.concatenate(vals).astype(np.float32) if vals else np.zeros(0, np.float32)
        out.append(S.CsrMatrix(m, n, indptr, ix, vv))
    return out


def test_rgms_hyb_parts_golden(cuda, G):
    """strata_rgms_plan_hyb (SURVEY §8b strata_rgms_hyb_bf16): per-relation hyb decompositions
    (k = hyb_auto_k of each slice, as driver.cpp:294-300) read in place -> the reference's
    "hyb" RGMS pipeline output, bitwise."""
    import torch
    R, m, n = (int(x) for x in G["rgms/shape"])
    slices = _relation_csrs(R, m, n, G["rgms/I_indptr"], G["rgms/I_indices"], G["rgms/J_indptr"],
                            G["rgms/J_indices"], G["rgms/A"])
    hybs = [S.decompose_hyb(c.to_device(cuda), 1, S.hyb_auto_k(c)) for c in slices]
    X = bf16(torch.from_numpy(G["rgms/hyb/X"]).to(cuda))
    W = bf16(torch.from_numpy(G["rgms/hyb/W"]).to(cuda))
    Y = S.RgmsPlan.from_hyb(hybs).run(X, W).cpu().numpy()
    assert np.array_equal(Y, G["rgms/hyb/Y"])


@pytest.mark.parametrize("c,k", [(1, 0), (2, 1), (3, 2)])
def test_rgms_hyb_parts_equal_csr_plan(cuda, c, k):
    """Split rows (l > 2^k), padding and column partitions in the parts: same Y as the CSR
    plan of the same relations, bitwise on integer operands."""
    import torch
    g = S.generate_matrix("powerlaw", 6000, 5000, 0, 0, 0, 6.0, 3)
    rel = S.split_relations(g, 7, 2)
    slices = []
    for r in range(7):
        lo, hi = int(rel.rel_ptr[r]), int(rel.rel_ptr[r + 1])
        dst, src, a = rel.dst[lo:hi], rel.src[lo:hi], rel.A[lo:hi]
        indptr = np.r_[0, np.cumsum(np.bincount(dst, minlength=rel.rows))].astype(np.int32)
        slices.append(S.CsrMatrix(rel.rows, rel.cols, indptr, src.astype(np.int32), a.astype(np.float32)))
    # relation 3 emptied: a hyb with no parts, and its edges gone from the CSR reference too
    lo3, hi3 = int(rel.rel_ptr[3]), int(rel.rel_ptr[4])
    slices[3] = S.CsrMatrix(rel.rows, rel.cols, np.zeros(rel.rows + 1, np.int32),
                            np.zeros(0, np.int32), np.zeros(0, np.float32))
    keep = np.r_[np.arange(0, lo3), np.arange(hi3, rel.nnz)]
    rel = S.RelSparse(7, rel.rows, rel.cols,
                      np.r_[rel.rel_ptr[:4], rel.rel_ptr[4:] - (hi3 - lo3)].astype(np.int32),
                      rel.dst[keep], rel.src[keep], rel.A[keep])
    hybs = [S.decompose_hyb(sl.to_device(cuda), c, k) for sl in slices]
    X = bf16(torch.from_numpy(S.dense_int((rel.cols, 32), 4)).to(cuda))
    W = bf16(torch.from_numpy(S.dense_int((7, 32, 32), 5)).to(cuda))
    Yh = S.RgmsPlan.from_hyb(hybs).run(X, W)
    Yc = S.RgmsPlan(rel.to_device(cuda)).run(X, W)
    assert torch.equal(Yh, Yc)


@pytest.mark.parametrize("din,dout", [(32, 32), (16, 16), (64, 64), (32, 128)])
def test_rgms_random_vs_oracle(cuda, din, dout):
    import torch
    m = S.generate_matrix("powerlaw", 20000, 20000, 0, 0, 0, 3.0, 5)
    rel = S.split_relations(m, 13, 1)
    X = S.dense_int((m.cols, din), 2)
    W = S.dense_int((13, din, dout), 3)
    # RelSparse reference arrays from the flattened edge list
    i_indptr, i_indices, j_indptr = [0], [], [0]
    for r in range(13):
        e0, e1 = rel.rel_ptr[r], rel.rel_ptr[r + 1]
        d_ = rel.dst[e0:e1]
        starts = np.flatnonzero(np.r_[True, d_[1:] != d_[:-1]]) if e1 > e0 else np.array([], int)
        i_indices += d_[starts].tolist()
        j_indptr += (e0 + np.r_[starts[1:], e1 - e0]).tolist() if e1 > e0 else []
        i_indptr.append(len(i_indices))
    want = port.rgms_refnum(13, m.rows, np.array(i_indptr, np.int32), np.array(i_indices, np.int32),
                            np.array(j_indptr, np.int32), rel.src, rel.A, X, W)
    Y = S.rgms(rel.to_device(cuda), bf16(torch.from_numpy(X).to(cuda)),
               bf16(torch.from_numpy(W).to(cuda))).cpu().numpy()
    assert np.array_equal(Y, want)


def test_rgms_am_shape_relation_split(cuda):
    """C4 structure: AM-shaped power-law graph split into 133 relations (every relation gets
    hyb_auto_k = 0, i.e. width-1 ELL rows)."""
    m = S.generate_matrix("powerlaw", 1885136, 1885136, 0, 0, 0, 3.0051, 1)
    assert m.nnz == 5668776
    rel = S.split_relations(m, 133, 1)
    per = np.diff(rel.rel_ptr)
    assert per.sum() == m.nnz and per.min() >= 42033 and per.max() <= 43251


def _rgms_dense_f64(rel, X, W):
    """Per-relation f64 restatement of the RGMS nest (kernels.cpp:138-167) for large checks:
    exact on integer operands, so it equals the reference's F32 pipeline bitwise."""
    Y = np.zeros((rel.rows, W.shape[2]), np.float64)
    Xd = X.astype(np.float64)
    for r in range(rel.relations):
        e0, e1 = int(rel.rel_ptr[r]), int(rel.rel_ptr[r + 1])
        if e1 == e0:
            continue
        msg = (Xd[rel.src[e0:e1]] @ W[r].astype(np.float64)) * rel.A[e0:e1, None]
        np.add.at(Y, rel.dst[e0:e1], msg)
    return Y


def test_rgms_c4_full_size(cuda):
    """C4 at full size (1.9M nodes, 5.67M edges, 133 relations, d 32 -> 32) through the plan /
    run split, bitwise vs the f64 restatement on integer operands; a second run on the same
    plan with new X and W (plan reuse) and a run with d_out = 64 (T workspace growth)."""
    import torch
    m = S.generate_matrix("powerlaw", 1885136, 1885136, 0, 0, 0, 3.0051, 1)
    rel = S.split_relations(m, 133, 1)
    plan = S.RgmsPlan(rel.to_device(cuda))
    for seed, dout in ((2, 32), (4, 32), (6, 64)):
        X = S.dense_int((m.cols, 32), seed)
        W = S.dense_int((133, 32, dout), seed + 1)
        Y = plan.run(bf16(torch.from_numpy(X).to(cuda)), bf16(torch.from_numpy(W).to(cuda)))
        want = _rgms_dense_f64(rel, X, W)
        assert np.array_equal(Y.cpu().numpy(), want.astype(np.float32)), (seed, dout)


def test_rgms_empty_relations_and_rows(cuda):
    """Relations without edges, rows without edges (Y row = 0, interp.cpp:584-587) and an
    edgeless RelSparse; dimension errors are Usage errors naming the supported set."""
    import torch
    R, rows, cols = 5, 300, 200
    rng = np.random.default_rng(3)
    dst = np.sort(rng.integers(0, rows // 2, 700)).astype(np.int32)  # rows >= 150 stay empty
    counts = np.array([0, 400, 0, 300, 0])
    rel_ptr = np.r_[0, np.cumsum(counts)].astype(np.int32)
    dsts = np.concatenate([np.sort(dst[:400]), np.sort(dst[400:])]).astype(np.int32)
    rel = S.RelSparse(R, rows, cols, rel_ptr, dsts, rng.integers(0, cols, 700).astype(np.int32),
                      rng.integers(1, 10, 700).astype(np.float32))
    X = S.dense_int((cols, 16), 5)
    W = S.dense_int((R, 16, 16), 6)
    Y = S.rgms(rel.to_device(cuda), bf16(torch.from_numpy(X).to(cuda)),
               bf16(torch.from_numpy(W).to(cuda))).cpu().numpy()
    assert np.array_equal(Y, _rgms_dense_f64(rel, X, W).astype(np.float32))
    assert not Y[150:].any()
    empty = S.RelSparse(2, 10, 10, np.zeros(3, np.int32), np.zeros(0, np.int32),
                        np.zeros(0, np.int32), np.zeros(0, np.float32))
    Xe = bf16(torch.ones((10, 16), device=cuda))
    We = bf16(torch.ones((2, 16, 16), device=cuda))
    Ye = S.rgms(S.RgmsPlan(empty.to_device(cuda)), Xe, We)
    assert Ye.shape == (10, 16) and not Ye.any()
    with pytest.raises(S.StrataError) as e:
        S.rgms(rel.to_device(cuda), bf16(torch.ones((cols, 48), device=cuda)),
               bf16(torch.ones((R, 48, 16), device=cuda)))
    assert e.value.kind == "Usage"


@pytest.mark.parametrize("case", ["all_direct", "no_direct", "mixed_hub"])
def test_rgms_direct_rows(cuda, case):
    """Rows whose edges form a single run are written to Y by pass 1 (no message row); the rest
    go through message rows and pass 2.  Exercise a graph where every row is direct, one where
    none is (every row has two relations), and a mix with a hub row above the long-row
    threshold; plus the sign of zero (a direct row summing to 0 must read +0.0, as the
    reference's 0 + x)."""
    import torch
    rng = np.random.default_rng(11)
    R, rows, cols = 4, 2000, 1500
    if case == "all_direct":      # one edge per row, relation = row % R
        dst = np.arange(rows)
        rel_of = dst % R
    elif case == "no_direct":     # two edges per row in two different relations
        dst = np.repeat(np.arange(rows), 2)
        rel_of = (dst + np.tile([0, 1], rows)) % R
    else:                         # light rows + one hub row with 5,000 edges in all relations
        dst = np.r_[rng.integers(0, rows, 3000), np.full(5000, 7)]
        rel_of = rng.integers(0, R, dst.size)
    order = np.lexsort((dst, rel_of))
    dst, rel_of = dst[order].astype(np.int32), rel_of[order]
    rel_ptr = np.r_[0, np.cumsum(np.bincount(rel_of, minlength=R))].astype(np.int32)
    src = rng.integers(0, cols, dst.size).astype(np.int32)
    A = rng.integers(1, 10, dst.size).astype(np.float32)
    rel = S.RelSparse(R, rows, cols, rel_ptr, dst, src, A)
    X = S.dense_int((cols, 32), 7)
    X[src[:50]] = 0  # some rows' messages are exactly zero
    W = S.dense_int((R, 32, 32), 8)
    plan = S.RgmsPlan(rel.to_device(cuda))
    Y = plan.run(bf16(torch.from_numpy(X).to(cuda)), bf16(torch.from_numpy(W).to(cuda))).cpu().numpy()
    want = _rgms_dense_f64(rel, X, W).astype(np.float32)
    assert np.array_equal(Y, want)
    assert not np.signbit(Y[Y == 0]).any()  # no -0.0
    if case == "all_direct":
        assert plan.message_rows == 0
    if case == "no_direct":
        assert plan.message_rows == dst.size


@pytest.mark.parametrize("din,dout", [(32, 32), (64, 128)])
def test_rgms_real_valued_vs_f64(cuda, din, dout):
    """Real-valued N(0,1) features and weights (rounded to bf16 — the operator's input type)
    with the generator's A in 1..9: within the north_star's 1e-2 of the F64 restatement of the
    RGMS nest (kernels.cpp:138-167), metric of driver.cpp:124-144.  Includes power-law hub rows
    (long-row chunk path) and rows with a single run (direct rows)."""
    import torch
    m = S.generate_matrix("powerlaw", 30000, 30000, 0, 0, 0, 6.0, 4)
    rel = S.split_relations(m, 13, 2)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(din + dout)
    Xb = bf16(torch.randn(m.cols, din, device=cuda, generator=gen))
    Wb = bf16(torch.randn(13, din, dout, device=cuda, generator=gen) / din ** 0.5)
    Y = S.RgmsPlan(rel.to_device(cuda)).run(Xb, Wb).cpu().numpy()
    want = _rgms_dense_f64(rel, Xb.float().cpu().numpy(), Wb.float().cpu().numpy())
    assert close_ref_metric(Y, want, 1e-2)
    assert ref_metric_err(Y, want) < 1e-4  # fp32 accumulation of exact bf16 products
