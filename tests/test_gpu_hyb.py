"""GPU parity: device decompose_hyb and hyb/CSR SpMM, through the C ABI, against the oracle.

Bars (BASELINE.json north_star): format arrays bit-exact; fp32 SpMM bitwise equal to the
reference on the reference's integer operands and rel-err <= 1e-5 (driver.cpp:124-144 metric)
against the reference F64 pipeline on real-valued operands.
"""
import os

import numpy as np
import pytest

import paper_2207_04606_b200 as S
from oracle import port

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")
TOL = 1e-5  # |x - y| <= TOL * max(|x|, |y|, 1)   (driver.cpp:124-144)


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def ref_metric_err(got, want):
    """max |x - y| / max(|x|, |y|, 1) — the reference's compare() metric (driver.cpp:124-144)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    if got.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)
    return float(np.max(np.abs(got - want) / denom))


def close_ref_metric(got, want, tol=TOL):
    return ref_metric_err(got, want) <= tol


def close_to_f64(got, want64):
    """Real-valued parity bar, strict: |x - y| <= 1e-5 * max(|x|, |y|, 1) against the
    reference's F64 pipeline (driver.cpp:124-144 metric; the north_star's rel-err), with no
    allowance for the reference F32 pipeline's own drift."""
    err = ref_metric_err(got, want64)
    assert err <= TOL, f"rel-err {err:.3e} > {TOL:g} vs the F64 reference"
    return True


def csr_of(G, name):
    rows, cols = (int(x) for x in G[f"{name}/shape"])
    return S.CsrMatrix(rows, cols, G[f"{name}/indptr"], G[f"{name}/indices"], G[f"{name}/values"])


def check_parts(h, parts_ref, padding_ref):
    assert h.padding_ratio == padding_ref
    assert len(h.parts) == len(parts_ref)
    for i, (P, R) in enumerate(zip(h.parts, parts_ref)):
        assert (P.partition, P.bucket, P.width, P.nrows, P.nnz, P.pad_slots, P.col_lo, P.col_hi) == \
            tuple(R[:8] if isinstance(R, np.ndarray) else
                  [R[f] for f in ("partition", "bucket", "width", "nrows", "nnz", "pad_slots",
                                  "col_lo", "col_hi")])
        yield i, h.part_arrays(i)


def test_decompose_golden_bitexact(cuda, G):
    n = 0
    for name in G["cases"]:
        m = csr_of(G, name)
        dcsr = m.to_device(cuda)
        for key in sorted({k.rsplit("/", 1)[0] for k in G.files
                           if k.startswith(f"{name}/hyb_") and k.endswith("/meta")}):
            c, k = (int(t[1:]) for t in key.split("/")[-1].split("_")[1:])
            h = S.decompose_hyb(dcsr, c, k)
            meta = G[key + "/meta"]
            for i, arrs in check_parts(h, list(meta), float(G[key + "/padding"][0])):
                P = h.parts[i]
                pre = f"hyb_p{P.partition}_b{P.bucket}_"
                assert list(arrs[pre + "I_indptr"]) == [0, P.nrows]
                assert np.array_equal(arrs[pre + "I_indices"], G[f"{key}/p{i}/I"]), key
                assert np.array_equal(arrs[pre + "J_indices"], G[f"{key}/p{i}/J"]), key
                assert np.array_equal(arrs["values"].view(np.uint32),
                                      G[f"{key}/p{i}/V"].view(np.uint32)), key
            n += 1
    assert n >= 40


@pytest.mark.parametrize("c,k", [(1, 5), (1, 3), (2, 4), (4, 5), (16, 5), (1, 0), (3, 9)])
def test_decompose_c1_shape_vs_oracle(cuda, c, k):
    m = S.generate_matrix("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
    h = S.decompose_hyb(m.to_device(cuda), c, k)
    parts, pr = port.hyb_decompose(m.rows, m.cols, m.indptr, m.indices, m.values, c, k)
    for i, arrs in check_parts(h, parts, pr):
        R = parts[i]
        pre = f"hyb_p{R['partition']}_b{R['bucket']}_"
        assert np.array_equal(arrs[pre + "I_indices"], R["I_indices"])
        assert np.array_equal(arrs[pre + "J_indices"], R["J_indices"])
        assert np.array_equal(arrs["values"], R["values"])


def test_get_part_readback(cuda):
    """strata_hyb_get_part (SURVEY 8b's readback name) = part_info + part_read in one call."""
    import ctypes as C
    from paper_2207_04606_b200._lib import check, lib
    m = S.generate_matrix("powerlaw", 3000, 2900, 0, 0, 0, 12.0, 3)
    h = S.decompose_hyb(m.to_device(cuda), 2, 3)
    assert len(h.parts) > 2
    for i, P in enumerate(h.parts):
        part, bucket = C.c_int(), C.c_int()
        width, nrows = C.c_int64(), C.c_int64()
        iptr = np.empty(2, np.int32)
        ii = np.empty(P.nrows, np.int32)
        jj = np.empty(P.nrows * P.width, np.int32)
        vv = np.empty(P.nrows * P.width, np.float32)
        check(lib.strata_hyb_get_part(h._h, i, C.byref(part), C.byref(bucket), C.byref(width),
                                      C.byref(nrows), iptr.ctypes.data, ii.ctypes.data,
                                      jj.ctypes.data, vv.ctypes.data))
        assert (part.value, bucket.value, width.value, nrows.value) == (P.partition, P.bucket, P.width, P.nrows)
        want = h.part_arrays(i)
        got = [iptr, ii, jj, vv]
        for g, w in zip(got, want.values()):
            assert np.array_equal(g.view(np.uint32), np.asarray(w).view(np.uint32))
    with pytest.raises(S.StrataError) as e:
        check(lib.strata_hyb_get_part(h._h, len(h.parts), None, None, None, None, None, None, None, None))
    assert e.value.kind == "Lookup"


def test_decompose_usage_errors(cuda):
    m = S.generate_matrix("powerlaw", 100, 100, 0, 0, 0, 4.0, 1).to_device(cuda)
    with pytest.raises(S.StrataError) as e:
        S.decompose_hyb(m, 0, 2)
    assert e.value.kind == "Usage"


def test_hyb_rules_names(cuda, G):
    m = S.CsrMatrix(4, 4, np.array([0, 2, 3, 7, 7], np.int32),
                    np.array([0, 2, 3, 0, 1, 2, 3], np.int32), np.arange(1, 8, dtype=np.float32))
    _, rules = S.hyb_rules(m.to_device(cuda), 2, 2, "hyb")
    got = [f"{r['name']}|{r['new_buffer']}|" + ",".join(f"{a}:{n}" for a, n in sorted(r["arrays"].items()))
           for r in rules]
    assert got == list(G["rules/example_c2_k2"])


def test_spmm_golden(cuda, G):
    import torch
    for name in G["cases"]:
        m = csr_of(G, name)
        dcsr = m.to_device(cuda)
        for c, k in [(1, int(G[f"{name}/auto_k"][0])), (1, 1), (3, 2), (1, 0)]:
            h = S.decompose_hyb(dcsr, c, k)
            for d in (8, 32):
                for tag in ("int", "real"):
                    key = f"{name}/spmm_d{d}_{tag}"
                    X = torch.from_numpy(G[key + "/X"]).to(cuda)
                    Y = S.spmm(h, X).cpu().numpy()
                    if tag == "int":
                        assert np.array_equal(Y, G[key + "/Y"]), (key, c, k)
                    else:
                        assert close_to_f64(Y, G[key + "/Y64"]), (key, c, k)
            Yc = S.spmm_csr(dcsr, torch.from_numpy(G[f"{name}/spmm_d32_int/X"]).to(cuda))
            assert np.array_equal(Yc.cpu().numpy(), G[f"{name}/spmm_d32_int/Y"])


@pytest.mark.parametrize("d", [32, 64, 128, 256, 512, 8, 48, 1, 100])
def test_spmm_feature_sizes(cuda, d):
    import torch
    m = S.generate_matrix("powerlaw", 4000, 3000, 0, 0, 0, 20.0, 5)
    h = S.decompose_hyb(m.to_device(cuda), 1, S.hyb_auto_k(m))
    X = S.dense_int((m.cols, d), 9)
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    got = S.spmm(h, torch.from_numpy(X).to(cuda)).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("d", [64, 256, 512])
def test_spmm_x_16_byte_aligned(cuda, d):
    """X at a 16-byte-only aligned address: d = 64 takes the 128-bit-slice variant, d = 256 / 512
    the VEC kernels' two-128-bit-load fallback; bitwise equal to the 32-byte-aligned call."""
    import torch
    m = S.generate_matrix("powerlaw", 3000, 2800, 0, 0, 0, 20.0, 5)
    h = S.decompose_hyb(m.to_device(cuda), 1, 3)
    X = torch.from_numpy(S.dense_int((m.cols, d), 6)).to(cuda)
    buf = torch.empty(m.cols * d + 4, device=cuda)
    X16 = buf[4: 4 + m.cols * d].view(m.cols, d)
    X16.copy_(X)
    ya, yu = S.spmm(h, X).cpu().numpy(), S.spmm(h, X16).cpu().numpy()
    assert np.array_equal(ya, yu)
    assert np.array_equal(ya, port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.cpu().numpy()))


def special_x(shape, seed):
    """Integer operand with IEEE specials planted: +-inf, NaN, -0, f32 subnormals (the kernels'
    integer-pipe f32 -> f64 conversion must route inf / NaN to the F2F path and keep subnormals
    exact)."""
    X = S.dense_int(shape, seed)
    r = np.random.default_rng(seed)
    rows = r.choice(shape[0], size=min(shape[0], 40), replace=False)
    kinds = [np.inf, -np.inf, np.nan, -0.0, 1e-40, -3e-42, 2 ** -149]
    for q, i in enumerate(rows):
        X[i, r.integers(shape[1])] = kinds[q % len(kinds)]
    X[rows[-1], :] = np.float32(1.5e-39)  # a whole subnormal row
    return X


def check_special(got, want32, want64):
    """Non-finite outputs exactly where the reference F32 pipeline has them (NaN, and inf with
    its sign); every finite output within the strict 1e-5 bar of the F64 pipeline (the f32
    reference rounds each partial sum, which in the subnormal range is coarser than our single
    rounding of the exact sum)."""
    assert np.array_equal(np.isnan(got), np.isnan(want32))
    inf = np.isinf(want32)
    assert np.array_equal(np.isinf(got), inf) and np.array_equal(got[inf], want32[inf])
    fin = np.isfinite(want32)
    assert close_to_f64(got[fin], want64[fin])
    return True


@pytest.mark.parametrize("d", [32, 64, 128, 256])
@pytest.mark.parametrize("c", [1, 2])
def test_spmm_nonfinite_and_subnormal_x(cuda, d, c):
    """inf / NaN in X propagate as in the reference's sums (IEEE); -0 and subnormals exact;
    integer rows bitwise.  (Pad slots are skipped, not multiplied by 0: a non-finite x at a
    padded column yields the CSR result, where the reference's hyb nest would give 0 * inf =
    NaN, storage.cpp:528 / kernels.cpp:85-108.)"""
    import torch
    m = S.generate_matrix("powerlaw", 3000, 2500, 0, 0, 0, 18.0, 4)
    X = special_x((m.cols, d), 11)
    with np.errstate(invalid="ignore", over="ignore"):
        want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
        want64 = port.spmm_csr_f64(m.rows, m.indptr, m.indices, m.values, X)
    assert np.isnan(want).any() and np.isinf(want).any()
    dm = m.to_device(cuda)
    for k in (S.hyb_auto_k(m), 1):
        got = S.spmm(S.decompose_hyb(dm, c, k), torch.from_numpy(X).to(cuda)).cpu().numpy()
        assert check_special(got, want, want64), (d, c, k)
    got = S.spmm_csr(dm, torch.from_numpy(X).to(cuda)).cpu().numpy()
    assert check_special(got, want, want64), d


def test_spmm_long_split_rows_deterministic(cuda):
    """Rows far above 2^k split into many bucket-k segments spanning many chunks (the
    carry + fix-up path); results must be exact on integer data and bitwise reproducible."""
    import torch
    m = S.generate_matrix("powerlaw", 20000, 20000, 0, 0, 0, 60.0, 7)
    assert np.diff(m.indptr).max() > 5000
    dcsr = m.to_device(cuda)
    for c, k in [(1, 0), (1, 2), (1, 6), (2, 3)]:
        h = S.decompose_hyb(dcsr, c, k)
        for d in (32, 64, 128):
            X = S.dense_int((m.cols, d), 3)
            want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
            Xd = torch.from_numpy(X).to(cuda)
            y1 = S.spmm(h, Xd).cpu().numpy()
            assert np.array_equal(y1, want), (c, k, d)
            Xr = torch.randn(m.cols, d, device=cuda)
            r1 = S.spmm(h, Xr).cpu().numpy()
            r2 = S.spmm(h, Xr).cpu().numpy()
            assert np.array_equal(r1.view(np.uint32), r2.view(np.uint32)), "not deterministic"
            xr = Xr.cpu().numpy()
            want64 = port.spmm_csr_f64(m.rows, m.indptr, m.indices, m.values, xr)
            ref32 = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, xr)
            assert close_to_f64(r1, want64), (c, k, d)
            # and clearly better than the reference's own f32 accumulation on long rows
            assert ref_metric_err(r1, want64) <= ref_metric_err(ref32, want64)


def test_spmm_empty_and_tiny(cuda):
    import torch
    for rows, cols in [(5, 7), (1, 1), (64, 3)]:
        m = S.CsrMatrix(rows, cols, np.zeros(rows + 1, np.int32), np.zeros(0, np.int32),
                        np.zeros(0, np.float32))
        h = S.decompose_hyb(m.to_device(cuda), 1, 2)
        assert h.parts == [] and h.padding_ratio == 0.0
        Y = torch.full((rows, 32), 7.0, device=cuda)
        S.spmm(h, torch.ones(cols, 32, device=cuda), Y)
        assert float(Y.abs().max()) == 0.0  # outputs are zero-initialised like interp.cpp:584


def test_spmm_host_e2e(cuda):
    import torch
    m = S.generate_matrix("powerlaw", 8000, 8000, 0, 0, 0, 16.0, 1)
    h = S.decompose_hyb(m.to_device(cuda), 1, S.hyb_auto_k(m))
    X = torch.from_numpy(S.dense_int((m.cols, 128), 1)).pin_memory()
    Y = torch.empty((m.rows, 128), dtype=torch.float32).pin_memory()
    S.spmm_host(h, X, Y)
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.numpy())
    assert np.array_equal(Y.numpy(), want)


def test_spmm_host_batch_pipelined(cuda):
    """Batched e2e form: 5 different feature matrices through two staging slots (slot reuse
    ordering across the copy-in / compute / copy-out streams), each equal to the oracle; a
    pageable (non-pinned) output and an empty batch are accepted."""
    import torch
    m = S.generate_matrix("powerlaw", 8000, 8000, 0, 0, 0, 16.0, 1)
    h = S.decompose_hyb(m.to_device(cuda), 1, S.hyb_auto_k(m))
    Xs = [torch.from_numpy(S.dense_int((m.cols, 64), 10 + b)).pin_memory() for b in range(5)]
    Ys = [torch.empty((m.rows, 64), dtype=torch.float32).pin_memory() for _ in range(4)]
    Ys.append(torch.empty((m.rows, 64), dtype=torch.float32))
    S.spmm_host_batch(h, Xs, Ys)
    for X, Y in zip(Xs, Ys):
        want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.numpy())
        assert np.array_equal(Y.numpy(), want)
    S.spmm_host_batch(h, [], [])


def test_spmm_c1_full_vs_oracle(cuda):
    """BASELINE config C1 (power-law n=65,536, avg 16, seed 1, d=32, hyb:c=1) at full size."""
    import torch
    m = S.generate_matrix("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
    assert m.nnz == 1048664
    h = S.decompose_hyb(m.to_device(cuda), 1, S.hyb_auto_k(m))
    assert [P.nrows for P in h.parts] == [5151, 28959, 15924, 8084, 26597]
    X = S.dense_int((m.cols, 32), 1)
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    got = S.spmm(h, torch.from_numpy(X).to(cuda)).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.slow
def test_spmm_products_full_vs_oracle(cuda):
    """BASELINE config C5 (products shape, d=128) at full size: bitwise on integer operands."""
    import torch
    m = S.generate_matrix("powerlaw", 2449029, 2449029, 0, 0, 0, 25.3, 1)
    assert m.nnz == 61943588
    h = S.decompose_hyb(m.to_device(cuda), 1, S.hyb_auto_k(m))
    assert [P.nrows for P in h.parts] == [755092, 858332, 435726, 1695641]
    assert abs(h.padding_ratio - 0.1290) < 5e-4
    X = S.dense_int((m.cols, 128), 1)
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    got = S.spmm(h, torch.from_numpy(X).to(cuda)).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("d", [32, 64, 128])
def test_spmm_csr_long_rows(cuda, d):
    """Row-split CSR SpMM (the reference's default "csr" format) on a power-law graph whose hub
    rows exceed the 2,048-non-zero threshold: chunked long rows and the two merge levels are
    bitwise equal to the oracle on integer operands, the rest of the rows too; real-valued data
    within the F64 bar."""
    import torch
    m = S.generate_matrix("powerlaw", 60000, 60000, 0, 0, 0, 20.0, 3)
    assert np.diff(m.indptr).max() > 2048 * 4
    dm = m.to_device(cuda)
    X = S.dense_int((m.cols, d), 5)
    Y = S.spmm_csr(dm, torch.from_numpy(X).to(cuda)).cpu().numpy()
    assert np.array_equal(Y, port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X))
    xr = np.random.default_rng(d).standard_normal((m.cols, d)).astype(np.float32)
    Yr = S.spmm_csr(dm, torch.from_numpy(xr).to(cuda)).cpu().numpy()
    want64 = port.spmm_csr_f64(m.rows, m.indptr, m.indices, m.values, xr)
    ref32 = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, xr)
    assert close_to_f64(Yr, want64)
    # the reference F32 order itself drifts on these hub rows; ours must not be worse
    assert ref_metric_err(Yr, want64) <= max(ref_metric_err(ref32, want64), 1e-7)
