"""CPU suite: pin the oracle (oracle/strata_oracle.c) to the reference.

1. The reference's own hand-derived known-answer tests (proj/tests/test_storage.cpp,
   proj/tests/test_kernels.cpp), restated as constants with file:line.
2. tests/golden/golden.npz, produced by the UNMODIFIED reference library
   (tests/golden/make_golden.py): decompose_hyb / csr_to_bsr / csr_to_ell arrays and
   interpret() outputs must match the oracle bit for bit, on integer AND real-valued data.
3. When oracle/_ref is built (this container), randomized oracle-vs-reference cases.
"""
import os

import numpy as np
import pytest

from oracle import port, ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


def example():
    # test_storage.cpp:18-25:  [[1,0,2,0],[0,0,0,3],[4,5,6,7],[0,0,0,0]]
    indptr = np.array([0, 2, 3, 7, 7], np.int32)
    indices = np.array([0, 2, 3, 0, 1, 2, 3], np.int32)
    values = np.arange(1, 8, dtype=np.float32)
    return 4, 4, indptr, indices, values


# ---- 1. reference KATs -------------------------------------------------------------------

def test_kat_hyb_buckets_example():
    # test_storage.cpp:122-134: hyb(1,2): bucket0 {row1}, bucket1 {row0}, bucket2 {row2}, pad 0
    parts, pr = port.hyb_decompose(*example(), 1, 2)
    assert [p["bucket"] for p in parts] == [0, 1, 2]
    assert [list(p["I_indices"]) for p in parts] == [[1], [0], [2]]
    assert pr == 0.0


def test_kat_hyb_split_example():
    # test_storage.cpp:136-146: hyb(1,1): row 2 (len 4) -> two bucket-1 segments; I = {0,2,2}
    parts, _ = port.hyb_decompose(*example(), 1, 1)
    b1 = [p for p in parts if p["bucket"] == 1][0]
    assert list(b1["I_indices"]) == [0, 2, 2]
    assert list(b1["J_indices"]) == [0, 2, 0, 1, 2, 3]


def test_kat_hyb_zero_matrix():
    # test_storage.cpp:148-154
    parts, pr = port.hyb_decompose(4, 4, np.zeros(5, np.int32), np.zeros(0, np.int32),
                                   np.zeros(0, np.float32), 2, 2)
    assert parts == [] and pr == 0.0


def test_kat_hyb_usage_error():
    with pytest.raises(port.OracleError) as e:
        port.hyb_decompose(*example(), 0, 2)
    assert e.value.code == 6  # ErrKind::Usage + 1


def test_kat_bsr_example():
    # test_storage.cpp:64-77
    jp, ji, bv = port.csr_to_bsr(*example(), 2)
    assert list(jp) == [0, 2, 4] and list(ji) == [0, 1, 0, 1]
    assert list(bv[:4]) == [1, 0, 0, 0] and bv[4] == 2 and bv[7] == 3


def test_kat_ell_example():
    # test_storage.cpp:95-120: w=2 fails naming row 2; w=4 pads with the last real column
    with pytest.raises(port.OracleError) as e:
        port.csr_to_ell(*example(), 2)
    assert e.value.code == 4 and "row 2" in str(e.value)
    J, V = port.csr_to_ell(*example(), 4)
    assert list(J[:4]) == [0, 2, 2, 2] and J[12] == 0 and J[15] == 0 and V[2] == 0


def test_kat_spmm_row_sums():
    # test_kernels.cpp:33-41: all-ones X -> row sums {3,3,22,0}
    rows, cols, ip, ix, v = example()
    Y = port.spmm_csr_refnum(rows, ip, ix, v, np.ones((4, 2), np.float32))
    assert Y[:, 0].tolist() == [3, 3, 22, 0]


def test_kat_auto_k():
    assert port.hyb_auto_k(0, 0) == 0
    assert port.hyb_auto_k(65536, 1048664) == 5   # C1
    assert port.hyb_auto_k(232965, 114615895) == 9
    assert port.hyb_auto_k(2449029, 61943588) == 5


# ---- 2. golden fixtures from the reference --------------------------------------------

def _case(G, name):
    rows, cols = (int(x) for x in G[f"{name}/shape"])
    return rows, cols, G[f"{name}/indptr"], G[f"{name}/indices"], G[f"{name}/values"]


def test_golden_hyb_arrays(G):
    n = 0
    for name in G["cases"]:
        rows, cols, ip, ix, v = _case(G, name)
        keys = sorted({k.rsplit("/", 1)[0] for k in G.files if k.startswith(f"{name}/hyb_") and k.endswith("/meta")})
        for key in keys:
            c, k = (int(t[1:]) for t in key.split("/")[-1].split("_")[1:])
            parts, pr = port.hyb_decompose(rows, cols, ip, ix, v, c, k)
            meta = G[key + "/meta"]
            assert len(parts) == meta.shape[0], key
            assert pr == float(G[key + "/padding"][0]), key
            for i, P in enumerate(parts):
                assert [P[f] for f in ("partition", "bucket", "width", "nrows", "nnz", "pad_slots",
                                       "col_lo", "col_hi")] == meta[i].tolist(), key
                assert np.array_equal(P["I_indices"], G[f"{key}/p{i}/I"]), key
                assert np.array_equal(P["J_indices"], G[f"{key}/p{i}/J"]), key
                assert np.array_equal(P["values"].view(np.uint32), G[f"{key}/p{i}/V"].view(np.uint32)), key
            n += 1
    assert n >= 40


def test_golden_spmm_bitexact(G):
    for name in G["cases"]:
        rows, cols, ip, ix, v = _case(G, name)
        for d in (8, 32):
            for tag in ("int", "real"):
                key = f"{name}/spmm_d{d}_{tag}"
                Y = port.spmm_csr_refnum(rows, ip, ix, v, G[key + "/X"])
                assert np.array_equal(Y.view(np.uint32), G[key + "/Y"].view(np.uint32)), key
                # hyb nest order gives the same bits
                parts, _ = port.hyb_decompose(rows, cols, ip, ix, v, 1, int(G[f"{name}/auto_k"][0]))
                Yh = port.spmm_hyb_refnum(rows, parts, G[key + "/X"])
                assert np.array_equal(Yh.view(np.uint32), Y.view(np.uint32)), key
                Y64 = port.spmm_csr_f64(rows, ip, ix, v, G[key + "/X"])
                assert np.array_equal(Y64, G[key + "/Y64"]), key


def test_golden_sddmm_bitexact(G):
    for name in G["cases"]:
        rows, cols, ip, ix, v = _case(G, name)
        for d in (8, 32):
            key = f"{name}/sddmm_d{d}"
            B = port.sddmm_csr_refnum(rows, cols, ip, ix, v, G[key + "/X"], G[key + "/Yd"])
            assert np.array_equal(B.view(np.uint32), G[key + "/B"].view(np.uint32)), key
            B64 = port.sddmm_csr_f64(rows, cols, ip, ix, v, G[key + "/X"], G[key + "/Yd"])
            assert np.array_equal(B64, G[key + "/B64"]), key


def test_golden_bsr(G):
    keys = sorted({k.rsplit("/", 1)[0] for k in G.files if k.startswith("bsr/")})
    for key in keys:
        rows, cols, prow, pcol, pad = (int(x) for x in G[key + "/shape"])
        b = int(key.rsplit("_b", 1)[1])
        ip, ix, v = G[key + "/csr_indptr"], G[key + "/csr_indices"], G[key + "/csr_values"]
        # driver.cpp:69-78 pads dims to multiples of b before build_csr
        assert prow % b == 0 and pcol % b == 0
        jp, ji, bv = port.csr_to_bsr(rows, cols, ip, ix, v, b)
        assert np.array_equal(jp, G[key + "/JO_indptr"]), key
        assert np.array_equal(ji, G[key + "/JO_indices"]), key
        assert np.array_equal(bv, G[key + "/values"]), key
        Y = port.bsr_spmm_refnum(prow // b, b, jp, ji, bv, G[key + "/X"])
        assert np.array_equal(Y, G[key + "/Y"]), key


def test_golden_rgms(G):
    R, m, n = (int(x) for x in G["rgms/shape"])
    for fmt in ("csr", "hyb"):
        Y = port.rgms_refnum(R, m, G["rgms/I_indptr"], G["rgms/I_indices"], G["rgms/J_indptr"],
                             G["rgms/J_indices"], G["rgms/A"], G[f"rgms/{fmt}/X"], G[f"rgms/{fmt}/W"])
        assert np.array_equal(Y, G[f"rgms/{fmt}/Y"]), fmt


def test_golden_ell(G):
    for name in ("example", "pl"):
        meta = G[f"ell/{name}/csr"]
        rows, cols, w = (int(x) for x in meta[:3])
        ip = meta[3:].astype(np.int32)
        J, V = port.csr_to_ell(rows, cols, ip, G[f"ell/{name}/indices"], G[f"ell/{name}/values"], w)
        assert np.array_equal(J, G[f"ell/{name}/J"]) and np.array_equal(V, G[f"ell/{name}/V"])


def test_generator_matches_reference_golden(G):
    """The product's generator (paper_2207_04606_b200, host C++) reproduces the reference's."""
    import paper_2207_04606_b200 as S
    m = S.generate_matrix("powerlaw", 600, 500, 0, 0, 0, 7.0, 11)
    rows, cols, ip, ix, v = _case(G, "powerlaw_600")
    assert (m.rows, m.cols) == (rows, cols)
    assert np.array_equal(m.indptr, ip) and np.array_equal(m.indices, ix)
    assert np.array_equal(m.values, v)
    for name, args in [("random_64", ("random", 64, 48, 0.2, 0, 0, 0, 5)),
                       ("banded_100", ("banded", 100, 100, 0, 3, 0, 0, 9)),
                       ("powerlaw_dense_rows", ("powerlaw", 300, 300, 0, 0, 0, 40.0, 2))]:
        m = S.generate_matrix(*args)
        rows, cols, ip, ix, v = _case(G, name)
        assert np.array_equal(m.indptr, ip) and np.array_equal(m.indices, ix), name
        assert np.array_equal(m.values, v), name
    dense = S.dense_int((500, 8), 17)
    assert np.array_equal(dense, G["powerlaw_600/spmm_d8_int/X"])


# ---- 3. randomized against the live reference (only where oracle/_ref is built) ---------

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built here")


@needs_ref
def test_random_hyb_vs_reference():
    rng = np.random.default_rng(7)
    for trial in range(30):
        n = int(rng.integers(1, 200))
        m = int(rng.integers(1, 200))
        coo = ref.Coo.generate("powerlaw", n, m, 0, 0, 0, float(rng.uniform(0.5, 30)), int(rng.integers(1, 1000)))
        st = ref.Storage.csr(coo)
        ip, ix, v = st.aux("J_indptr"), st.aux("J_indices"), st.values().astype(np.float32)
        c, k = int(rng.integers(1, 5)), int(rng.integers(0, 6))
        h = st.decompose_hyb(c, k)
        parts, pr = port.hyb_decompose(n, m, ip, ix, v, c, k)
        assert pr == h.padding_ratio
        assert len(parts) == len(h.parts)
        for a, b in zip(parts, h.parts):
            for f in ("I_indices", "J_indices", "values"):
                assert np.array_equal(a[f], b[f])


@needs_ref
def test_generator_c1_matches_reference():
    import paper_2207_04606_b200 as S
    mine = S.generate_matrix("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
    st = ref.Storage.csr(ref.Coo.generate("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1))
    assert mine.nnz == 1048664
    assert np.array_equal(mine.indptr, st.aux("J_indptr"))
    assert np.array_equal(mine.indices, st.aux("J_indices"))
    assert np.array_equal(mine.values, st.values().astype(np.float32))
    mine = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
    st = ref.Storage.csr(ref.Coo.generate("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1))
    assert mine.nnz == 1627136
    assert np.array_equal(mine.indices, st.aux("J_indices"))
    assert np.array_equal(mine.values, st.values().astype(np.float32))


def test_golden_dbsr_srbcrs(G):
    """The DBSR / SR-BCRS restatements (storage.cpp:336-440) against the reference library's
    arrays, and the reference pipeline's SpMM for both formats equal to the CSR SpMM restatement
    (integer operands: every format computes the same exact product)."""
    for name in ("example", "bs128", "pl"):
        meta = G[f"fmt/{name}/csr"]
        rows, cols = int(meta[0]), int(meta[1])
        ip, ix, v = meta[2:].astype(np.int32), G[f"fmt/{name}/indices"], G[f"fmt/{name}/values"]
        for b in (2, 32):
            key = f"dbsr/{name}_b{b}"
            io, jp, ji, bv = port.csr_to_dbsr(rows, cols, ip, ix, v, b)
            assert np.array_equal(io, G[key + "/IO_indices"]), key
            assert np.array_equal(jp, G[key + "/JO_indptr"]), key
            assert np.array_equal(ji, G[key + "/JO_indices"]), key
            assert np.array_equal(bv, G[key + "/values"]), key
        for t, g in ((2, 2), (3, 5), (8, 32)):
            key = f"srbcrs/{name}_t{t}_g{g}"
            gp, jt, sv = port.csr_to_srbcrs(rows, cols, ip, ix, v, t, g)
            assert np.array_equal(gp, G[key + "/G_indptr"]), key
            assert np.array_equal(jt, G[key + "/JT_indices"]), key
            assert np.array_equal(sv, G[key + "/values"]), key
        for fmt in ("dbsr", "srbcrs"):
            X = G[f"fmtspmm/{name}/{fmt}/X"]
            want = port.spmm_csr_refnum(rows, ip, ix, v, X[:cols])
            Y = G[f"fmtspmm/{name}/{fmt}/Y"]
            assert np.array_equal(Y[:rows], want) and not Y[rows:].any(), (name, fmt)
