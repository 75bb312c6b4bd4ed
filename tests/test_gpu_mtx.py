"""GPU: device Matrix Market ingest vs the linked reference read_matrix_market (mmio.cpp:17-55).

Triplets (row, col, f64 value, order) must equal the reference's bit for bit, errors must carry
the reference's kind and message (first failing line in file order), and the device CSR built
from the parsed triplets must equal the reference build_csr (storage.cpp:89-124, F32 values)."""
import numpy as np
import pytest
import torch

import paper_2207_04606_b200 as S
from oracle import ref
from mtx_cases import PREAMBLE_CASES, entry_cases, random_real_file

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _ref(text):
    try:
        return ("ok", ref.Coo.read_matrix_market(text))
    except ref.RefError as e:
        return ("err", e.code, str(e))


def _check(text):
    want = _ref(text)
    try:
        got = S.read_matrix_market(text)
    except S.StrataError as e:
        assert want[0] == "err", f"ours failed ({e}) where the reference parsed"
        assert (e.code, str(e)) == want[1:]
        return None
    assert want[0] == "ok", f"reference failed with {want[2]!r}, ours parsed"
    rc = want[1]
    assert (got.rows, got.cols, got.ntriplets) == (rc.rows, rc.cols, rc.nnz)
    gr, gc, gv = got.triplets()
    wr, wc, wv = rc.triplets()
    assert np.array_equal(gr, wr) and np.array_equal(gc, wc)
    # bitwise, -0.0 included
    assert np.array_equal(gv.view(np.int64), wv.view(np.int64)), \
        [(a, b) for a, b in zip(gv, wv) if a != b or np.signbit(a) != np.signbit(b)][:5]
    return got, rc


@pytest.mark.parametrize("name", sorted(entry_cases()))
def test_entry_cases(cuda, name):
    _check(entry_cases()[name])


@pytest.mark.parametrize("name", sorted(PREAMBLE_CASES))
def test_preamble_cases(cuda, name):
    _check(PREAMBLE_CASES[name])


@pytest.mark.parametrize("fmt", ["%.17g", "%.6e", "%.3f", "%r", "%.25g"])
@pytest.mark.parametrize("symmetric", [False, True])
def test_random_real_values_bitexact(cuda, fmt, symmetric):
    """Values spread over 10^-320 .. 10^300 (subnormals included) in several printf forms:
    decimal -> double must round exactly like strtod."""
    if fmt == "%r":
        text = random_real_file(500, 700, 20000, 3, "%s", symmetric)
    else:
        text = random_real_file(500, 700, 20000, 3, fmt, symmetric)
    _check(text)


def test_reference_writer_round_trip_and_csr(cuda):
    """write_matrix_market (mmio.cpp:63-72, precision 17) of the reference generator's C1 graph
    (1,048,664 entries), parsed on the device, then build_csr on the device."""
    coo = ref.Coo.generate("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
    r, c, v = coo.triplets()
    rng = np.random.default_rng(5)
    v = v * rng.standard_normal(v.size)  # real-valued, full 17-digit decimal strings
    real = ref.Coo.from_arrays(coo.rows, coo.cols, r, c, v)
    text = real.write_matrix_market()
    got, rc = _check(text)
    csr = got.to_csr(cuda)
    w_ptr, w_idx, w_val = _ref_csr(rc)
    assert np.array_equal(csr.indptr.cpu().numpy(), w_ptr)
    assert np.array_equal(csr.indices.cpu().numpy(), w_idx)
    assert np.array_equal(csr.values.cpu().numpy().view(np.int32), w_val.astype(np.float32).view(np.int32))


def _ref_csr(coo):
    st = ref.Storage.csr(coo)
    return st.aux("J_indptr"), st.aux("J_indices"), st.values()


def test_symmetric_then_csr_duplicate_error(cuda):
    """A symmetric file listing both (i, j) and (j, i) mirrors into a duplicate: build_csr's
    Validation error, the first duplicate in sorted order, like the reference."""
    text = (b"%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 1\n1 2 5\n3 3 1\n")
    m = _check(text)[0]
    with pytest.raises(S.StrataError) as e:
        m.to_csr(cuda)
    with pytest.raises(ref.RefError) as w:
        ref.Storage.csr(ref.Coo.read_matrix_market(text))
    assert (e.value.code, str(e.value)) == (w.value.code, str(w.value))


def test_read_file(cuda, tmp_path):
    text = random_real_file(50, 60, 3000, 9, "%.9g")
    p = tmp_path / "a.mtx"
    p.write_bytes(text)
    m = S.read_matrix_market_file(str(p))
    wr, wc, wv = ref.Coo.read_matrix_market(text).triplets()
    gr, gc, gv = m.triplets()
    assert np.array_equal(gr, wr) and np.array_equal(gc, wc) and np.array_equal(gv, wv)


def test_read_file_errors(cuda, tmp_path):
    """Empty and missing files give the reference's messages (mmio.cpp:21 / :59)."""
    p = tmp_path / "empty.mtx"
    p.write_bytes(b"")
    with pytest.raises(S.StrataError) as e:
        S.read_matrix_market_file(str(p))
    with pytest.raises(ref.RefError) as w:
        ref.Coo.read_matrix_market(b"")
    assert str(e.value) == str(w.value)
    with pytest.raises(S.StrataError) as e:
        S.read_matrix_market_file(str(tmp_path / "missing.mtx"))
    assert "cannot open" in str(e.value)


def test_large_text_staged_copy(cuda, tmp_path):
    """A text above the 128 MB staging threshold goes through the multi-threaded pinned ring
    (pageable bytes) and the mapped-file path: triplets equal the generated values, and the
    reference parser agrees on a prefix."""
    n = 9_000_000  # 18-byte lines: 162 MB
    r = np.random.default_rng(3)
    rows = r.integers(1, 10_000_000, n)
    cols = r.integers(1, 10_000_000, n)
    vals = r.integers(1, 10, n)
    lines = np.empty((n, 18), np.uint8)
    for k in range(7):
        p10 = 10 ** (6 - k)
        lines[:, k] = (rows // p10) % 10 + 48
        lines[:, 8 + k] = (cols // p10) % 10 + 48
    lines[:, 7] = lines[:, 15] = 32
    lines[:, 16] = vals + 48
    lines[:, 17] = 10
    text = (f"%%MatrixMarket matrix coordinate real general\n9999999 9999999 {n}\n".encode()
            + lines.tobytes())
    del lines
    for m in (S.read_matrix_market(text), None):
        if m is None:
            p = tmp_path / "big.mtx"
            p.write_bytes(text)
            m = S.read_matrix_market_file(str(p))
        gr, gc, gv = m.triplets()
        assert np.array_equal(gr, rows - 1) and np.array_equal(gc, cols - 1)
        assert np.array_equal(gv, vals.astype(np.float64))
    head = text[:text.index(b"\n", text.index(b"\n") + 1) + 1 + 18 * 1000]
    head = head.replace(f" {n}\n".encode(), b" 1000\n", 1)
    wr2, wc2, wv2 = ref.Coo.read_matrix_market(head).triplets()
    assert np.array_equal(gr[:1000], wr2) and np.array_equal(gc[:1000], wc2)
    assert np.array_equal(gv[:1000], wv2)
