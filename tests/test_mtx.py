"""CPU: the Matrix Market preamble (banner, comments, size line; mmio.cpp:17-38) is read on the
host, so its errors and empty matrices are checked here against the linked reference
read_matrix_market; the entry lines are parsed on the device (tests/test_gpu_mtx.py)."""
import os

import pytest

import paper_2207_04606_b200 as S
from oracle import ref
from mtx_cases import PREAMBLE_CASES

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _ref(text):
    try:
        c = ref.Coo.read_matrix_market(text)
        return ("ok", c.rows, c.cols, c.nnz)
    except ref.RefError as e:
        return ("err", e.code, str(e))


def _ours(text):
    try:
        m = S.read_matrix_market(text)
        return ("ok", m.rows, m.cols, m.ntriplets)
    except S.StrataError as e:
        return ("err", e.code, str(e))


@needs_ref
@pytest.mark.parametrize("name", sorted(PREAMBLE_CASES))
def test_preamble_matches_reference(name):
    text = PREAMBLE_CASES[name]
    assert _ours(text) == _ref(text), name


def test_read_file_errors(tmp_path):
    with pytest.raises(S.StrataError) as e:
        S.read_matrix_market_file(str(tmp_path / "missing.mtx"))
    assert e.value.kind == "Usage" and str(e.value) == f"cannot open {tmp_path / 'missing.mtx'}"
    p = tmp_path / "hdr.mtx"
    p.write_bytes(PREAMBLE_CASES["bad_size"])
    with pytest.raises(S.StrataError) as e:
        S.read_matrix_market_file(str(p))
    assert str(e.value) == "bad matrix market size line"
    p.write_bytes(PREAMBLE_CASES["zero_nnz"])
    m = S.read_matrix_market_file(str(p))
    assert (m.rows, m.cols, m.ntriplets) == (7, 3, 0)
