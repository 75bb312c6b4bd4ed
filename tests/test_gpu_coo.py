"""GPU: device build_csr (storage.cpp:89-124) from COO triplets — bit-exact CSR, and the
reference's Validation errors (out of range first, then the first duplicate in sorted order)."""
import numpy as np
import pytest
import torch

import paper_2207_04606_b200 as S

pytestmark = pytest.mark.gpu


def _coo_of(m, rng):
    rows = np.repeat(np.arange(m.rows, dtype=np.int32), np.diff(m.indptr))
    perm = rng.permutation(m.nnz)
    return rows[perm], m.indices[perm], m.values[perm]


@pytest.mark.parametrize("shape", [(65536, 65536, 16.0), (3000, 2000, 3.0), (1, 1, 1.0)])
def test_build_csr_device_matches_generator_csr(cuda, shape):
    n, c, avg = shape
    m = S.generate_matrix("powerlaw", n, c, 0, 0, 0, avg, 3)
    r, col, v = _coo_of(m, np.random.default_rng(0))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    d = S.build_csr_device(m.rows, m.cols, t(r), t(col), t(v))
    assert np.array_equal(d.indptr.cpu().numpy(), m.indptr)
    assert np.array_equal(d.indices.cpu().numpy(), m.indices)
    assert np.array_equal(d.values.cpu().numpy(), m.values)


def test_build_csr_device_errors(cuda):
    t = lambda a, dt=np.int32: torch.from_numpy(np.array(a, dt)).to(cuda)
    # the example matrix of test_storage.cpp:30-36 with a duplicated (2, 1) and (0, 2)
    rows, cols = [2, 0, 1, 2, 0, 2, 2, 0], [1, 0, 3, 0, 2, 2, 1, 2]
    with pytest.raises(S.StrataError) as e:
        S.build_csr_device(4, 4, t(rows), t(cols), t(np.ones(8), np.float32))
    assert e.value.kind == "Validation" and str(e.value) == "duplicate coordinate (0, 2)"
    with pytest.raises(S.StrataError) as e:
        S.build_csr_device(4, 4, t([0, 4]), t([0, 0]), t(np.ones(2), np.float32))
    assert e.value.kind == "Validation" and str(e.value) == "coordinate out of range"
    with pytest.raises(S.StrataError) as e:  # range is checked before duplicates
        S.build_csr_device(4, 4, t([0, 0, 9]), t([1, 1, 0]), t(np.ones(3), np.float32))
    assert str(e.value) == "coordinate out of range"
    d = S.build_csr_device(5, 3, t([]), t([]), t([], np.float32))
    assert np.array_equal(d.indptr.cpu().numpy(), np.zeros(6, np.int32)) and d.nnz == 0
