"""CPU suite: the C-ABI library loads, exports every symbol include/strata_b200.h declares, and
its host-only logic (argument validation, error convention, partitioning) behaves like the
reference's.  No compute call is made without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "strata_b200.h")).read()
    return sorted(set(re.findall(r"\b(strata_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2207_04606_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert sorted(_lib.EXPORTED) == syms


def test_abi_version_and_error_convention():
    from paper_2207_04606_b200 import _lib
    assert _lib.lib.strata_abi_version() >= 100
    h = C.c_void_p()
    # storage.cpp:273 -> ErrKind::Usage, raised before any device work (like the reference)
    rc = _lib.lib.strata_hyb_decompose(None, None, None, 4, 4, 0, 0, 2, None, C.byref(h))
    assert rc == 6 and b"c >= 1" in _lib.lib.strata_last_error()
    rc = _lib.lib.strata_hyb_decompose(None, None, None, 4, 4, 0, 1, -1, None, C.byref(h))
    assert rc == 6


def test_no_silent_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2207_04606_b200 as S
    assert not S.device_ok()
    from paper_2207_04606_b200 import _lib
    h = C.c_void_p()
    ip = np.array([0, 1], np.int32)
    rc = _lib.lib.strata_hyb_decompose(ip.ctypes.data, ip.ctypes.data, ip.ctypes.data, 1, 1, 1, 1,
                                       0, None, C.byref(h))
    assert rc == 9  # STRATA_ERR_CUDA: fails loudly, never computes on the host


def test_hyb_auto_k_matches_reference_rule():
    import paper_2207_04606_b200 as S
    from oracle import port
    for rows, nnz in [(0, 0), (5, 0), (4, 7), (65536, 1048664), (232965, 114615895),
                      (2449029, 61943588), (10, 1000), (3, 3)]:
        assert S.ops.lib.strata_hyb_auto_k(rows, nnz) == port.hyb_auto_k(rows, nnz)


def test_partition_rows_balanced_by_nnz():
    import paper_2207_04606_b200 as S
    m = S.generate_matrix("powerlaw", 20000, 20000, 0, 0, 0, 12.0, 3)
    for parts in (1, 2, 3, 4, 8):
        b = S.partition_rows(m.indptr, parts)
        assert b[0] == 0 and b[-1] == m.rows and np.all(np.diff(b) >= 0)
        for p in range(1, parts):
            # cut p is the first row whose indptr reaches nnz*p/parts
            target = (m.nnz * p) // parts
            assert m.indptr[b[p]] >= target
            assert b[p] == 0 or m.indptr[b[p] - 1] < target


def test_python_binding_checks_reject_bad_operands():
    """ops.py checks shape / dtype / layout / device before a raw pointer crosses the C ABI,
    with the reference's ErrKind::Exec wording (interp.cpp:576-582)."""
    import torch
    from paper_2207_04606_b200 import ops
    X = torch.zeros(4, 8)
    with pytest.raises(ops.StrataError) as e:          # host tensor where device memory is due
        ops._dense(X, "X", (4, 8), "f32")
    assert e.value.kind == "Exec"
    with pytest.raises(ops.StrataError) as e:
        ops._dense(X, "X", (5, 8), "f32")
    assert "binding size mismatch for X: got 32" in str(e.value)
    with pytest.raises(ops.StrataError) as e:
        ops._dense(X.to(torch.float64), "X", (4, 8), "f32")
    assert "dtype mismatch" in str(e.value)
    with pytest.raises(ops.StrataError) as e:
        ops._dense(X.t(), "X", (8, 4), "f32")
    assert "contiguous" in str(e.value)
    ops._host(X, "X", (4, 8))
    with pytest.raises(ops.StrataError):
        ops._host(X, "X", (4, 9))
