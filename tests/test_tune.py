"""Format tuner (tune.hpp / tune.cpp): search-space enumeration on the CPU; device trials,
correctness gate, padding and row-work balance on the GPU."""
import json

import numpy as np
import pytest

import paper_2207_04606_b200 as S
from paper_2207_04606_b200 import tune as T
from oracle import port


def test_hyb_c_grid_enumeration():
    # tune.cpp:19-36: csr first, then c in {1,2,4,8,16}; k resolved per matrix unless fixed
    s = T.SearchSpace.hyb_c_grid()
    assert s.formats == ["csr", "hyb:c=1", "hyb:c=2", "hyb:c=4", "hyb:c=8", "hyb:c=16"]
    assert s.schedules == [""]
    s = T.SearchSpace.hyb_c_grid(k0=0, scan_k=True, include_csr=False)
    assert s.formats[:3] == ["hyb:c=1,k=0", "hyb:c=1,k=0", "hyb:c=1,k=1"]
    assert len(s.formats) == 15
    pts = T.enumerate_points(T.SearchSpace(["csr", "hyb:c=2"], ["", "x"]))
    assert [(p.id, p.format, p.schedule) for p in pts] == [
        (0, "csr", ""), (1, "csr", "x"), (2, "hyb:c=2", ""), (3, "hyb:c=2", "x")]
    assert [p.format for p in T.enumerate_points(T.SearchSpace())] == ["csr"]


def test_parse_format():
    m = S.CsrMatrix(4, 4, np.array([0, 2, 3, 7, 7], np.int32),
                    np.array([0, 2, 3, 0, 1, 2, 3], np.int32), np.ones(7, np.float32))
    assert T.parse_format("csr", m) == ("csr", None, None)
    assert T.parse_format("hyb:c=4,k=3", m) == ("hyb", 4, 3)
    assert T.parse_format("hyb", m) == ("hyb", 1, S.hyb_auto_k(m))
    with pytest.raises(S.StrataError):
        T.parse_format("dia", m)
    with pytest.raises(S.StrataError):
        T.parse_format("hyb:q=1", m)


def _balance_np(h):
    worst = 1.0
    for i, P in enumerate(h.parts):
        a = h.part_arrays(i)
        J = a[f"hyb_p{P.partition}_b{P.bucket}_J_indices"].reshape(P.nrows, P.width)
        real = 1 + (J[:, 1:] != J[:, :-1]).sum(axis=1) if P.width > 1 else np.ones(P.nrows)
        if P.nrows:
            worst = max(worst, real.max() / real.mean())
    return worst


@pytest.mark.gpu
def test_run_trials_c1(cuda):
    m = S.generate_matrix("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
    rep = T.run_trials("spmm", m, 32, T.SearchSpace.hyb_c_grid(), repeats=5, warmup=2,
                       flush_cache=True)
    assert len(rep.trials) == 6 and all(t.valid and t.correct for t in rep.trials)
    assert rep.trials[rep.best].median_ns == min(t.median_ns for t in rep.trials)
    j = json.loads(T.report_json(rep))
    assert j["best_point"] == rep.trials[rep.best].point.id
    assert sum(t["best"] for t in j["trials"]) == 1
    # padding and balance of a point equal an independent restatement on the readback
    for t in rep.trials[1:]:
        _, c, k = T.parse_format(t.point.format, m)
        _, pr = port.hyb_decompose(m.rows, m.cols, m.indptr, m.indices, m.values, c, k)
        assert t.padding == pr
    h = S.decompose_hyb(m.to_device(cuda), 2, S.hyb_auto_k(m))
    assert abs(rep.trials[2].balance - _balance_np(h)) < 1e-12


@pytest.mark.gpu
def test_run_trials_gate_and_errors(cuda):
    m = S.generate_matrix("powerlaw", 3000, 3000, 0, 0, 0, 8.0, 3)
    with pytest.raises(S.StrataError):
        T.run_trials("spmm", m, 16, T.SearchSpace(["dia"]), repeats=1, warmup=0)
    with pytest.raises(S.StrataError):
        T.run_trials("sddmm", m, 16, T.SearchSpace.hyb_c_grid(), repeats=1, warmup=0)
    rep = T.run_trials("spmm", m, 16, T.SearchSpace(["hyb:c=3,k=2", "dia"]), repeats=2, warmup=0)
    assert rep.trials[0].valid and rep.trials[0].correct and not rep.trials[1].valid
