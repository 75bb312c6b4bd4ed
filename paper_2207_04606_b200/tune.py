"""Format tuner: the reference's grid search over hyb(c, k) (tune.hpp / tune.cpp) on the device.

Mirrors proj/include/strata/tune.hpp:
  SearchSpace.hyb_c_grid(k0=-1, scan_k=False, include_csr=True)   tune.cpp:19-36
  enumerate(space)                                                 tune.cpp:38-48
  run_trials(op, m, d, space, repeats, warmup, flush_cache, seed)  tune.cpp:100-165
  report_json(report)                                              tune.cpp:167-190

Differences that follow from running on the GPU (same selection rule: the lowest median among
points that pass the correctness gate):
  * conversion (decompose_hyb) runs untimed, like the reference's ``preconverted`` option;
  * each run is timed with CUDA events on the stream (median over ``repeats`` after ``warmup``);
    ``flush_cache`` writes a buffer larger than L2 between runs (thrash_cache, tune.cpp:78-86);
  * the correctness gate compares every point with the CSR format's result on the reference's
    integer operand (mt19937(seed) uniform_int(-3, 3), tune.cpp:108-111): every partial sum is
    an exact integer in f32, so all correct formats agree bitwise.  (The reference gates
    against its dense oracle; the dense m x n oracle is not formed on the device.)
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

import ctypes as C

from ._lib import StrataError, check, lib
from . import ops

__all__ = ["SearchSpace", "SearchPoint", "TrialResult", "TuneReport", "enumerate_points",
           "run_trials", "report_json", "parse_format"]


@dataclass
class SearchSpace:
    formats: list = field(default_factory=list)
    schedules: list = field(default_factory=list)

    @staticmethod
    def hyb_c_grid(k0: int = -1, scan_k: bool = False, include_csr: bool = True) -> "SearchSpace":
        """c over {1, 2, 4, 8, 16}; k fixed (k0 >= 0), scanned k0 +/- 1, or resolved per matrix
        (hyb_auto_k); plus the untuned CSR baseline (tune.cpp:19-36)."""
        s = SearchSpace()
        if include_csr:
            s.formats.append("csr")
        for c in (1, 2, 4, 8, 16):
            if scan_k and k0 >= 0:
                for off in (-1, 0, 1):
                    s.formats.append(f"hyb:c={c},k={max(0, k0 + off)}")
            elif k0 >= 0:
                s.formats.append(f"hyb:c={c},k={k0}")
            else:
                s.formats.append(f"hyb:c={c}")
        s.schedules.append("")
        return s


@dataclass
class SearchPoint:
    id: int
    format: str
    schedule: str = ""


@dataclass
class TrialResult:
    point: SearchPoint
    median_ns: float = 0.0
    flops: int = 0
    loads: int = 0
    valid: bool = False
    correct: bool = False
    padding: float = 0.0
    balance: float = 1.0
    error: str = ""


@dataclass
class TuneReport:
    trials: list = field(default_factory=list)
    best: int = -1


def enumerate_points(space: SearchSpace) -> list:
    formats = space.formats or ["csr"]
    schedules = space.schedules or [""]
    out, i = [], 0
    for f in formats:
        for sc in schedules:
            out.append(SearchPoint(i, f, sc))
            i += 1
    return out


def parse_format(fmt: str, m) -> tuple:
    """FormatRequest::parse subset for the SpMM tuner: "csr" | "hyb[:c=C][,k=K]"."""
    fmt = fmt.strip()
    if fmt == "csr":
        return ("csr", None, None)
    if not fmt.startswith("hyb"):
        raise StrataError(6, f"tuner: unsupported format '{fmt}'")
    c, k = 1, -1
    if ":" in fmt:
        for kv in fmt.split(":", 1)[1].split(","):
            key, _, val = kv.partition("=")
            if key.strip() == "c":
                c = int(val)
            elif key.strip() == "k":
                k = int(val)
            else:
                raise StrataError(6, f"unknown format option '{key}'")
    if k < 0:
        k = ops.hyb_auto_k(m)
    return ("hyb", c, k)


def run_trials(op: str, m, d: int, space: SearchSpace, repeats: int = 100, warmup: int = 10,
               flush_cache: bool = False, seed: int = 1, device="cuda") -> TuneReport:
    """Time every point of ``space`` for ``op`` ("spmm") on host CSR ``m`` with d features."""
    import torch
    if repeats < 1:
        raise StrataError(6, "repeats must be >= 1")
    if op != "spmm":
        raise StrataError(6, f"tuner: op '{op}' has a single format on the device path")
    dev = torch.device(device)
    stream = torch.cuda.current_stream(dev)
    X = torch.from_numpy(ops.dense_int((m.cols, d), seed)).to(dev)
    dcsr = m.to_device(dev)
    Yref = ops.spmm_csr(dcsr, X)  # gate: integer operands -> every correct format is bitwise equal
    junk = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_cache else None
    report = TuneReport()
    for pt in enumerate_points(space):
        tr = TrialResult(pt)
        try:
            kind, c, k = parse_format(pt.format, m)
            if kind == "csr":
                fn = lambda Y: ops.spmm_csr(dcsr, X, Y)  # noqa: E731
                tr.flops = 2 * m.nnz * d
            else:
                h = ops.decompose_hyb(dcsr, c, k)
                tr.padding = h.padding_ratio
                bal = C.c_double()
                check(lib.strata_hyb_row_work_balance(h.handle, C.byref(bal), stream.cuda_stream))
                tr.balance = bal.value
                slots = h.schedule_info()["slots"]
                tr.flops = 2 * slots * d  # pads are multiplied, as the reference's stage III
                fn = lambda Y, h=h: ops.spmm(h, X, Y)  # noqa: E731
            Y = torch.empty_like(Yref)
            fn(Y)
            tr.correct = bool(torch.equal(Y, Yref))
            if not tr.correct:
                tr.error = "result differs from the CSR format on integer operands"
            tr.loads = tr.flops // 2
            samples = []
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for rep in range(warmup + repeats):
                if junk is not None:
                    junk.add_(1)
                e0.record(stream)
                fn(Y)
                e1.record(stream)
                e1.synchronize()
                if rep >= warmup:
                    samples.append(e0.elapsed_time(e1) * 1e6)
            samples.sort()
            tr.median_ns = samples[len(samples) // 2]
            tr.valid = True
        except StrataError as e:
            tr.valid = False
            tr.error = str(e)
        report.trials.append(tr)
    for i, tr in enumerate(report.trials):
        if tr.valid and tr.correct and (report.best < 0 or
                                        tr.median_ns < report.trials[report.best].median_ns):
            report.best = i
    if report.best < 0:
        raise StrataError(6, "tuner: no valid point in the search space")
    return report


def report_json(report: TuneReport) -> str:
    """Same fields as tune.cpp:167-190."""
    trials = []
    for i, tr in enumerate(report.trials):
        t = {"point": tr.point.id, "params": {"format": tr.point.format, "schedule": tr.point.schedule},
             "median_ns": tr.median_ns, "flops": tr.flops, "loads": tr.loads, "valid": tr.valid,
             "correct": tr.correct, "padding_ratio": tr.padding, "row_work_balance": tr.balance,
             "best": i == report.best}
        if tr.error:
            t["error"] = tr.error
        trials.append(t)
    best = report.trials[report.best].point.id if report.best >= 0 else -1
    return json.dumps({"trials": trials, "best_point": best}, indent=2)
