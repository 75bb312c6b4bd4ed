"""Python mirror of the reference operator API for the hot path (host side of the C ABI).

Names, argument meaning and error behaviour follow proj/include/strata (paths relative to
/root/reference/proj):

  generate_matrix   driver.hpp:84-85   (+ build_csr storage.hpp:111, emitted as CSR directly)
  decompose_hyb     storage.hpp:131-132   -> HybDecomposition (parts, padding_ratio)
  hyb_rules         transform.hpp:102-103 (rule / binding names, Appendix C of SURVEY.md)
  hyb_auto_k        storage.hpp:173
  csr_to_bsr        storage.hpp:117
  csr_to_ell        storage.hpp:124
  spmm / sddmm / bsr_spmm / rgms: the four canonical pipelines' run step
                    (driver.cpp:163-217, :241-314 + interp.cpp:564-622)

Device memory, streams and dtype plumbing come from PyTorch; every computation goes through
libstrata_b200.so.  A StrataError carries the reference ErrKind name in ``.kind``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import StrataError, check, lib

__all__ = [
    "StrataError", "CsrMatrix", "generate_matrix", "dense_int", "hyb_auto_k", "EllBucketPart",
    "HybDecomposition", "decompose_hyb", "hyb_rules", "spmm", "spmm_host", "spmm_csr", "sddmm",
    "partition_rows", "device_ok",
]


def device_ok() -> bool:
    return bool(lib.strata_device_ok())


def _ptr(t) -> int:
    """Raw pointer of a torch tensor or numpy array (0 for None)."""
    if t is None:
        return 0
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class CsrMatrix:
    """Host CSR with f32 values: the TensorStorage that build_csr returns (kind=Csr)."""
    rows: int
    cols: int
    indptr: np.ndarray   # int32 [rows+1]   aux "J_indptr"
    indices: np.ndarray  # int32 [nnz]      aux "J_indices"
    values: np.ndarray   # float32 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    def to_device(self, device="cuda"):
        import torch
        return DeviceCsr(self.rows, self.cols,
                         torch.from_numpy(self.indptr).to(device),
                         torch.from_numpy(self.indices).to(device),
                         torch.from_numpy(self.values).to(device))

    def row_slice(self, r0: int, r1: int) -> "CsrMatrix":
        """Rows [r0, r1) as a (r1-r0) x cols CSR (the row-shard of a multi-GPU run)."""
        q0, q1 = int(self.indptr[r0]), int(self.indptr[r1])
        return CsrMatrix(r1 - r0, self.cols, (self.indptr[r0:r1 + 1] - q0).astype(np.int32),
                         self.indices[q0:q1].copy(), self.values[q0:q1].copy())


@dataclass
class DeviceCsr:
    rows: int
    cols: int
    indptr: object
    indices: object
    values: object

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])


def generate_matrix(kind: str, n: int, m: int, density: float = 0.0, band: int = 0,
                    block: int = 0, avg_degree: float = 0.0, seed: int = 1) -> CsrMatrix:
    """generate_matrix(...) followed by build_csr with F32 values — same graph as the reference."""
    h = C.c_void_p()
    check(lib.strata_generate_csr(kind.encode(), n, m, density, band, block, avg_degree, seed,
                                  C.byref(h)))
    try:
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.strata_csr_host_info(h, C.byref(r), C.byref(c), C.byref(z)))
        nnz = z.value
        indptr = np.empty(r.value + 1, np.int32)
        indices = np.empty(nnz, np.int32)
        values = np.empty(nnz, np.float32)
        C.memmove(indptr.ctypes.data, lib.strata_csr_host_indptr(h), indptr.nbytes)
        if nnz:
            C.memmove(indices.ctypes.data, lib.strata_csr_host_indices(h), indices.nbytes)
            C.memmove(values.ctypes.data, lib.strata_csr_host_values(h), values.nbytes)
        return CsrMatrix(r.value, c.value, indptr, indices, values)
    finally:
        lib.strata_csr_host_destroy(h)


def dense_int(shape, seed: int) -> np.ndarray:
    """mt19937(seed) uniform_int(-3, 3) row-major operand (tune.cpp:108-111)."""
    out = np.empty(int(np.prod(shape)), np.float32)
    check(lib.strata_dense_int(out.size, seed, out.ctypes.data))
    return out.reshape(shape)


def hyb_auto_k(csr) -> int:
    return int(lib.strata_hyb_auto_k(csr.rows, csr.nnz))


@dataclass
class EllBucketPart:
    """storage.hpp:84-91 (+ the ELL storage's nnz / pad_slots)."""
    partition: int
    bucket: int
    width: int
    col_lo: int
    col_hi: int
    nrows: int
    nnz: int
    pad_slots: int
    prefix: str = ""

    @property
    def names(self) -> dict:
        pre = f"{self.prefix}hyb_p{self.partition}_b{self.bucket}_"
        return {"I_indptr": pre + "I_indptr", "I_indices": pre + "I_indices",
                "J_indices": pre + "J_indices"}


class HybDecomposition:
    """Device-resident hyb(c, k) decomposition; mirrors storage.hpp:92-106."""

    def __init__(self, handle: C.c_void_p, prefix: str = ""):
        self._h = handle
        r, c_, cc, kk = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        check(lib.strata_hyb_dims(handle, C.byref(r), C.byref(c_), C.byref(cc), C.byref(kk)))
        self.rows, self.cols, self.c, self.k = r.value, c_.value, cc.value, kk.value
        pr = C.c_double()
        check(lib.strata_hyb_padding_ratio(handle, C.byref(pr)))
        self.padding_ratio = pr.value
        n = C.c_int()
        check(lib.strata_hyb_num_parts(handle, C.byref(n)))
        self.parts = []
        for i in range(n.value):
            p, b = C.c_int(), C.c_int()
            w, nr, nz, pad, lo, hi = (C.c_int64() for _ in range(6))
            check(lib.strata_hyb_part_info(handle, i, C.byref(p), C.byref(b), C.byref(w),
                                           C.byref(nr), C.byref(nz), C.byref(pad), C.byref(lo),
                                           C.byref(hi)))
            self.parts.append(EllBucketPart(p.value, b.value, w.value, lo.value, hi.value,
                                            nr.value, nz.value, pad.value, prefix))

    @property
    def handle(self):
        return self._h

    def schedule_info(self) -> dict:
        v = [C.c_int64() for _ in range(4)]
        n = C.c_int()
        check(lib.strata_hyb_schedule_info(self._h, *(C.byref(x) for x in v), C.byref(n)))
        return dict(slots=v[0].value, chunks=v[1].value, crossing_runs=v[2].value,
                    empty_rows=v[3].value, launches_per_spmm=n.value)

    def part_arrays(self, i: int) -> dict:
        """Bit-exact host readback of part i under the reference's aux-array names."""
        P = self.parts[i]
        iptr = np.empty(2, np.int32)
        ii = np.empty(P.nrows, np.int32)
        jj = np.empty(P.nrows * P.width, np.int32)
        vv = np.empty(P.nrows * P.width, np.float32)
        check(lib.strata_hyb_part_read(self._h, i, iptr.ctypes.data, ii.ctypes.data,
                                       jj.ctypes.data, vv.ctypes.data))
        n = P.names
        return {n["I_indptr"]: iptr, n["I_indices"]: ii, n["J_indices"]: jj, "values": vv}

    def close(self):
        if self._h:
            lib.strata_hyb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decompose_hyb(csr: DeviceCsr, c: int, k: int, prefix: str = "", stream=None) -> HybDecomposition:
    h = C.c_void_p()
    check(lib.strata_hyb_decompose(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values),
                                   csr.rows, csr.cols, csr.nnz, c, k, _stream(stream), C.byref(h)))
    return HybDecomposition(h, prefix)


def hyb_rules(csr: DeviceCsr, c: int, k: int, name: str = "hyb"):
    """transform.cpp:525-557: c*(k+1) rules (empty buckets included) with the reference's names.

    Returns a list of dicts {name, new_buffer, arrays: {aux name: size}, nvalues}; non-empty
    rules carry the device decomposition part index in ``part``."""
    h = decompose_hyb(csr, c, k, prefix=name + "_")
    by_pb = {(P.partition, P.bucket): i for i, P in enumerate(h.parts)}
    rules = []
    for p in range(c):
        for b in range(k + 1):
            rname = f"{name}_p{p}_b{b}"
            pre = f"{name}_hyb_p{p}_b{b}_"
            i = by_pb.get((p, b))
            nrows = h.parts[i].nrows if i is not None else 0
            rules.append({"name": rname, "new_buffer": "A_" + rname, "part": i,
                          "arrays": {pre + "I_indptr": 2, pre + "I_indices": nrows,
                                     pre + "J_indices": nrows * (1 << b)},
                          "nvalues": nrows * (1 << b)})
    return h, rules


def spmm(hyb: HybDecomposition, X, Y=None, stream=None):
    """Y = A @ X over the hyb decomposition (device tensors, f32).  Y is overwritten."""
    import torch
    d = X.shape[1]
    if Y is None:
        Y = torch.empty((hyb.rows, d), dtype=torch.float32, device=X.device)
    check(lib.strata_spmm_hyb_f32(hyb.handle, _ptr(X), _ptr(Y), d, _stream(stream)))
    return Y


def spmm_host(hyb: HybDecomposition, X_host, Y_host, stream=None):
    """End-to-end form: host (pinned) X in, host Y out, copies inside the call."""
    d = X_host.shape[1]
    check(lib.strata_spmm_hyb_f32_host(hyb.handle, _ptr(X_host), _ptr(Y_host), d,
                                       _stream(stream)))
    return Y_host


def spmm_csr(csr: DeviceCsr, X, Y=None, stream=None):
    import torch
    d = X.shape[1]
    if Y is None:
        Y = torch.empty((csr.rows, d), dtype=torch.float32, device=X.device)
    check(lib.strata_spmm_csr_f32(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values), _ptr(X),
                                  _ptr(Y), csr.rows, csr.cols, d, _stream(stream)))
    return Y


def sddmm(csr: DeviceCsr, X, Yt_dn, B=None, stream=None):
    """B[nnz] = A .* (X @ Y) on the pattern; X [rows][d], Y [d][cols] (reference layout)."""
    import torch
    d = X.shape[1]
    if B is None:
        B = torch.empty((csr.nnz,), dtype=torch.float32, device=X.device)
    check(lib.strata_sddmm_csr_f32(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values), _ptr(X),
                                   _ptr(Yt_dn), _ptr(B), csr.rows, csr.cols, csr.nnz, d,
                                   _stream(stream)))
    return B


def partition_rows(indptr: np.ndarray, parts: int) -> np.ndarray:
    """nnz-balanced contiguous row ranges (bounds[parts+1]) for the row-sharded multi-GPU path."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int32)
    bounds = np.empty(parts + 1, np.int64)
    check(lib.strata_partition_rows(indptr.ctypes.data, indptr.shape[0] - 1, parts,
                                    bounds.ctypes.data))
    return bounds
