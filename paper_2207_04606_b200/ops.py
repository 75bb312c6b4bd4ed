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
    "StrataError", "CsrMatrix", "build_csr_device", "generate_matrix", "dense_int", "hyb_auto_k", "EllBucketPart",
    "HybDecomposition", "decompose_hyb", "hyb_rules", "spmm", "spmm_host", "spmm_host_batch",
    "spmm_multi", "ipc_handle", "ipc_open", "ipc_close",
    "spmm_csr", "sddmm", "gnn_layer", "gnn_layer_work_floats", "gemm",
    "partition_rows", "device_ok", "MatrixMarket", "read_matrix_market",
    "read_matrix_market_file",
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


def _dense(t, name: str, shape, dtype: str, device=None):
    """Binding check of a dense device operand before its raw pointer crosses the C ABI (which
    cannot see shapes): the reference's interpret() rejects a wrongly sized binding with
    ErrKind::Exec "binding size mismatch for <name>: got <n>, declared <m>" (interp.cpp:576-582);
    dtype, layout (row-major contiguous) and device are checked the same way."""
    import torch
    want = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32}[dtype]
    if not isinstance(t, torch.Tensor):
        raise StrataError(7, f"binding for {name} must be a torch tensor")
    got_n, want_n = int(t.numel()), int(np.prod(shape))
    if tuple(t.shape) != tuple(shape):
        raise StrataError(7, f"binding size mismatch for {name}: got {got_n} "
                             f"{list(t.shape)}, declared {want_n} {list(shape)}")
    if t.dtype != want:
        raise StrataError(7, f"binding dtype mismatch for {name}: got {t.dtype}, declared {dtype}")
    if not t.is_contiguous():
        raise StrataError(7, f"binding for {name} must be row-major contiguous")
    if t.device.type != "cuda" or (device is not None and t.device != device):
        raise StrataError(7, f"binding for {name} is on {t.device}, expected "
                             f"{device if device is not None else 'a CUDA device'}")
    return t


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _stream_if_device(stream=None) -> int:
    """The caller's stream, or the legacy default stream where no device is visible (host-only
    errors of an ingest call can still be reported then)."""
    import torch
    if stream is None and not torch.cuda.is_available():
        return 0
    return _stream(stream)


@dataclass
class CsrMatrix:
    """Host CSR with f32 values: the TensorStorage that build_csr returns (kind=Csr)."""
    rows: int
    cols: int
    indptr: np.ndarray   # int32 [rows+1]   aux "J_indptr"
    indices: np.ndarray  # int32 [nnz]      aux "J_indices"
    values: np.ndarray   # float32 [nnz]
    row_order: np.ndarray = None  # powerlaw generator's triplet row order (see split_relations)

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


def build_csr_device(rows: int, cols: int, row, col, val, stream=None) -> "DeviceCsr":
    """build_csr (storage.cpp:89-124) on the device: COO triplets (device int32 row / col, f32
    val) -> DeviceCsr sorted by (row, col); StrataError(kind='Validation') on out-of-range or
    duplicate coordinates with the reference's messages."""
    import torch
    dev = row.device
    nnz = int(row.shape[0])
    indptr = torch.empty(rows + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    values = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    check(lib.strata_csr_from_coo(_ptr(row), _ptr(col), _ptr(val), nnz, rows, cols, _ptr(indptr),
                                  _ptr(indices), _ptr(values), _stream(stream)))
    return DeviceCsr(rows, cols, indptr, indices[:nnz], values[:nnz])


class MatrixMarket:
    """Device COO parsed from a Matrix Market file: the reference CooMatrix (storage.hpp:45-54)
    that read_matrix_market returns, with its triplets in the reference's order (symmetric
    files: the mirrored entry right after its off-diagonal entry, mmio.cpp:50-51) resident in
    HBM as int32 row / col, f64 value and its f32 rounding."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.strata_mtx_info(handle, C.byref(r), C.byref(c), C.byref(z)))
        self.rows, self.cols, self.ntriplets = r.value, c.value, z.value

    def triplets(self):
        """Host copy (row int64, col int64, value float64) of CooMatrix.triplets."""
        n = self.ntriplets
        r, c, v = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.float64)
        check(lib.strata_mtx_read(self._h, r.ctypes.data, c.ctypes.data, v.ctypes.data))
        return r, c, v

    def to_csr(self, device="cuda", stream=None) -> "DeviceCsr":
        """build_csr (storage.cpp:89-124) of the parsed triplets, on the device (F32 values)."""
        import torch
        rp, cp, v64, v32 = (C.c_void_p() for _ in range(4))
        check(lib.strata_mtx_device(self._h, C.byref(rp), C.byref(cp), C.byref(v64), C.byref(v32)))
        nnz = self.ntriplets
        indptr = torch.empty(self.rows + 1, dtype=torch.int32, device=device)
        indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
        values = torch.empty(max(nnz, 1), dtype=torch.float32, device=device)
        check(lib.strata_csr_from_coo(rp.value or 0, cp.value or 0, v32.value or 0, nnz, self.rows,
                                      self.cols, _ptr(indptr), _ptr(indices), _ptr(values),
                                      _stream(stream)))
        return DeviceCsr(self.rows, self.cols, indptr, indices[:nnz], values[:nnz])

    def close(self):
        if self._h:
            lib.strata_mtx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_matrix_market(text, stream=None) -> MatrixMarket:
    """read_matrix_market(std::istream&) (mmio.hpp:22, mmio.cpp:17-55): the stream's bytes
    (bytes or str) parsed on the device.  StrataError(kind='Usage') with the reference's
    messages."""
    if isinstance(text, str):
        text = text.encode()
    # zero-copy view of any contiguous byte buffer (bytes, bytearray, memoryview, mmap, uint8
    # array): the C ABI reads it in place (a ctypes string-buffer copy of a 1.1 GB text cost
    # ~0.5 s, five times the H2D copy itself)
    buf = np.frombuffer(text, np.uint8)
    h = C.c_void_p()
    check(lib.strata_mtx_parse(buf.ctypes.data if buf.size else None, buf.size, C.byref(h),
                               _stream_if_device(stream)))
    return MatrixMarket(h)


def read_matrix_market_file(path: str, stream=None) -> MatrixMarket:
    """read_matrix_market_file(path) (mmio.hpp:23, mmio.cpp:57-61)."""
    h = C.c_void_p()
    check(lib.strata_mtx_read_file(str(path).encode(), C.byref(h), _stream_if_device(stream)))
    return MatrixMarket(h)


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
        order = None
        if kind == "powerlaw":
            order = np.empty(r.value, np.int32)
            check(lib.strata_csr_host_row_order(h, order.ctypes.data))
        return CsrMatrix(r.value, c.value, indptr, indices, values, order)
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
    if getattr(X, "dim", lambda: 0)() != 2:
        raise StrataError(7, "binding for X must be a [cols][d] matrix")
    d = int(X.shape[1])
    _dense(X, "X", (hyb.cols, d), "f32")
    if Y is None:
        Y = torch.empty((hyb.rows, d), dtype=torch.float32, device=X.device)
    _dense(Y, "Y", (hyb.rows, d), "f32", X.device)
    check(lib.strata_spmm_hyb_f32(hyb.handle, _ptr(X), _ptr(Y), d, _stream(stream)))
    return Y


def gnn_layer_work_floats(hyb: HybDecomposition, d_in: int, d_out: int) -> int:
    """Floats of the intermediate (T = X@W or Y = A@X) that gnn_layer needs."""
    return int(lib.strata_gnn_layer_work_floats(hyb.handle, d_in, d_out))


def gnn_layer(hyb: HybDecomposition, X, W, Z=None, work=None, stream=None):
    """GNN layer step Z = A @ X @ W (f32, device): hyb SpMM aggregation + the tcgen05 3xTF32
    transform, associated so the SpMM gathers the narrower rows (strata_gnn_layer_f32)."""
    import torch
    d_in, d_out = int(X.shape[1]), int(W.shape[1])
    if W.shape[0] != d_in:
        raise StrataError(6, "gnn_layer: W must be [d_in][d_out]")
    _dense(X, "X", (hyb.cols, d_in), "f32")
    _dense(W, "W", (d_in, d_out), "f32", X.device)
    if Z is None:
        Z = torch.empty((hyb.rows, d_out), dtype=torch.float32, device=X.device)
    _dense(Z, "Z", (hyb.rows, d_out), "f32", X.device)
    need = max(gnn_layer_work_floats(hyb, d_in, d_out), 1)
    if work is None:
        work = torch.empty(need, dtype=torch.float32, device=X.device)
    if work.numel() < need or work.dtype != torch.float32 or not work.is_contiguous():
        raise StrataError(7, f"binding size mismatch for work: got {work.numel()}, declared {need}")
    check(lib.strata_gnn_layer_f32(hyb.handle, _ptr(X), _ptr(W), _ptr(Z), _ptr(work), d_in, d_out,
                                   _stream(stream)))
    return Z


def gemm(Y, W, Z=None, stream=None):
    """Dense transform Z = Y @ W (f32, device, row-major) on the tensor cores (strata_gemm_f32:
    tcgen05 kind::tf32 with the 3xTF32 split, fp32-accurate)."""
    import torch
    if Y.dim() != 2 or W.dim() != 2 or W.shape[0] != Y.shape[1]:
        raise StrataError(6, "gemm: Y must be [M][K] and W [K][N]")
    M, K, N = int(Y.shape[0]), int(Y.shape[1]), int(W.shape[1])
    _dense(Y, "Y", (M, K), "f32")
    _dense(W, "W", (K, N), "f32", Y.device)
    if Z is None:
        Z = torch.empty((M, N), dtype=torch.float32, device=Y.device)
    _dense(Z, "Z", (M, N), "f32", Y.device)
    check(lib.strata_gemm_f32(_ptr(Y), _ptr(W), _ptr(Z), M, K, N, _stream(stream)))
    return Z


def _host(t, name: str, shape):
    """Binding check of a host (pinned) f32 operand of the end-to-end entry points."""
    import torch
    if isinstance(t, torch.Tensor):
        ok = t.device.type == "cpu" and t.dtype == torch.float32 and t.is_contiguous()
    else:
        ok = isinstance(t, np.ndarray) and t.dtype == np.float32 and t.flags.c_contiguous
    if not ok:
        raise StrataError(7, f"binding for {name} must be a contiguous f32 host array")
    if tuple(t.shape) != tuple(shape):
        raise StrataError(7, f"binding size mismatch for {name}: got {int(np.prod(t.shape))}, "
                             f"declared {int(np.prod(shape))}")


def spmm_host(hyb: HybDecomposition, X_host, Y_host, stream=None):
    """End-to-end form: host (pinned) X in, host Y out, copies inside the call."""
    d = int(X_host.shape[1])
    _host(X_host, "X", (hyb.cols, d))
    _host(Y_host, "Y", (hyb.rows, d))
    check(lib.strata_spmm_hyb_f32_host(hyb.handle, _ptr(X_host), _ptr(Y_host), d,
                                       _stream(stream)))
    return Y_host


def spmm_multi(hyb: HybDecomposition, X, dst_ptrs, stream=None):
    """Y rows of ``hyb`` stored to every device address in ``dst_ptrs`` (ints: row-major
    [rows][d] f32 buffers, possibly peer-mapped; see sharding.PeerAllGather)."""
    d = int(X.shape[1])
    _dense(X, "X", (hyb.cols, d), "f32")
    n = len(dst_ptrs)
    arr = (C.c_void_p * n)(*dst_ptrs)
    check(lib.strata_spmm_hyb_f32_multi(hyb.handle, _ptr(X), C.cast(arr, C.c_void_p), n, d,
                                        _stream(stream)))


def ipc_handle(t) -> tuple:
    """(64-byte CUDA IPC handle of the allocation holding device tensor t, offset of t in it)."""
    buf = C.create_string_buffer(64)
    off = C.c_int64()
    check(lib.strata_ipc_get_handle(_ptr(t), buf, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation (handle from ipc_handle); returns its base address."""
    p = C.c_void_p()
    check(lib.strata_ipc_open_handle(C.c_char_p(handle), C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    check(lib.strata_ipc_close(C.c_void_p(ptr)))


def spmm_host_batch(hyb: HybDecomposition, X_hosts, Y_hosts, stream=None):
    """Batched end-to-end form: host (pinned) X_hosts[b] -> Y_hosts[b]; copy-in of the next
    matrix and copy-out of the previous one overlap each SpMM."""
    if len(X_hosts) != len(Y_hosts):
        raise StrataError(6, "spmm_host_batch: X and Y lists differ in length")
    n = len(X_hosts)
    if n == 0:
        return Y_hosts
    d = int(X_hosts[0].shape[1])
    for x, y in zip(X_hosts, Y_hosts):
        _host(x, "X", (hyb.cols, d))
        _host(y, "Y", (hyb.rows, d))
    xs = (C.c_void_p * n)(*[_ptr(x) for x in X_hosts])
    ys = (C.c_void_p * n)(*[_ptr(y) for y in Y_hosts])
    check(lib.strata_spmm_hyb_f32_host_batch(hyb.handle, C.cast(xs, C.c_void_p),
                                             C.cast(ys, C.c_void_p), n, d, _stream(stream)))
    return Y_hosts


def spmm_csr(csr: DeviceCsr, X, Y=None, stream=None):
    import torch
    d = int(X.shape[1])
    _dense(X, "X", (csr.cols, d), "f32")
    if Y is None:
        Y = torch.empty((csr.rows, d), dtype=torch.float32, device=X.device)
    _dense(Y, "Y", (csr.rows, d), "f32", X.device)
    check(lib.strata_spmm_csr_f32(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values), _ptr(X),
                                  _ptr(Y), csr.rows, csr.cols, d, _stream(stream)))
    return Y


def sddmm(csr: DeviceCsr, X, Yt_dn, B=None, stream=None):
    """B[nnz] = A .* (X @ Y) on the pattern; X [rows][d], Y [d][cols] (reference layout)."""
    import torch
    d = int(X.shape[1])
    _dense(X, "X", (csr.rows, d), "f32")
    _dense(Yt_dn, "Y", (d, csr.cols), "f32", X.device)
    if B is None:
        B = torch.empty((csr.nnz,), dtype=torch.float32, device=X.device)
    _dense(B, "B", (csr.nnz,), "f32", X.device)
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


# ---- BSR (storage.hpp:117, storage.cpp:138-188) + tensor-core BSR SpMM ---------------------

class BsrMatrix:
    """Device-resident BSR storage: JO_indptr / JO_indices / values (f32 + bf16 copy)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        v = [C.c_int64() for _ in range(5)]
        check(lib.strata_bsr_info(handle, *(C.byref(x) for x in v)))
        self.mb, self.nb, self.b, self.nblocks, self.pad_slots = (x.value for x in v)

    @property
    def handle(self):
        return self._h

    def arrays(self, prefix: str = "bsr_") -> dict:
        jp = np.empty(self.mb + 1, np.int32)
        ji = np.empty(max(self.nblocks, 1), np.int32)
        bv = np.empty(max(self.nblocks * self.b * self.b, 1), np.float32)
        check(lib.strata_bsr_read(self._h, jp.ctypes.data, ji.ctypes.data, bv.ctypes.data))
        return {prefix + "JO_indptr": jp, prefix + "JO_indices": ji[:self.nblocks],
                "values": bv[:self.nblocks * self.b * self.b]}

    def close(self):
        if self._h:
            lib.strata_bsr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def csr_to_bsr(csr: DeviceCsr, b: int, stream=None) -> BsrMatrix:
    h = C.c_void_p()
    check(lib.strata_bsr_from_csr(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values),
                                  csr.rows, csr.cols, csr.nnz, b, _stream(stream), C.byref(h)))
    return BsrMatrix(h)


def bsr_spmm(bsr: BsrMatrix, X_bf16, Y=None, stream=None):
    """Y[mb*b][d] (f32) = A_bsr @ X on tcgen05 tensor cores; X is bf16 [nb*b][d]."""
    import torch
    d = int(X_bf16.shape[1])
    _dense(X_bf16, "X", (bsr.nb * bsr.b, d), "bf16")
    if Y is None:
        Y = torch.empty((bsr.mb * bsr.b, d), dtype=torch.float32, device=X_bf16.device)
    _dense(Y, "Y", (bsr.mb * bsr.b, d), "f32", X_bf16.device)
    check(lib.strata_bsr_spmm_bf16(bsr.handle, _ptr(X_bf16), _ptr(Y), d, _stream(stream)))
    return Y


def bsr_spmm_batched(bsr: BsrMatrix, values_bf16, X_bf16, Y=None, stream=None):
    """Multi-head block-sparse SpMM (batched SpMM of sparse attention): the heads
    share the block structure of ``bsr`` and bring their own block values.
    values_bf16 [H][nblocks][b][b] (row-major blocks, the reference's A_bsr layout per head),
    X_bf16 [H][nb*b][d] -> Y [H][mb*b][d] f32, Y[h] = A_h @ X[h]."""
    import torch
    H, _, d = (int(x) for x in X_bf16.shape)
    if tuple(values_bf16.shape) != (H, bsr.nblocks, bsr.b, bsr.b):
        raise StrataError(6, "bsr_spmm_batched: values must be [heads][nblocks][b][b]")
    _dense(X_bf16, "X", (H, bsr.nb * bsr.b, d), "bf16")
    _dense(values_bf16, "A_bsr", (H, bsr.nblocks, bsr.b, bsr.b), "bf16", X_bf16.device)
    if Y is None:
        Y = torch.empty((H, bsr.mb * bsr.b, d), dtype=torch.float32, device=X_bf16.device)
    _dense(Y, "Y", (H, bsr.mb * bsr.b, d), "f32", X_bf16.device)
    check(lib.strata_bsr_spmm_bf16_batched(bsr.handle, _ptr(values_bf16), _ptr(X_bf16), _ptr(Y),
                                           H, d, _stream(stream)))
    return Y


# ---- DBSR / SR-BCRS (storage.cpp:336-440) ---------------------------------------------------

class DbsrMatrix:
    """Device DBSR: the BSR of the matrix plus its stored block rows (IO_indices)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        v = [C.c_int64() for _ in range(6)]
        check(lib.strata_dbsr_info(handle, *(C.byref(x) for x in v)))
        self.mb, self.nb, self.b, self.nstored, self.nblocks, self.pad_slots = (x.value for x in v)

    @property
    def handle(self):
        return self._h

    def arrays(self, prefix: str = "dbsr_") -> dict:
        io = np.empty(max(self.nstored, 1), np.int32)
        jp = np.empty(self.nstored + 1, np.int32)
        ji = np.empty(max(self.nblocks, 1), np.int32)
        bv = np.empty(max(self.nblocks * self.b * self.b, 1), np.float32)
        check(lib.strata_dbsr_read(self._h, io.ctypes.data, jp.ctypes.data, ji.ctypes.data,
                                   bv.ctypes.data))
        return {prefix + "IO_indptr": np.array([0, self.nstored], np.int32),
                prefix + "IO_indices": io[:self.nstored], prefix + "JO_indptr": jp,
                prefix + "JO_indices": ji[:self.nblocks],
                "values": bv[:self.nblocks * self.b * self.b]}

    def __del__(self):
        if getattr(self, "_h", None):
            lib.strata_dbsr_destroy(self._h)
            self._h = None


def csr_to_dbsr(csr: DeviceCsr, b: int, stream=None) -> DbsrMatrix:
    h = C.c_void_p()
    check(lib.strata_dbsr_from_csr(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values), csr.rows,
                                   csr.cols, csr.nnz, b, _stream(stream), C.byref(h)))
    return DbsrMatrix(h)


def dbsr_spmm(dbsr: DbsrMatrix, X_bf16, Y=None, stream=None):
    """Y[mb*b][d] (f32) = A_dbsr @ X on tcgen05 (stored block rows only)."""
    import torch
    d = int(X_bf16.shape[1])
    _dense(X_bf16, "X", (dbsr.nb * dbsr.b, d), "bf16")
    if Y is None:
        Y = torch.empty((dbsr.mb * dbsr.b, d), dtype=torch.float32, device=X_bf16.device)
    _dense(Y, "Y", (dbsr.mb * dbsr.b, d), "f32", X_bf16.device)
    check(lib.strata_dbsr_spmm_bf16(dbsr.handle, _ptr(X_bf16), _ptr(Y), d, _stream(stream)))
    return Y


class SrbcrsMatrix:
    """Device SR-BCRS(t, g): G_indptr / JT_indices / slot-major values."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        v = [C.c_int64() for _ in range(5)]
        check(lib.strata_srbcrs_info(handle, *(C.byref(x) for x in v)))
        self.mb, self.t, self.g, self.groups, self.pad_slots = (x.value for x in v)

    @property
    def handle(self):
        return self._h

    def arrays(self, prefix: str = "srbcrs_") -> dict:
        gp = np.empty(self.mb + 1, np.int32)
        jt = np.empty(max(self.groups * self.g, 1), np.int32)
        v = np.empty(max(self.groups * self.g * self.t, 1), np.float32)
        check(lib.strata_srbcrs_read(self._h, gp.ctypes.data, jt.ctypes.data, v.ctypes.data))
        return {prefix + "G_indptr": gp, prefix + "JT_indices": jt[:self.groups * self.g],
                "values": v[:self.groups * self.g * self.t]}

    def __del__(self):
        if getattr(self, "_h", None):
            lib.strata_srbcrs_destroy(self._h)
            self._h = None


def csr_to_srbcrs(csr: DeviceCsr, t: int, g: int, stream=None) -> SrbcrsMatrix:
    h = C.c_void_p()
    check(lib.strata_srbcrs_from_csr(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values),
                                     csr.rows, csr.cols, csr.nnz, t, g, _stream(stream), C.byref(h)))
    return SrbcrsMatrix(h)


def srbcrs_spmm(sr: SrbcrsMatrix, X_bf16, Y=None, stream=None):
    """Y[mb*t][d] (f32) = A_srbcrs @ X on tcgen05 (t = 8, g = 32)."""
    import torch
    d = int(X_bf16.shape[1])
    if X_bf16.dtype != torch.bfloat16 or not X_bf16.is_contiguous() or X_bf16.dim() != 2:
        raise StrataError(7, "binding for X must be a contiguous bf16 [cols][d] matrix")
    if Y is None:
        Y = torch.empty((sr.mb * sr.t, d), dtype=torch.float32, device=X_bf16.device)
    _dense(Y, "Y", (sr.mb * sr.t, d), "f32", X_bf16.device)
    check(lib.strata_srbcrs_spmm_bf16(sr.handle, _ptr(X_bf16), _ptr(Y), d, _stream(stream)))
    return Y


__all__ += ["DbsrMatrix", "csr_to_dbsr", "dbsr_spmm", "SrbcrsMatrix", "csr_to_srbcrs",
            "srbcrs_spmm"]


# ---- fused attention layer step (SDDMM -> edge softmax -> SpMM) ------------------------------

class AttentionPlan:
    """Row/chunk work plan of a CSR pattern for ``attention`` (strata_attn_plan_create)."""

    def __init__(self, csr: DeviceCsr, stream=None):
        self.csr = csr
        h = C.c_void_p()
        check(lib.strata_attn_plan_create(_ptr(csr.indptr), csr.rows, csr.nnz, C.byref(h),
                                          _stream(stream)))
        self._h = h

    def __call__(self, Q, K, V, Z=None, stream=None):
        """Z[i] = sum_j softmax_j(A_ij <Q_i, K_j>) V_j over the stored j of row i."""
        import torch
        d = int(Q.shape[1])
        _dense(Q, "Q", (self.csr.rows, d), "f32")
        _dense(K, "K", (self.csr.cols, d), "f32", Q.device)
        _dense(V, "V", (self.csr.cols, d), "f32", Q.device)
        if Z is None:
            Z = torch.empty((self.csr.rows, d), dtype=torch.float32, device=Q.device)
        _dense(Z, "Z", (self.csr.rows, d), "f32", Q.device)
        check(lib.strata_attn_csr_f32(self._h, _ptr(self.csr.indptr), _ptr(self.csr.indices),
                                      _ptr(self.csr.values), _ptr(Q), _ptr(K), _ptr(V), _ptr(Z), d,
                                      _stream(stream)))
        return Z

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.strata_attn_plan_destroy(h)
            self._h = None


__all__ += ["AttentionPlan"]


def bsr_sddmm(bsr: BsrMatrix, Q_bf16, K_bf16, S=None, stream=None):
    """Block-sparse SDDMM (sparse-attention scores) on tcgen05: Q [H][mb*b][d], K [H][nb*b][d]
    bf16 -> S [H][nblocks][b][b] f32 = A_bsr (.) Q K^T on the stored blocks (2-D Q/K: H = 1)."""
    import torch
    Q3 = Q_bf16 if Q_bf16.dim() == 3 else Q_bf16.unsqueeze(0)
    K3 = K_bf16 if K_bf16.dim() == 3 else K_bf16.unsqueeze(0)
    H, _, d = (int(x) for x in Q3.shape)
    _dense(Q3, "Q", (H, bsr.mb * bsr.b, d), "bf16")
    _dense(K3, "K", (H, bsr.nb * bsr.b, d), "bf16", Q3.device)
    if S is None:
        S = torch.empty((H, bsr.nblocks, bsr.b, bsr.b), dtype=torch.float32, device=Q3.device)
    _dense(S, "S", (H, bsr.nblocks, bsr.b, bsr.b), "f32", Q3.device)
    check(lib.strata_bsr_sddmm_bf16(bsr.handle, _ptr(Q3), _ptr(K3), _ptr(S), H, d, _stream(stream)))
    return S


__all__ += ["bsr_sddmm"]


# ---- ELL (storage.hpp:124, storage.cpp:190-227) --------------------------------------------

def csr_to_ell(csr: DeviceCsr, w: int, stream=None):
    """Device ELL arrays (J_indices[rows*w], values[rows*w]); StrataError(kind='Capacity')
    naming the row when a row exceeds w."""
    import torch
    dev = csr.indptr.device
    J = torch.empty(max(csr.rows * w, 1), dtype=torch.int32, device=dev)
    V = torch.empty(max(csr.rows * w, 1), dtype=torch.float32, device=dev)
    check(lib.strata_ell_from_csr(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values),
                                  csr.rows, csr.cols, w, _ptr(J), _ptr(V), _stream(stream)))
    return J[:csr.rows * w], V[:csr.rows * w]


# ---- RGMS / RGCN (kernels.cpp:138-167, driver.cpp:241-314) ---------------------------------

@dataclass
class RelSparse:
    """kernels.hpp RelSparse flattened to relation-major edges: rel_ptr[R+1], dst (row i),
    src (col j), A.  Built from the reference arrays I_indptr/I_indices/J_indptr/J_indices."""
    relations: int
    rows: int
    cols: int
    rel_ptr: np.ndarray
    dst: np.ndarray
    src: np.ndarray
    A: np.ndarray

    @staticmethod
    def from_reference_arrays(R, rows, cols, I_indptr, I_indices, J_indptr, J_indices, A):
        I_indptr = np.asarray(I_indptr, np.int64)
        J_indptr = np.asarray(J_indptr, np.int64)
        rel_ptr = J_indptr[I_indptr].astype(np.int32)          # edges of relation r
        counts = np.diff(J_indptr)
        dst = np.repeat(np.asarray(I_indices, np.int32), counts)
        return RelSparse(R, rows, cols, rel_ptr, dst.astype(np.int32),
                         np.asarray(J_indices, np.int32), np.asarray(A, np.float32))

    @property
    def nnz(self) -> int:
        return int(self.src.shape[0])

    def to_device(self, device="cuda"):
        import torch
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return RelSparse(self.relations, self.rows, self.cols, t(self.rel_ptr), t(self.dst),
                         t(self.src), t(self.A))


class RgmsPlan:
    """Device plan of one RelSparse (strata_rgms_plan): the build step of build_rgms_pipeline
    (driver.cpp:241-314).  ``run`` is the interpret step: Y = sum_r A_r @ X @ W_r."""

    def __init__(self, rel: RelSparse, stream=None):
        self.rows, self.cols, self.relations, self.nnz = rel.rows, rel.cols, rel.relations, rel.nnz
        h = C.c_void_p()
        check(lib.strata_rgms_plan(_ptr(rel.rel_ptr), _ptr(rel.dst), _ptr(rel.src), _ptr(rel.A),
                                   rel.relations, rel.rows, rel.cols, rel.nnz, C.byref(h),
                                   _stream(stream)))
        self._h = h

    @classmethod
    def from_hyb(cls, hybs, stream=None) -> "RgmsPlan":
        """The "hyb" format of build_rgms_pipeline (driver.cpp:290-300): one HybDecomposition
        per relation (strata_rgms_plan_hyb reads their parts in place, pads dropped)."""
        self = cls.__new__(cls)
        self.rows, self.cols, self.relations = hybs[0].rows, hybs[0].cols, len(hybs)
        arr = (C.c_void_p * len(hybs))(*[h.handle.value for h in hybs])
        h = C.c_void_p()
        check(lib.strata_rgms_plan_hyb(arr, len(hybs), C.byref(h), _stream(stream)))
        self._h = h
        self._hybs = list(hybs)  # keep the parts alive while the plan is in use
        self.nnz = None
        return self

    @property
    def message_rows(self) -> int:
        """T rows a run writes and reads back: the (relation, destination) runs of rows with two
        or more runs (a row's sole run is written to Y directly by pass 1)."""
        t, b = C.c_int64(), C.c_int64()
        check(lib.strata_rgms_info(self._h, C.byref(t), C.byref(b)))
        return b.value // 4

    def run(self, X_bf16, W_bf16, Y=None, stream=None):
        import torch
        d_in, d_out = int(W_bf16.shape[1]), int(W_bf16.shape[2])
        _dense(X_bf16, "X", (self.cols, d_in), "bf16")
        _dense(W_bf16, "W", (self.relations, d_in, d_out), "bf16", X_bf16.device)
        if Y is None:
            Y = torch.empty((self.rows, d_out), dtype=torch.float32, device=X_bf16.device)
        _dense(Y, "Y", (self.rows, d_out), "f32", X_bf16.device)
        check(lib.strata_rgms_run_bf16(self._h, _ptr(X_bf16), _ptr(W_bf16), _ptr(Y), d_in, d_out,
                                       _stream(stream)))
        return Y

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            import torch
            torch.cuda.synchronize()
            lib.strata_rgms_destroy(h)
            self._h = None


def rgms(rel, X_bf16, W_bf16, Y=None, stream=None):
    """Y[m][d_out] (f32) = sum_r A_r @ X @ W_r.  ``rel`` is a device RelSparse (one-shot
    strata_rgms_bf16: plan + run) or an RgmsPlan (run only)."""
    import torch
    if isinstance(rel, RgmsPlan):
        return rel.run(X_bf16, W_bf16, Y, stream)
    d_in, d_out = int(W_bf16.shape[1]), int(W_bf16.shape[2])
    _dense(X_bf16, "X", (rel.cols, d_in), "bf16")
    _dense(W_bf16, "W", (rel.relations, d_in, d_out), "bf16", X_bf16.device)
    if Y is None:
        Y = torch.empty((rel.rows, d_out), dtype=torch.float32, device=X_bf16.device)
    _dense(Y, "Y", (rel.rows, d_out), "f32", X_bf16.device)
    check(lib.strata_rgms_bf16(_ptr(rel.rel_ptr), _ptr(rel.dst), _ptr(rel.src), _ptr(rel.A),
                               rel.relations, rel.rows, rel.cols, rel.nnz, _ptr(X_bf16),
                               _ptr(W_bf16), _ptr(Y), d_in, d_out, _stream(stream)))
    return Y


def split_relations(m: CsrMatrix, relations: int, seed: int):
    """strata_cli.cpp:70-82: triplet t (in the generator's triplet order == CSR order here)
    goes to relation mt19937(seed)() % R.  Returns the RelSparse (kernels.cpp:19-62 layout)."""
    if m.row_order is None:
        raise StrataError(6, "split_relations needs the generator's triplet order (powerlaw)")
    draws = np.empty(m.nnz, np.uint32)
    _mt19937_stream(seed, draws)
    # CSR position of the t-th reference triplet: rows in generator order, columns ascending.
    lens = np.diff(m.indptr).astype(np.int64)
    ro = m.row_order.astype(np.int64)
    starts = np.repeat(m.indptr[:-1][ro].astype(np.int64) - np.cumsum(lens[ro]) + lens[ro], lens[ro])
    csr_pos = starts + np.arange(m.nnz, dtype=np.int64)
    rel = np.empty(m.nnz, np.int64)
    rel[csr_pos] = draws % relations
    rows_of = np.repeat(np.arange(m.rows, dtype=np.int64), lens)
    order = np.lexsort((m.indices, rows_of, rel))  # relation-major, (row, col) inside
    rel_sorted = rel[order]
    rel_ptr = np.searchsorted(rel_sorted, np.arange(relations + 1)).astype(np.int32)
    return RelSparse(relations, m.rows, m.cols, rel_ptr, rows_of[order].astype(np.int32),
                     m.indices[order].astype(np.int32), m.values[order].astype(np.float32))


def _mt19937_stream(seed: int, out: np.ndarray):
    """Raw 32-bit outputs of std::mt19937(seed): numpy's MT19937 with the legacy
    init_genrand seeding produces the identical tempered word sequence."""
    bg = np.random.MT19937(0)
    bg._legacy_seeding(seed)
    out[:] = bg.random_raw(out.size).astype(np.uint32)


__all__ += ["BsrMatrix", "csr_to_bsr", "bsr_spmm", "bsr_spmm_batched", "csr_to_ell", "RelSparse", "RgmsPlan", "rgms",
            "split_relations"]
