"""ctypes binding of liboracle.so (plain-C restatement; TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle`")
        _lib = C.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def hyb_decompose(rows, cols, indptr, indices, values, c, k):
    """Returns (parts, padding_ratio); parts = list of dicts like HybDecomposition::parts."""
    L = lib()
    nb = c * (k + 1)
    seg = np.zeros(max(nb, 1), np.int64)
    nnzc = np.zeros(max(nb, 1), np.int64)
    rc = L.or_hyb_count(C.c_int64(rows), C.c_int64(cols), C.c_void_p(_p(indptr)),
                        C.c_void_p(_p(indices)), c, k, C.c_void_p(_p(seg)), C.c_void_p(_p(nnzc)))
    if rc:
        raise OracleError(rc, "hyb requires c >= 1 and k >= 0")
    I = [np.zeros(int(seg[b]), np.int32) for b in range(nb)]
    J = [np.zeros(int(seg[b]) << (b % (k + 1)), np.int32) for b in range(nb)]
    V = [np.zeros(int(seg[b]) << (b % (k + 1)), np.float32) for b in range(nb)]
    # keep a dummy element so every pointer is valid
    keep = [np.zeros(1, np.int32), np.zeros(1, np.float32)]
    Ip = (C.c_void_p * nb)(*[_p(a) if a.size else _p(keep[0]) for a in I])
    Jp = (C.c_void_p * nb)(*[_p(a) if a.size else _p(keep[0]) for a in J])
    Vp = (C.c_void_p * nb)(*[_p(a) if a.size else _p(keep[1]) for a in V])
    L.or_hyb_fill(C.c_int64(rows), C.c_int64(cols), C.c_void_p(_p(indptr)),
                  C.c_void_p(_p(indices)), C.c_void_p(_p(values)), c, k, Ip, Jp, Vp)
    parts = []
    part_w = (cols + c - 1) // c
    pads = slots = 0
    for bin_ in range(nb):
        if seg[bin_] == 0:
            continue
        p, b = divmod(bin_, k + 1)
        w = 1 << b
        nr = int(seg[bin_])
        parts.append(dict(partition=p, bucket=b, width=w, nrows=nr, nnz=int(nnzc[bin_]),
                          pad_slots=nr * w - int(nnzc[bin_]), col_lo=p * part_w,
                          col_hi=min(cols, (p + 1) * part_w), I_indices=I[bin_],
                          J_indices=J[bin_], values=V[bin_]))
        pads += nr * w - int(nnzc[bin_])
        slots += nr * w
    return parts, (pads / slots if slots else 0.0)


def csr_to_bsr(rows, cols, indptr, indices, values, b):
    L = lib()
    L.or_csr_to_bsr.restype = C.c_int64
    nblk = L.or_csr_to_bsr(C.c_int64(rows), C.c_int64(cols), C.c_void_p(_p(indptr)),
                           C.c_void_p(_p(indices)), C.c_void_p(_p(values)), C.c_int64(b),
                           None, None, None)
    mb = (rows + b - 1) // b
    jp = np.zeros(mb + 1, np.int32)
    ji = np.zeros(max(nblk, 1), np.int32)
    bv = np.zeros(max(nblk * b * b, 1), np.float32)
    L.or_csr_to_bsr(C.c_int64(rows), C.c_int64(cols), C.c_void_p(_p(indptr)),
                    C.c_void_p(_p(indices)), C.c_void_p(_p(values)), C.c_int64(b),
                    C.c_void_p(_p(jp)), C.c_void_p(_p(ji)), C.c_void_p(_p(bv)))
    return jp, ji[:nblk], bv[:nblk * b * b]


def csr_to_ell(rows, cols, indptr, indices, values, w):
    L = lib()
    J = np.zeros(max(rows * w, 1), np.int32)
    V = np.zeros(max(rows * w, 1), np.float32)
    bad = C.c_int64(-1)
    rc = L.or_csr_to_ell(C.c_int64(rows), C.c_int64(cols), C.c_void_p(_p(indptr)),
                         C.c_void_p(_p(indices)), C.c_void_p(_p(values)), C.c_int64(w),
                         C.c_void_p(_p(J)), C.c_void_p(_p(V)), C.byref(bad))
    if rc:
        raise OracleError(rc, f"row {bad.value}" if rc == 4 else "bad ELL width")
    return J[:rows * w], V[:rows * w]


def hyb_auto_k(rows, nnz):
    return lib().or_hyb_auto_k(C.c_int64(rows), C.c_int64(nnz))


def spmm_csr_refnum(rows, indptr, indices, A, X, threads=os.cpu_count()):
    d = X.shape[1]
    X = np.ascontiguousarray(X, np.float32)
    Y = np.empty((rows, d), np.float32)
    lib().or_spmm_csr_refnum(C.c_int64(rows), C.c_int64(d), C.c_void_p(_p(indptr)),
                             C.c_void_p(_p(indices)), C.c_void_p(_p(A)),
                             C.c_void_p(_p(X)),
                             C.c_void_p(_p(Y)), threads)
    return Y


def spmm_hyb_refnum(rows, parts, X):
    d = X.shape[1]
    X = np.ascontiguousarray(X, np.float32)
    Y = np.empty((rows, d), np.float32)
    n = len(parts)
    pr = np.array([p["nrows"] for p in parts] or [0], np.int64)
    pw = np.array([p["width"] for p in parts] or [1], np.int64)
    Ip = (C.c_void_p * max(n, 1))(*[_p(p["I_indices"]) for p in parts])
    Jp = (C.c_void_p * max(n, 1))(*[_p(p["J_indices"]) for p in parts])
    Vp = (C.c_void_p * max(n, 1))(*[_p(p["values"]) for p in parts])
    lib().or_spmm_hyb_refnum(C.c_int64(rows), C.c_int64(d), n, C.c_void_p(_p(pr)),
                             C.c_void_p(_p(pw)), Ip, Jp, Vp, C.c_void_p(_p(X)), C.c_void_p(_p(Y)))
    return Y


def spmm_csr_f64(rows, indptr, indices, A, X, threads=os.cpu_count()):
    d = X.shape[1]
    A = np.ascontiguousarray(A, np.float64)
    X = np.ascontiguousarray(X, np.float64)
    Y = np.empty((rows, d), np.float64)
    lib().or_spmm_csr_f64(C.c_int64(rows), C.c_int64(d), C.c_void_p(_p(indptr)),
                          C.c_void_p(_p(indices)),
                          C.c_void_p(_p(A)),
                          C.c_void_p(_p(X)), C.c_void_p(_p(Y)),
                          threads)
    return Y


def sddmm_csr_refnum(rows, cols, indptr, indices, A, X, Ydn, threads=os.cpu_count()):
    d = X.shape[1]
    X = np.ascontiguousarray(X, np.float32)
    Ydn = np.ascontiguousarray(Ydn, np.float32)
    B = np.empty(indices.shape[0], np.float32)
    lib().or_sddmm_csr_refnum(C.c_int64(rows), C.c_int64(cols), C.c_int64(d),
                              C.c_void_p(_p(indptr)), C.c_void_p(_p(indices)), C.c_void_p(_p(A)),
                              C.c_void_p(_p(X)),
                              C.c_void_p(_p(Ydn)),
                              C.c_void_p(_p(B)), threads)
    return B


def sddmm_csr_f64(rows, cols, indptr, indices, A, X, Ydn, threads=os.cpu_count()):
    d = X.shape[1]
    A = np.ascontiguousarray(A, np.float64)
    X = np.ascontiguousarray(X, np.float64)
    Ydn = np.ascontiguousarray(Ydn, np.float64)
    B = np.empty(indices.shape[0], np.float64)
    lib().or_sddmm_csr_f64(C.c_int64(rows), C.c_int64(cols), C.c_int64(d),
                           C.c_void_p(_p(indptr)), C.c_void_p(_p(indices)),
                           C.c_void_p(_p(A)),
                           C.c_void_p(_p(X)),
                           C.c_void_p(_p(Ydn)),
                           C.c_void_p(_p(B)), threads)
    return B


def bsr_spmm_refnum(mb, b, jo_indptr, jo_indices, bvals, X, threads=os.cpu_count()):
    d = X.shape[1]
    X = np.ascontiguousarray(X, np.float32)
    Y = np.empty((mb * b, d), np.float32)
    lib().or_bsr_spmm_refnum(C.c_int64(mb), C.c_int64(b), C.c_int64(d), C.c_void_p(_p(jo_indptr)),
                             C.c_void_p(_p(jo_indices)), C.c_void_p(_p(bvals)),
                             C.c_void_p(_p(X)),
                             C.c_void_p(_p(Y)), threads)
    return Y


def rgms_refnum(R, m, i_indptr, i_indices, j_indptr, j_indices, A, X, W):
    din, dout = W.shape[1], W.shape[2]
    X = np.ascontiguousarray(X, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    Y = np.empty((m, dout), np.float32)
    lib().or_rgms_refnum(C.c_int64(R), C.c_int64(m), C.c_int64(din), C.c_int64(dout),
                         C.c_void_p(_p(i_indptr)), C.c_void_p(_p(i_indices)),
                         C.c_void_p(_p(j_indptr)), C.c_void_p(_p(j_indices)), C.c_void_p(_p(A)),
                         C.c_void_p(_p(X)),
                         C.c_void_p(_p(W)), C.c_void_p(_p(Y)))
    return Y


def csr_to_dbsr(rows, cols, indptr, indices, values, b):
    """storage.cpp:336-370: the BSR of the matrix plus its stored block rows.
    Returns (IO_indices, JO_indptr over stored rows, JO_indices, values)."""
    jp, ji, bv = csr_to_bsr(rows, cols, indptr, indices, values, b)
    stored = np.flatnonzero(np.diff(jp) > 0).astype(np.int32)            # :342-344
    jptr = np.r_[0, jp[stored + 1]].astype(np.int32)                      # :362-363
    return stored, jptr, ji, bv


def csr_to_srbcrs(rows, cols, indptr, indices, values, t, g):
    """storage.cpp:372-440 (numpy restatement, small sizes): per tile row of t rows the sorted
    distinct columns, cut into groups of g (last group padded with the last column, :411-420);
    values slot-major [groups*g][t] placed by lower_bound (:421-436).
    Returns (G_indptr, JT_indices, values)."""
    if t < 1 or g < 1:
        raise OracleError(6, "SR-BCRS requires t >= 1 and g >= 1")
    indptr = np.asarray(indptr, np.int64)
    mb = -(-rows // t)
    tiles = []
    gptr = np.zeros(mb + 1, np.int32)
    for r in range(mb):
        q0, q1 = indptr[min(r * t, rows)], indptr[min((r + 1) * t, rows)]
        u = np.unique(indices[q0:q1])
        tiles.append(u)
        ng = -(-len(u) // g) if len(u) else 0
        gptr[r + 1] = gptr[r] + ng
    total = int(gptr[mb])
    jt = np.zeros(total * g, np.int32)
    vals = np.zeros(total * g * t, np.float32)
    for r, u in enumerate(tiles):
        base = int(gptr[r]) * g
        n = (int(gptr[r + 1]) - int(gptr[r])) * g
        if len(u):
            jt[base:base + len(u)] = u
            jt[base + len(u):base + n] = u[-1]
    for i in range(rows):
        r = i // t
        u = tiles[r]
        base = int(gptr[r]) * g
        for q in range(indptr[i], indptr[i + 1]):
            slot = int(np.searchsorted(u, indices[q]))
            vals[(base + slot) * t + (i % t)] = values[q]
    return gptr, jt, vals
