"""ctypes binding of oracle/_ref/libstrata_ref.so — the UNMODIFIED reference library
(TEST INFRASTRUCTURE ONLY; see oracle/Makefile and oracle/ref_shim.cpp)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libstrata_ref.so")
_lib = None
vp = C.c_void_p
i64 = C.c_int64

F32, F64, I32 = 1, 2, 0


def available() -> bool:
    return os.path.exists(LIB_PATH)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle ref` where "
                              "/root/reference exists")
        L = C.CDLL(LIB_PATH)
        L.sref_last_error.restype = C.c_char_p
        L.sref_generate.argtypes = [C.c_char_p, i64, i64, C.c_double, i64, i64, C.c_double,
                                    C.c_uint64, C.POINTER(vp)]
        L.sref_coo_from_arrays.argtypes = [i64, i64, i64, vp, vp, vp, C.POINTER(vp)]
        L.sref_coo_info.argtypes = [vp, vp, vp, vp]
        L.sref_coo_triplets.argtypes = [vp, vp, vp, vp]
        L.sref_coo_free.argtypes = [vp]
        L.sref_read_matrix_market.argtypes = [C.c_char_p, i64, C.POINTER(vp)]
        L.sref_write_matrix_market.argtypes = [vp, C.c_char_p, i64]
        L.sref_write_matrix_market.restype = i64
        L.sref_split_relations.argtypes = [vp, i64, C.c_uint64, vp]
        L.sref_dense_int.argtypes = [i64, C.c_uint64, vp]
        L.sref_build_csr.argtypes = [vp, C.c_int, C.POINTER(vp)]
        L.sref_csr_to_bsr.argtypes = [vp, i64, C.POINTER(vp)]
        L.sref_csr_to_dbsr.argtypes = [vp, i64, C.POINTER(vp)]
        L.sref_csr_to_srbcrs.argtypes = [vp, i64, i64, C.POINTER(vp)]
        L.sref_csr_to_ell.argtypes = [vp, i64, C.POINTER(vp)]
        L.sref_hyb_auto_k.argtypes = [vp]
        L.sref_storage_info.argtypes = [vp, vp]
        L.sref_storage_aux.argtypes = [vp, C.c_char_p, vp, i64]
        L.sref_storage_aux.restype = i64
        L.sref_storage_values.argtypes = [vp, vp]
        L.sref_padding_ratio.argtypes = [vp, C.POINTER(C.c_double)]
        L.sref_validate_storage.argtypes = [vp]
        L.sref_storage_free.argtypes = [vp]
        L.sref_decompose_hyb.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]
        L.sref_hyb_num_parts.argtypes = [vp]
        L.sref_hyb_padding.argtypes = [vp]
        L.sref_hyb_padding.restype = C.c_double
        L.sref_hyb_part_info.argtypes = [vp, C.c_int, vp]
        L.sref_hyb_part_storage.argtypes = [vp, C.c_int]
        L.sref_hyb_part_storage.restype = vp
        L.sref_hyb_free.argtypes = [vp]
        L.sref_hyb_rules.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, C.c_char_p, i64]
        L.sref_pipeline_matrix.argtypes = [C.c_int, vp, i64, C.c_int, C.c_char_p, C.c_int,
                                           C.POINTER(vp)]
        L.sref_pipeline_rgms.argtypes = [vp, i64, i64, i64, C.c_int, C.c_char_p, C.c_uint64,
                                         C.POINTER(vp)]
        L.sref_pipeline_set.argtypes = [vp, C.c_char_p, vp, i64]
        L.sref_pipeline_get.argtypes = [vp, C.c_char_p, vp, i64]
        L.sref_pipeline_get.restype = i64
        L.sref_pipeline_run.argtypes = [vp, vp, i64, C.POINTER(i64)]
        L.sref_pipeline_free.argtypes = [vp]
        _lib = L
    return _lib


def _chk(rc):
    if rc:
        raise RefError(rc, lib().sref_last_error().decode())


def _p(a):
    return a.ctypes.data if a is not None else None


class Coo:
    def __init__(self, h):
        self.h = h
        r, c, z = i64(), i64(), i64()
        lib().sref_coo_info(h, C.byref(r), C.byref(c), C.byref(z))
        self.rows, self.cols, self.nnz = r.value, c.value, z.value

    @staticmethod
    def generate(kind, n, m, density=0.0, band=0, block=0, avg_degree=0.0, seed=1):
        h = vp()
        _chk(lib().sref_generate(kind.encode(), n, m, density, band, block, avg_degree, seed,
                                 C.byref(h)))
        return Coo(h)

    @staticmethod
    def from_arrays(rows, cols, r, c, v):
        r = np.ascontiguousarray(r, np.int64)
        c = np.ascontiguousarray(c, np.int64)
        v = np.ascontiguousarray(v, np.float64)
        h = vp()
        _chk(lib().sref_coo_from_arrays(rows, cols, r.size, _p(r), _p(c), _p(v), C.byref(h)))
        return Coo(h)

    def triplets(self):
        r = np.empty(self.nnz, np.int64)
        c = np.empty(self.nnz, np.int64)
        v = np.empty(self.nnz, np.float64)
        lib().sref_coo_triplets(self.h, _p(r), _p(c), _p(v))
        return r, c, v

    @staticmethod
    def read_matrix_market(text: bytes):
        """mmio.cpp:17-55 over an in-memory stream; raises RefError like the reference."""
        h = vp()
        _chk(lib().sref_read_matrix_market(text, len(text), C.byref(h)))
        return Coo(h)

    def write_matrix_market(self) -> bytes:
        """mmio.cpp:63-72 (sorted triplets, precision 17)."""
        n = lib().sref_write_matrix_market(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib().sref_write_matrix_market(self.h, buf, n + 1)
        return buf.raw[:n]

    def split_relations(self, R, seed):
        outs = (vp * R)()
        _chk(lib().sref_split_relations(self.h, R, seed, outs))
        return [Coo(vp(outs[i])) for i in range(R)]

    def __del__(self):
        try:
            lib().sref_coo_free(self.h)
        except Exception:
            pass


class Storage:
    def __init__(self, h, owned=True):
        self.h = h
        self.owned = owned
        info = np.zeros(8, np.int64)
        lib().sref_storage_info(h, _p(info))
        (self.rows, self.cols, self.nnz, self.pad_slots, self.block, self.nvalues,
         self.orig_rows, self.orig_cols) = (int(x) for x in info)

    @staticmethod
    def csr(coo: Coo, dtype=F32):
        h = vp()
        _chk(lib().sref_build_csr(coo.h, dtype, C.byref(h)))
        return Storage(h)

    def to_bsr(self, b):
        h = vp()
        _chk(lib().sref_csr_to_bsr(self.h, b, C.byref(h)))
        return Storage(h)

    def to_dbsr(self, b):
        h = vp()
        _chk(lib().sref_csr_to_dbsr(self.h, b, C.byref(h)))
        return Storage(h)

    def to_srbcrs(self, t, g):
        h = vp()
        _chk(lib().sref_csr_to_srbcrs(self.h, t, g, C.byref(h)))
        return Storage(h)

    def to_ell(self, w):
        h = vp()
        _chk(lib().sref_csr_to_ell(self.h, w, C.byref(h)))
        return Storage(h)

    def aux(self, name):
        n = lib().sref_storage_aux(self.h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, np.int32)
        lib().sref_storage_aux(self.h, name.encode(), _p(out), n)
        return out

    def values(self):
        out = np.empty(self.nvalues, np.float64)
        lib().sref_storage_values(self.h, _p(out))
        return out

    def padding_ratio(self):
        r = C.c_double()
        _chk(lib().sref_padding_ratio(self.h, C.byref(r)))
        return r.value

    def validate(self):
        return lib().sref_validate_storage(self.h)

    def hyb_auto_k(self):
        return lib().sref_hyb_auto_k(self.h)

    def decompose_hyb(self, c, k, prefix=""):
        h = vp()
        _chk(lib().sref_decompose_hyb(self.h, c, k, prefix.encode(), C.byref(h)))
        return Hyb(h, prefix)

    def hyb_rules(self, c, k, name="hyb"):
        buf = C.create_string_buffer(1 << 20)
        _chk(lib().sref_hyb_rules(self.h, c, k, name.encode(), buf, len(buf)))
        out = []
        for line in buf.value.decode().strip().splitlines():
            f = line.split()
            arrays = {a.split(":")[0]: int(a.split(":")[1]) for a in f[2:-1]}
            out.append({"name": f[0], "new_buffer": f[1], "arrays": arrays, "nvalues": int(f[-1])})
        return out

    def __del__(self):
        if self.owned:
            try:
                lib().sref_storage_free(self.h)
            except Exception:
                pass


class Hyb:
    def __init__(self, h, prefix):
        self.h = h
        self.prefix = prefix
        self.padding_ratio = lib().sref_hyb_padding(h)
        self.parts = []
        for i in range(lib().sref_hyb_num_parts(h)):
            info = np.zeros(8, np.int64)
            lib().sref_hyb_part_info(h, i, _p(info))
            p, b, w, nr, nz, pad, lo, hi = (int(x) for x in info)
            st = Storage(vp(lib().sref_hyb_part_storage(h, i)), owned=False)
            pre = f"{prefix}hyb_p{p}_b{b}_"
            self.parts.append(dict(partition=p, bucket=b, width=w, nrows=nr, nnz=nz,
                                   pad_slots=pad, col_lo=lo, col_hi=hi,
                                   I_indptr=st.aux(pre + "I_indptr"),
                                   I_indices=st.aux(pre + "I_indices"),
                                   J_indices=st.aux(pre + "J_indices"),
                                   values=st.values().astype(np.float32)))

    def __del__(self):
        try:
            lib().sref_hyb_free(self.h)
        except Exception:
            pass


class Pipeline:
    """build_matrix_pipeline / build_rgms_pipeline + interpret, through the reference."""

    def __init__(self, h):
        self.h = h

    @staticmethod
    def matrix(op: str, coo: Coo, d: int, dtype=F32, fmt="csr", threads=1):
        h = vp()
        _chk(lib().sref_pipeline_matrix(0 if op == "spmm" else 1, coo.h, d, dtype, fmt.encode(),
                                        threads, C.byref(h)))
        return Pipeline(h)

    @staticmethod
    def rgms(rels, d_in, d_out, dtype=F32, fmt="csr", seed=7):
        arr = (vp * len(rels))(*[r.h for r in rels])
        h = vp()
        _chk(lib().sref_pipeline_rgms(arr, len(rels), d_in, d_out, dtype, fmt.encode(), seed,
                                      C.byref(h)))
        return Pipeline(h)

    def set(self, name, data):
        data = np.ascontiguousarray(data, np.float64).ravel()
        _chk(lib().sref_pipeline_set(self.h, name.encode(), _p(data), data.size))

    def get(self, name):
        n = lib().sref_pipeline_get(self.h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, np.float64)
        lib().sref_pipeline_get(self.h, name.encode(), _p(out), n)
        return out

    def run(self):
        n = i64()
        _chk(lib().sref_pipeline_run(self.h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        _chk(lib().sref_pipeline_run(self.h, _p(out), n.value, C.byref(n)))
        return out

    def run_sized(self, n):
        """One interpret() whose output (n elements, known to the caller) is copied out by the
        same call."""
        out = np.empty(n, np.float64)
        got = i64()
        _chk(lib().sref_pipeline_run(self.h, _p(out), n, C.byref(got)))
        if got.value != n:
            raise RefError(7, f"output has {got.value} elements, expected {n}")
        return out

    def run_timed(self):
        """One interpret() of stage III (the reference tuner's timed call, tune.cpp:137)."""
        n = i64()
        _chk(lib().sref_pipeline_run(self.h, None, 0, C.byref(n)))

    def __del__(self):
        try:
            lib().sref_pipeline_free(self.h)
        except Exception:
            pass


def dense_int(count, seed):
    out = np.empty(count, np.float64)
    lib().sref_dense_int(count, seed, _p(out))
    return out
