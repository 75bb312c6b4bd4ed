"""Generate tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle ref` built the library):
    python tests/golden/make_golden.py
The outputs are small, committed fixtures; the GPU box never needs /root/reference.

Every array comes straight out of the reference: generate_matrix (driver.cpp:365-416),
build_csr (storage.cpp:89-124), decompose_hyb (storage.cpp:271-334), csr_to_bsr
(storage.cpp:138-188), csr_to_ell (storage.cpp:190-227), hyb_rules (transform.cpp:525-557),
and interpret() of the canonical pipelines (driver.cpp:173-217, :241-314; interp.cpp:564-622).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def csr_arrays(st):
    return st.aux("J_indptr"), st.aux("J_indices"), st.values().astype(np.float32)


def example_coo():
    # test_storage.cpp:18-25 worked example
    r = [0, 0, 1, 2, 2, 2, 2]
    c = [0, 2, 3, 0, 1, 2, 3]
    v = [1, 2, 3, 4, 5, 6, 7]
    return ref.Coo.from_arrays(4, 4, r, c, v)


def hyb_cases():
    """(name, coo) graphs for the decomposition + SpMM goldens."""
    cases = [("example", example_coo())]
    cases.append(("powerlaw_600", ref.Coo.generate("powerlaw", 600, 500, 0, 0, 0, 7.0, 11)))
    cases.append(("powerlaw_dense_rows", ref.Coo.generate("powerlaw", 300, 300, 0, 0, 0, 40.0, 2)))
    cases.append(("random_64", ref.Coo.generate("random", 64, 48, 0.2, 0, 0, 0, 5)))
    cases.append(("banded_100", ref.Coo.generate("banded", 100, 100, 0, 3, 0, 0, 9)))
    # empty rows / empty matrix edge cases
    cases.append(("empty_5x7", ref.Coo.from_arrays(5, 7, [], [], [])))
    cases.append(("one_by_one", ref.Coo.from_arrays(1, 1, [0], [0], [5.0])))
    return cases


def main():
    out = {}
    rng = np.random.default_rng(1234)
    for name, coo in hyb_cases():
        csr = ref.Storage.csr(coo)
        ip, ix, v = csr_arrays(csr)
        out[f"{name}/shape"] = np.array([csr.rows, csr.cols], np.int64)
        out[f"{name}/indptr"], out[f"{name}/indices"], out[f"{name}/values"] = ip, ix, v
        out[f"{name}/auto_k"] = np.array([csr.hyb_auto_k()], np.int64)
        for c, k in [(1, 0), (1, 1), (1, 2), (1, 3), (2, 2), (3, 1), (4, 3), (1, csr.hyb_auto_k())]:
            h = csr.decompose_hyb(c, k)
            key = f"{name}/hyb_c{c}_k{k}"
            out[key + "/padding"] = np.array([h.padding_ratio])
            meta = []
            for i, P in enumerate(h.parts):
                meta.append([P["partition"], P["bucket"], P["width"], P["nrows"], P["nnz"],
                             P["pad_slots"], P["col_lo"], P["col_hi"]])
                out[f"{key}/p{i}/I"] = P["I_indices"]
                out[f"{key}/p{i}/J"] = P["J_indices"]
                out[f"{key}/p{i}/V"] = P["values"]
            out[key + "/meta"] = np.array(meta, np.int64).reshape(-1, 8)
        # interpreter SpMM (integer and real-valued operands), d = 8 and 32
        for d in (8, 32):
            Xi = ref.dense_int(csr.cols * d, 17).reshape(csr.cols, d)
            Xr = rng.standard_normal((csr.cols, d)).astype(np.float32).astype(np.float64)
            for tag, X in (("int", Xi), ("real", Xr)):
                pl = ref.Pipeline.matrix("spmm", coo, d, ref.F32, "hyb:c=1")
                pl.set("X", X)
                out[f"{name}/spmm_d{d}_{tag}/X"] = X.astype(np.float32)
                out[f"{name}/spmm_d{d}_{tag}/Y"] = pl.run().astype(np.float32).reshape(-1, d)
                pl64 = ref.Pipeline.matrix("spmm", coo, d, ref.F64, "csr")
                pl64.set("X", X)
                out[f"{name}/spmm_d{d}_{tag}/Y64"] = pl64.run().reshape(-1, d)
        # SDDMM (Y is [d][n])
        for d in (8, 32):
            Xs = rng.standard_normal((csr.rows, d)).astype(np.float32)
            Yd = rng.standard_normal((d, csr.cols)).astype(np.float32)
            pl = ref.Pipeline.matrix("sddmm", coo, d, ref.F32, "csr")
            pl.set("X", Xs)
            pl.set("Y", Yd)
            out[f"{name}/sddmm_d{d}/X"], out[f"{name}/sddmm_d{d}/Yd"] = Xs, Yd
            out[f"{name}/sddmm_d{d}/B"] = pl.run().astype(np.float32)
            pl64 = ref.Pipeline.matrix("sddmm", coo, d, ref.F64, "csr")
            pl64.set("X", Xs)
            pl64.set("Y", Yd)
            out[f"{name}/sddmm_d{d}/B64"] = pl64.run()
    out["cases"] = np.array([n for n, _ in hyb_cases()])

    # BSR: block-sparse mask (the C3 generator at small scale) and the example, b = 2 / 32
    for name, coo, b in [("bs128", ref.Coo.generate("blocksparse", 128, 96, 0.3, 0, 32, 0, 1), 32),
                         ("example", example_coo(), 2),
                         ("pl_b32", ref.Coo.generate("powerlaw", 100, 70, 0, 0, 0, 5.0, 4), 32)]:
        csr = ref.Storage.csr(coo)
        bs = csr.to_bsr(b)
        key = f"bsr/{name}_b{b}"
        out[key + "/csr_indptr"], out[key + "/csr_indices"], out[key + "/csr_values"] = csr_arrays(csr)
        out[key + "/shape"] = np.array([csr.rows, csr.cols, bs.rows, bs.cols, bs.pad_slots], np.int64)
        out[key + "/JO_indptr"] = bs.aux("JO_indptr")
        out[key + "/JO_indices"] = bs.aux("JO_indices")
        out[key + "/values"] = bs.values().astype(np.float32)
        d = 64
        X = ref.dense_int(bs.cols * d, 3).reshape(bs.cols, d)
        pl = ref.Pipeline.matrix("spmm", coo, d, ref.F32, f"bsr:b={b}")
        pl.set("X", X)
        out[key + "/X"] = X.astype(np.float32)
        out[key + "/Y"] = pl.run().astype(np.float32).reshape(-1, d)

    # DBSR (storage.cpp:336-370) and SR-BCRS (storage.cpp:372-440): arrays + the reference's
    # SpMM pipeline output for the tensor-core shapes (b = 32; t = 8, g = 32)
    for name, coo in [("example", example_coo()),
                      ("bs128", ref.Coo.generate("blocksparse", 128, 96, 0.3, 0, 32, 0, 1)),
                      ("pl", ref.Coo.generate("powerlaw", 300, 250, 0, 0, 0, 6.0, 5))]:
        csr = ref.Storage.csr(coo)
        ip, ix, v = csr_arrays(csr)
        out[f"fmt/{name}/csr"] = np.concatenate([[csr.rows, csr.cols], ip]).astype(np.int64)
        out[f"fmt/{name}/indices"], out[f"fmt/{name}/values"] = ix, v
        for b in (2, 32):
            db = csr.to_dbsr(b)
            key = f"dbsr/{name}_b{b}"
            out[key + "/IO_indices"] = db.aux("IO_indices")
            out[key + "/JO_indptr"] = db.aux("JO_indptr")
            out[key + "/JO_indices"] = db.aux("JO_indices")
            out[key + "/values"] = db.values().astype(np.float32)
            out[key + "/shape"] = np.array([db.rows, db.cols, db.pad_slots], np.int64)
        for t, g in ((2, 2), (3, 5), (8, 32)):
            sr = csr.to_srbcrs(t, g)
            key = f"srbcrs/{name}_t{t}_g{g}"
            out[key + "/G_indptr"] = sr.aux("G_indptr")
            out[key + "/JT_indices"] = sr.aux("JT_indices")
            out[key + "/values"] = sr.values().astype(np.float32)
            out[key + "/shape"] = np.array([sr.rows, sr.cols, sr.pad_slots], np.int64)
        d = 64
        for fmt in ("dbsr:b=32", "srbcrs:t=8,g=32"):
            pl = ref.Pipeline.matrix("spmm", coo, d, ref.F32, fmt)
            rows_x = -(-csr.cols // 32) * 32 if fmt.startswith("dbsr") else csr.cols  # pad_for_format
            X = ref.dense_int(rows_x * d, 11).reshape(rows_x, d)
            pl.set("X", X)
            key = f"fmtspmm/{name}/{fmt.split(':')[0]}"
            out[key + "/X"] = X.astype(np.float32)
            out[key + "/Y"] = pl.run().astype(np.float32).reshape(-1, d)

    # RGMS: power-law graph split into relations (strata_cli.cpp:70-82), csr and hyb formats
    base = ref.Coo.generate("powerlaw", 400, 400, 0, 0, 0, 3.0, 1)
    R = 5
    rels = base.split_relations(R, 1)
    for fmt in ("csr", "hyb"):
        pl = ref.Pipeline.rgms(rels, 16, 16, ref.F32, fmt, seed=7)
        out[f"rgms/{fmt}/Y"] = pl.run().astype(np.float32).reshape(-1, 16)
        out[f"rgms/{fmt}/X"] = pl.get("X").astype(np.float32).reshape(-1, 16)
        out[f"rgms/{fmt}/W"] = pl.get("W").astype(np.float32).reshape(R, 16, 16)
        out["rgms/A"], out["rgms/I_indptr"] = pl.get("A").astype(np.float32), pl.get("I_indptr").astype(np.int32)
        out["rgms/I_indices"] = pl.get("I_indices").astype(np.int32)
        out["rgms/J_indptr"] = pl.get("J_indptr").astype(np.int32)
        out["rgms/J_indices"] = pl.get("J_indices").astype(np.int32)
    out["rgms/shape"] = np.array([R, 400, 400], np.int64)

    # ELL at exact capacity and a capacity failure (test_storage.cpp:95-120 style)
    for name, coo in [("example", example_coo()), ("pl", ref.Coo.generate("powerlaw", 50, 40, 0, 0, 0, 4.0, 8))]:
        csr = ref.Storage.csr(coo)
        ip, ix, v = csr_arrays(csr)
        w = int(max(1, np.diff(ip).max()))
        e = csr.to_ell(w)
        out[f"ell/{name}/csr"] = np.concatenate([[csr.rows, csr.cols, w], ip]).astype(np.int64)
        out[f"ell/{name}/indices"], out[f"ell/{name}/values"] = ix, v
        out[f"ell/{name}/J"] = e.aux("J_indices")
        out[f"ell/{name}/V"] = e.values().astype(np.float32)

    # hyb_rules names (transform.cpp:525-557)
    csr = ref.Storage.csr(example_coo())
    rules = csr.hyb_rules(2, 2, "hyb")
    out["rules/example_c2_k2"] = np.array(
        [f"{r['name']}|{r['new_buffer']}|" + ",".join(f"{a}:{n}" for a, n in sorted(r["arrays"].items()))
         for r in rules])

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **out)
    print("wrote", os.path.join(OUT, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
