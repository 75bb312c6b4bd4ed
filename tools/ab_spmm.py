"""Time hyb SpMM (C5 products shape d=128, C2 Reddit shape d=64, C1 d=32) and SDDMM (C2) with
CUDA events.  Used to A/B library builds: STRATA_B200_LIB=path python tools/ab_spmm.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda:0")
    out = {"lib": os.environ.get("STRATA_B200_LIB", "default")}
    for name, n, avg, d in [("C5", 2449029, 25.3, 128), ("C2", 232965, 567.5267, 64),
                            ("C1", 65536, 16.0, 32)]:
        m = S.generate_matrix("powerlaw", n, n, 0, 0, 0, avg, 1)
        dcsr = m.to_device(dev)
        h = S.decompose_hyb(dcsr, 1, S.hyb_auto_k(m))
        X = torch.randint(-3, 4, (m.cols, d), device=dev, dtype=torch.float32)
        Y = torch.empty((m.rows, d), device=dev)
        out[f"{name}_spmm_ms"] = round(timeit(lambda: S.spmm(h, X, Y)), 4)
        out[f"{name}_csr_ms"] = round(timeit(lambda: S.spmm_csr(dcsr, X, Y), 3), 4)
        if name == "C2":
            Xs = torch.randint(-3, 4, (m.rows, d), device=dev, dtype=torch.float32)
            Yd = torch.randint(-3, 4, (d, m.cols), device=dev, dtype=torch.float32)
            B = torch.empty((m.nnz,), device=dev)
            out["C2_sddmm_ms"] = round(timeit(lambda: S.sddmm(dcsr, Xs, Yd, B)), 4)
            for dd in (32, 128):
                Xs = torch.randint(-3, 4, (m.rows, dd), device=dev, dtype=torch.float32)
                Yd = torch.randint(-3, 4, (dd, m.cols), device=dev, dtype=torch.float32)
                out[f"C2_sddmm_d{dd}_ms"] = round(timeit(lambda: S.sddmm(dcsr, Xs, Yd, B)), 4)
        del h, X, Y, dcsr
        torch.cuda.empty_cache()
    # dense transform of the GNN layer at C5 shape (strata_gemm_f32, 3xTF32 tcgen05)
    Yg = torch.randn(2449029, 128, device=dev)
    for n_out in (128, 64):
        Wg = torch.randn(128, n_out, device=dev)
        Zg = torch.empty(2449029, n_out, device=dev)
        if hasattr(S, "gemm"):
            out[f"gemm_c5_128x{n_out}_ms"] = round(timeit(lambda: S.gemm(Yg, Wg, Zg)), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
