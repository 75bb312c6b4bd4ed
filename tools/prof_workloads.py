"""Run one BASELINE workload a few times (for ncu captures): python tools/prof_workloads.py
{products|reddit_spmm|reddit_sddmm|bsr|bsr12|bsr12_sddmm|dbsr|gnn|rgcn|srbcrs|attention}
[reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402


def main():
    which = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda:0")
    if which == "products":
        m = S.generate_matrix("powerlaw", 2449029, 2449029, 0, 0, 0, 25.3, 1)
        h = S.decompose_hyb(m.to_device(dev), 1, S.hyb_auto_k(m))
        X = torch.randint(-3, 4, (m.cols, 128), device=dev, dtype=torch.float32)
        fn = lambda: S.spmm(h, X)
    elif which.startswith("reddit"):
        m = S.generate_matrix("powerlaw", 232965, 232965, 0, 0, 0, 567.5267, 1)
        dcsr = m.to_device(dev)
        if which == "reddit_spmm":
            h = S.decompose_hyb(dcsr, 1, S.hyb_auto_k(m))
            X = torch.randint(-3, 4, (m.cols, 64), device=dev, dtype=torch.float32)
            fn = lambda: S.spmm(h, X)
        else:
            X = torch.randint(-3, 4, (m.rows, 64), device=dev, dtype=torch.float32)
            Yd = torch.randint(-3, 4, (64, m.cols), device=dev, dtype=torch.float32)
            fn = lambda: S.sddmm(dcsr, X, Yd)
    elif which == "bsr":
        m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
        bs = S.csr_to_bsr(m.to_device(dev), 32)
        X = torch.randint(-3, 4, (4096, 64), device=dev).to(torch.bfloat16)
        fn = lambda: S.bsr_spmm(bs, X)
    elif which == "bsr12":  # 12-head batched variant
        m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
        bs = S.csr_to_bsr(m.to_device(dev), 32)
        V = torch.randint(1, 10, (12, bs.nblocks, 32, 32), device=dev).to(torch.bfloat16)
        X = torch.randint(-3, 4, (12, 4096, 64), device=dev).to(torch.bfloat16)
        fn = lambda: S.bsr_spmm_batched(bs, V, X)
    elif which == "srbcrs":  # pruned-weight SR-BCRS(8, 32) (5 % unstructured), d = 128
        m = S.generate_matrix("random", 4096, 4096, 0.05, 0, 0, 0, 3)
        sr = S.csr_to_srbcrs(m.to_device(dev), 8, 32)
        X = torch.randint(-3, 4, (4096, 128), device=dev).to(torch.bfloat16)
        fn = lambda: S.srbcrs_spmm(sr, X)
    elif which == "attention":  # fused SDDMM -> softmax -> SpMM at C2, d = 64
        m = S.generate_matrix("powerlaw", 232965, 232965, 0, 0, 0, 567.5267, 1)
        plan = S.AttentionPlan(m.to_device(dev))
        Q = torch.randn(m.rows, 64, device=dev) * 0.1
        K = torch.randn(m.cols, 64, device=dev) * 0.1
        V = torch.randn(m.cols, 64, device=dev)
        fn = lambda: plan(Q, K, V)
    elif which == "rgcn":
        m = S.generate_matrix("powerlaw", 1885136, 1885136, 0, 0, 0, 3.0051, 1)
        plan = S.RgmsPlan(S.split_relations(m, 133, 1).to_device(dev))
        X = torch.randint(-3, 4, (m.cols, 32), device=dev).to(torch.bfloat16)
        W = torch.randint(-3, 4, (133, 32, 32), device=dev).to(torch.bfloat16)
        fn = lambda: plan.run(X, W)
    elif which == "bsr12_sddmm":  # 12-head block-sparse SDDMM (sparse-attention scores)
        m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
        bs = S.csr_to_bsr(m.to_device(dev), 32)
        Q = torch.randint(-3, 4, (12, 4096, 64), device=dev).to(torch.bfloat16)
        K = torch.randint(-3, 4, (12, 4096, 64), device=dev).to(torch.bfloat16)
        fn = lambda: S.bsr_sddmm(bs, Q, K)
    elif which == "dbsr":  # DBSR(32) pruned-weight SpMM, 2 % block mask, d = 128
        m = S.generate_matrix("blocksparse", 8192, 8192, 0.02, 0, 32, 0, 4)
        db = S.csr_to_dbsr(m.to_device(dev), 32)
        X = torch.randint(-3, 4, (8192, 128), device=dev).to(torch.bfloat16)
        fn = lambda: S.dbsr_spmm(db, X)
    elif which == "gnn":  # C5 GNN layer 128 -> 128: hyb SpMM then the tcgen05 3xTF32 transform
        m = S.generate_matrix("powerlaw", 2449029, 2449029, 0, 0, 0, 25.3, 1)
        h = S.decompose_hyb(m.to_device(dev), 1, S.hyb_auto_k(m))
        X = torch.randint(-3, 4, (m.cols, 128), device=dev, dtype=torch.float32)
        W = torch.randint(-3, 4, (128, 128), device=dev, dtype=torch.float32)
        fn = lambda: S.gnn_layer(h, X, W)
    else:
        raise SystemExit(f"unknown workload {which}")
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print("done", which)


if __name__ == "__main__":
    main()
