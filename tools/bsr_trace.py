"""Development: per-CTA phase timestamps of the BSR SpMM kernel (library built with
-DSTRATA_BSR_TRACE; STRATA_B200_LIB=ab/trace/libstrata_b200.so python tools/bsr_trace.py).
Also times the C3 call three ways: python loop, CUDA graph of 20 calls, single launch."""
import ctypes as C
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402
from paper_2207_04606_b200._lib import lib  # noqa: E402

dev = torch.device("cuda:0")
m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
bs = S.csr_to_bsr(m.to_device(dev), 32)
X = torch.randint(-3, 4, (4096, 64), device=dev).to(torch.bfloat16)
Y = torch.empty((4096, 64), device=dev)
for _ in range(5):
    S.bsr_spmm(bs, X, Y)
torch.cuda.synchronize()
out = {}
if hasattr(lib, "strata_debug_bsr_trace"):
    buf = np.zeros((1024, 8), np.uint64)
    S.bsr_spmm(bs, X, Y)
    torch.cuda.synchronize()
    lib.strata_debug_bsr_trace(C.c_void_p(buf.ctypes.data))
    t = buf[:128, :6].astype(np.int64)
    t0 = t[:, 0].min()
    rel = t - t0
    out["phase_us_median"] = {k: float(np.median(rel[:, i]) / 1e3) for i, k in
                              enumerate(["start", "setup", "first_full", "last_full", "done", "end"])}
    out["phase_us_max"] = {k: float(rel[:, i].max() / 1e3) for i, k in
                           enumerate(["start", "setup", "first_full", "last_full", "done", "end"])}
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        S.bsr_spmm(bs, X, Y)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            S.bsr_spmm(bs, X, Y)
    g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        g.replay()
    e1.record(s)
    s.synchronize()
    out["graph_us_per_call"] = e0.elapsed_time(e1) / 200 * 1e3
    e0.record(s)
    S.bsr_spmm(bs, X, Y)
    e1.record(s)
    s.synchronize()
    out["single_launch_us"] = e0.elapsed_time(e1) * 1e3
print(json.dumps(out))
