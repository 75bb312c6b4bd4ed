"""CUDA-graph timing of the C3 BSR SpMM (single and 12-head) for A/B builds
(STRATA_B200_LIB=...), the way bench.py times the launch-bound op."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_04606_b200 as S  # noqa: E402
from bench import _time_graph_ms  # noqa: E402

dev = torch.device("cuda:0")
m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
bs = S.csr_to_bsr(m.to_device(dev), 32)
X = torch.randint(-3, 4, (4096, 64), device=dev).to(torch.bfloat16)
Y = torch.empty((4096, 64), device=dev)
out = {"lib": os.environ.get("STRATA_B200_LIB", "default")}
out["c3_graph_us"] = round(_time_graph_ms(torch, lambda: S.bsr_spmm(bs, X, Y)) * 1e3, 3)
H = 12
Vh = torch.randint(1, 10, (H, bs.nblocks, 32, 32), device=dev).to(torch.bfloat16)
Xh = torch.randint(-3, 4, (H, 4096, 64), device=dev).to(torch.bfloat16)
Yh = torch.empty((H, 4096, 64), device=dev)
out["c3_12head_graph_us"] = round(_time_graph_ms(torch, lambda: S.bsr_spmm_batched(bs, Vh, Xh, Yh)) * 1e3, 3)
Qh = torch.randint(-3, 4, (H, 4096, 64), device=dev).to(torch.bfloat16)
Kh = torch.randint(-3, 4, (H, 4096, 64), device=dev).to(torch.bfloat16)
Sh = torch.empty((H, bs.nblocks, 32, 32), device=dev)
try:
    out["c3_sddmm_12head_graph_us"] = round(_time_graph_ms(torch, lambda: S.bsr_sddmm(bs, Qh, Kh, Sh)) * 1e3, 3)
except Exception as e:  # noqa: BLE001
    out["sddmm_error"] = str(e)[:80]
print(json.dumps(out))
