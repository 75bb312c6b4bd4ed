import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2207_04606_b200 as S
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from ab_spmm import timeit  # noqa: E402
dev = torch.device("cuda:0")
wm = S.generate_matrix("random", 4096, 4096, 0.05, 0, 0, 0, 3)
sr = S.csr_to_srbcrs(wm.to_device(dev), 8, 32)
out = {"lib": os.environ.get("STRATA_B200_LIB", "default")}
for d in (64, 128):
    X = torch.randint(-3, 4, (4096, d), device=dev).to(torch.bfloat16)
    Y = torch.empty((sr.mb * 8, d), device=dev)
    out[f"srbcrs_d{d}_us"] = round(timeit(lambda: S.srbcrs_spmm(sr, X, Y), 50) * 1e3, 2)
print(json.dumps(out))
