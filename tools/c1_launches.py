import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2207_04606_b200 as S
dev = torch.device("cuda:0")
m = S.generate_matrix("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
h = S.decompose_hyb(m.to_device(dev), 1, S.hyb_auto_k(m))
X = torch.randint(-3, 4, (m.cols, 32), device=dev, dtype=torch.float32)
Y = torch.empty((m.rows, 32), device=dev)
for _ in range(5): S.spmm(h, X, Y)
torch.cuda.synchronize()
print(h.schedule_info())
