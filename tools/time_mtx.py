"""Break down the C5 Matrix Market ingest: pageable H2D of the text vs the parse call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2207_04606_b200 as S  # noqa: E402

dev = torch.device("cuda:0")
m = S.generate_matrix("powerlaw", 2449029, 2449029, 0, 0, 0, 25.3, 1)
rows = np.repeat(np.arange(m.rows, dtype=np.int64), np.diff(m.indptr)) + 1
cols = m.indices.astype(np.int64) + 1
lines = np.empty((m.nnz, 18), np.uint8)
for k in range(7):
    p10 = 10 ** (6 - k)
    lines[:, k] = (rows // p10) % 10 + 48
    lines[:, 8 + k] = (cols // p10) % 10 + 48
lines[:, 7] = lines[:, 15] = 32
lines[:, 16] = m.values.astype(np.int64) % 10 + 48
lines[:, 17] = 10
text = (f"%%MatrixMarket matrix coordinate real general\n{m.rows} {m.cols} {m.nnz}\n".encode()
        + lines.tobytes())
del lines
arr = np.frombuffer(text, np.uint8)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = torch.from_numpy(arr).to(dev)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    mm = S.read_matrix_market(text)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    pin = torch.from_numpy(arr).pin_memory()
    t3 = time.perf_counter()
    g2 = pin.to(dev, non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"pageable_h2d_ms {1e3*(t1-t0):.1f} parse_ms {1e3*(t2-t1):.1f} pin_ms {1e3*(t3-t2):.1f} pinned_h2d_ms {1e3*(t4-t3):.1f}")
    del g, mm, pin, g2

import tempfile  # noqa: E402
with tempfile.NamedTemporaryFile(suffix=".mtx", delete=False) as f:
    f.write(text)
    path = f.name
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mm = S.read_matrix_market_file(path)
    torch.cuda.synchronize()
    print(f"file_ms {1e3*(time.perf_counter()-t0):.1f}")
    del mm
os.unlink(path)
