"""Run the device format tuner (hyb c-grid + CSR) at the C1 / C2 / C5 shapes; prints one JSON
line per config with each point's median time (the §8f "c-grid" experiment)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_04606_b200 as S  # noqa: E402
from paper_2207_04606_b200 import tune as T  # noqa: E402

for name, n, avg, d in [("C1", 65536, 16.0, 32), ("C2", 232965, 567.5267, 64),
                        ("C5", 2449029, 25.3, 128)]:
    m = S.generate_matrix("powerlaw", n, n, 0, 0, 0, avg, 1)
    rep = T.run_trials("spmm", m, d, T.SearchSpace.hyb_c_grid(), repeats=5, warmup=2)
    print(json.dumps({"config": name, "best": rep.trials[rep.best].point.format,
                      "points": {t.point.format: {"ms": round(t.median_ns / 1e6, 4),
                                                  "padding": round(t.padding, 4),
                                                  "balance": round(t.balance, 2),
                                                  "correct": t.correct} for t in rep.trials}}))
