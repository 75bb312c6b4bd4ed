#!/usr/bin/env python
"""Summarise ncu artefacts into profiles/ (tracked).

  python tools/ncu_summary.py rep  gpurun_out/prof_spmm.ncu-rep profiles/r01_v2_ncu_spmm_products.csv \
         [--traffic-key products_spmm_n1]
  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_v2_launches_products.csv

`rep` keeps the metrics the roofline/design discussion cites (DRAM bytes, L2 hit rate,
occupancy limits, warp-stall samples) and, with --traffic-key, records
dram__bytes_read.sum + dram__bytes_write.sum (bytes per launch) in profiles/traffic.json,
which bench.py reports as roofline.traffic.  `launches` folds the
`--metrics gpu__time_duration.sum` launch list into per-kernel count / mean / share.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("dram__bytes", "gpu__time_duration", "lts__t_sector_hit_rate", "l1tex__t_sector_hit_rate",
        "sm__throughput.avg.pct", "sm__warps_active", "launch__", "smsp__pcsamp_warps_issue",
        "smsp__pcsamp_sample_count", "sm__pipe_tensor", "sm__inst_executed_pipe_tc",
        "lts__t_bytes.sum", "dram__throughput", "gpu__compute_memory_throughput",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg ", "lts__throughput",
        "lts__t_bytes", "l1tex__throughput", "lts__t_sectors_srcunit_tex_op_read.sum")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def rep(path, out, traffic_key=None, kernel_index=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2 + kernel_index]
    keep = [(k, u, v) for k, u, v in zip(hdr, units, vals)
            if any(k.startswith(p) or p in k for p in KEEP) and not k.startswith("FBSP")]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit", "value"])
        w.writerow(["kernel", "", name])
        for k, u, v in keep:
            w.writerow([k, u, v])
    if traffic_key:
        d = {k: (u, v) for k, u, v in keep}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u, v = d[k]
            tot += float(v.replace(",", "")) * UNIT.get(u, 1)
        p = os.path.join(ROOT, "profiles", "traffic.json")
        j = json.load(open(p)) if os.path.exists(p) else {}
        j[traffic_key] = int(tot)
        json.dump(j, open(p, "w"), indent=1, sort_keys=True)
        print(f"{traffic_key}: {tot / 1e9:.3f} GB per launch ({os.path.basename(path)})")
    print(f"wrote {out} ({len(keep)} metrics, kernel {name[:80]})")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, vi = H.index("Kernel Name"), H.index("Metric Value")
    agg = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki]
        k = k.split("(")[0] if not k.startswith("void ") else k[5:].split("(")[0]
        agg.setdefault(k, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "mean_ns", "total_ns", "share"])
        for k, v in agg.items():
            w.writerow([k, len(v), round(sum(v) / len(v), 1), round(sum(v), 1),
                        round(sum(v) / tot, 4)])
    print(f"wrote {out} ({len(agg)} kernels)")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    key = None
    if "--traffic-key" in sys.argv:
        key = sys.argv[sys.argv.index("--traffic-key") + 1]
    if mode == "rep":
        rep(src, dst, key)
    else:
        launches(src, dst)
