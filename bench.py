#!/usr/bin/env python
"""bench.py — hyb SpMM at ogbn-products shape on 1..8 B200 (row-sharded + NCCL all-gather).

Metric (BASELINE.json): "SpMM/SDDMM GFLOP/s & %HBM roofline at 1/2/4/8 B200 vs CPU ref".
Headline workload (BASELINE.json configs[4], the one the north_star's >=60%-of-HBM target and
the 1/2/4/8-GPU scaling are quoted on): hyb SpMM fp32, power-law graph of ogbn-products shape
(n = 2,449,029, avg degree 25.3, seed 1 -> nnz 61,943,588), d = 128, hyb:c=1 (auto k = 5).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

One step = one SpMM over this rank's nnz-balanced row shard followed (N > 1) by the NCCL
all-gather that reassembles Y on every GPU.  Inputs (X = 1.25 GB, ELL arrays 0.57 GB) are far
larger than L2 (126 MB), so no explicit L2 flush is needed between iterations.
``value`` = total FLOPs of the step (2 nnz d) / max-over-ranks device time.

The CPU baseline / --impl reference arm runs the UNMODIFIED reference interpreter
(oracle/_ref/libstrata_ref.so: build_matrix_pipeline + interpret, tune.cpp:121-146) on a bounded
row sample of the same graph; it is the only place this file touches oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMM/SDDMM GFLOP/s & %HBM roofline at 1/2/4/8 B200 vs CPU ref"
PRODUCTS = dict(kind="powerlaw", n=2449029, m=2449029, avg=25.3, seed=1, d=128)
REDDIT = dict(kind="powerlaw", n=232965, m=232965, avg=567.5267, seed=1, d=64)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j["hbm_gbs"], j.get("bf16_tflops", 1683.3), "measured"
    return 6650.0, 1590.0, "fallback"


def b_alg_spmm(nnz, m, n, d):
    """Gather-model algorithmic bytes: structure + one X row per
    non-zero + Y once."""
    return nnz * (4 + 4) + (m + 1) * 4 + nnz * d * 4 + m * d * 4


def b_min_spmm(nnz, m, n, d):
    """SURVEY §8d's B_min: the same with X read once (n rows) instead of once per non-zero."""
    return nnz * (4 + 4) + (m + 1) * 4 + n * d * 4 + m * d * 4


def b_alg_sddmm(nnz, m, n, d):
    return nnz * (4 + 4 + 4) + (m + 1) * 4 + m * d * 4 + nnz * d * 4


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every ~5 ms during the timed region
    through NVML (the library behind nvidia-smi; a 50 ms timed region still gets ~10 samples),
    with an nvidia-smi -lms 100 fallback when NVML is unavailable."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap")]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.sm, self.smax, self.reasons = [], [], set()
        self.stop_flag = threading.Event()
        self.nvml = None
        self.proc = None
        self.lines = []

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self._physical_index())
            self.nvml = (N, h)
            self.smax.append(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self._poll_once()  # one sample before the region starts (NVML is warm)
            self.sm.clear()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=index,clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [x.strip() for x in vis.split(",") if x.strip()]
            if self.gpu < len(ids) and ids[self.gpu].isdigit():
                return int(ids[self.gpu])
        return self.gpu

    def _poll_once(self):
        N, h = self.nvml
        self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
        mask = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, attr in self.REASONS:
            if mask & getattr(N, attr):
                self.reasons.add(name)

    def _poll(self):
        while not self.stop_flag.is_set():
            try:
                self._poll_once()
            except Exception:
                return
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.t.join(timeout=2)
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                    "sm_max_mhz": max(self.smax) if self.smax else None,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = [r[0] for r in self.REASONS]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                self.sm.append(float(f[1]))
                self.smax.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    self.reasons.add(name)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.smax) if self.smax else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvidia-smi"}


# ---------------------------------------------------------------------------------------
# CPU reference arm / baseline
# ---------------------------------------------------------------------------------------

def reference_sample_pipelines(m, d, rows_per_slice, nslices):
    """Row slices of the graph as standalone reference pipelines (hyb:c=1, F32).  Columns are
    compacted to those the slice touches so the X binding stays small; the interpreter's cost
    per multiply-add does not depend on the column space."""
    from oracle import ref
    pls, nnz_total = [], 0
    for s in range(nslices):
        r0 = s * rows_per_slice
        r1 = min(m.rows, r0 + rows_per_slice)
        q0, q1 = int(m.indptr[r0]), int(m.indptr[r1])
        cols = m.indices[q0:q1]
        uniq, inv = np.unique(cols, return_inverse=True)
        rr = np.repeat(np.arange(r1 - r0, dtype=np.int64), np.diff(m.indptr[r0:r1 + 1]))
        coo = ref.Coo.from_arrays(r1 - r0, max(1, uniq.size), rr, inv.astype(np.int64),
                                  m.values[q0:q1].astype(np.float64))
        pl = ref.Pipeline.matrix("spmm", coo, d, ref.F32, "hyb:c=1")
        pl.set("X", np.asarray(ref.dense_int(max(1, uniq.size) * d, 7)))
        pls.append(pl)
        nnz_total += q1 - q0
    return pls, nnz_total


def run_reference_step(pls):
    """One step: every slice interpreted concurrently (interpret() is reentrant; ctypes drops
    the GIL), wall-clock timed like tune.cpp:133-146."""
    threads = [threading.Thread(target=pl.run_timed) for pl in pls]
    t0 = time.perf_counter()
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return time.perf_counter() - t0


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_single(m, d, target_s=12.0):
    """Rank-0 CPU baseline for the device arm: the reference interpreter on one core over a
    bounded row sample (hyb refuses to run parallel: interp.cpp:21-49)."""
    from oracle import ref
    if not ref.available():
        return cpu_baseline_port(m, d)
    # calibrate the per-MAC cost on a small slice, then size the sample for ~target_s
    pls, nnz = reference_sample_pipelines(m, d, 200, 1)
    dt = run_reference_step(pls)
    per_mac = dt / max(1, nnz * d)
    rows = int(min(m.rows, max(200, target_s / per_mac / d / (m.nnz / m.rows))))
    pls, nnz = reference_sample_pipelines(m, d, rows, 1)
    dt = run_reference_step(pls)
    return {"value": round(2.0 * nnz * d / dt / 1e9, 6), "unit": "GFLOP/s", "cores": 1,
            "kind": "reference",
            "sample": f"rows [0,{rows}) of the same graph ({nnz} nnz, d={d}, hyb:c=1, F32 "
                      f"pipeline, columns compacted), one interpret() = {dt:.2f} s; "
                      f"CPU: {cpu_model()}"}


def cpu_baseline_port(m, d):
    from oracle import port
    rows = min(m.rows, 200000)
    nnz = int(m.indptr[rows])
    X = np.ones((m.cols, d), np.float32)
    t0 = time.perf_counter()
    port.spmm_csr_refnum(rows, m.indptr[:rows + 1], m.indices, m.values, X)
    dt = time.perf_counter() - t0
    return {"value": round(2.0 * nnz * d / dt / 1e9, 6), "unit": "GFLOP/s",
            "cores": os.cpu_count(), "kind": "port",
            "sample": f"rows [0,{rows}) ({nnz} nnz, d={d}) with the C restatement"}


class RefCsr:
    """CSR arrays of a graph built entirely by the reference library (oracle/_ref):
    generate_matrix (driver.cpp:365-416) + build_csr (storage.cpp:89-124)."""

    def __init__(self, cfg):
        from oracle import ref
        coo = ref.Coo.generate(cfg["kind"], cfg["n"], cfg["m"], 0.0, 0, 0, cfg["avg"], cfg["seed"])
        st = ref.Storage.csr(coo, ref.F32)
        self.coo = coo
        self.rows, self.cols = st.rows, st.cols
        self.indptr = st.aux("J_indptr")
        self.indices = st.aux("J_indices")
        self.values = st.values().astype(np.float32)
        self.nnz = int(self.indices.shape[0])


def reference_c1_full(d=32, runs=1, warm=0, X=None):
    """BASELINE configs[0] at full size on the reference's own executor: power-law 65,536 nodes,
    avg degree 16, seed 1 (1,048,664 nnz), hyb:c=1 SpMM, d = 32, F32 pipeline, X from the
    tuner's seeding (tune.cpp:108-111) unless given; build_matrix_pipeline + interpret
    (driver.cpp:173-217, interp.cpp:564-622), one core (hyb refuses to parallelise,
    interp.cpp:21-49).  Returns (median seconds per run, nnz, Y of the last run as float64)."""
    from oracle import ref
    coo = ref.Coo.generate("powerlaw", 65536, 65536, 0.0, 0, 0, 16.0, 1)
    pl = ref.Pipeline.matrix("spmm", coo, d, ref.F32, "hyb:c=1")
    pl.set("X", ref.dense_int(coo.cols * d, 7) if X is None else np.asarray(X, np.float64))
    for _ in range(warm):
        pl.run_timed()
    times, Y = [], None
    for _ in range(max(runs, 1)):
        t0 = time.perf_counter()
        Y = pl.run_sized(coo.rows * d)  # one interpret(), output copied out by the same call
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), coo.nnz, Y


def run_reference_arm(args):
    """--impl reference: the reference's own CPU executor only (oracle/_ref = the unmodified
    reference library).  Nothing from this repo's package is imported or loaded here."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libstrata_ref.so not built"}))
        return 0
    cfg = PRODUCTS
    t0 = time.time()
    m = RefCsr(cfg)  # reference generator + build_csr
    gen_s = time.time() - t0
    d = cfg["d"]
    threads = os.cpu_count() or 1
    # size each thread's slice for ~2 s of interpretation per step
    pls, nnz = reference_sample_pipelines(m, d, 200, 1)
    per_mac = run_reference_step(pls) / max(1, nnz * d)
    rows = int(max(50, 2.0 / per_mac / d / (m.nnz / m.rows)))
    pls, nnz = reference_sample_pipelines(m, d, rows, threads)
    for _ in range(args.warmup):
        run_reference_step(pls)
    times = [run_reference_step(pls) for _ in range(args.steps)]
    t = float(np.median(times))
    gflops = 2.0 * nnz * d / t / 1e9
    sample = (f"{threads} concurrent reference pipelines (hyb:c=1, F32, build_matrix_pipeline + "
              f"interpret), row slices of {rows} rows of the products-shape graph generated by "
              f"the reference ({nnz} nnz total, d={d}); median of {args.steps} steps; "
              f"CPU: {cpu_model()}")
    extra = {"generate_and_build_csr_s": round(gen_s, 2), "graph_nnz": m.nnz}
    if not args.no_extra:
        # BASELINE configs[0] (C1) at full size, the same workload the device arm times in
        # extra.c1_same_config: one core, whole graph.
        t1, nnz1, _ = reference_c1_full(runs=2, warm=1)
        extra["c1_same_config"] = {
            "workload": "hyb SpMM fp32, power-law 65,536 nodes, avg 16, seed 1, d=32, hyb:c=1",
            "nnz": nnz1, "ms": round(t1 * 1e3, 2), "gflops": round(2.0 * nnz1 * 32 / t1 / 1e9, 6),
            "cores": 1, "same_config": True,
            "how": "reference generate_matrix + build_matrix_pipeline + interpret, median of 2"}
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gflops, 6), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator, seed 1)",
        "config": {"workload": "hyb SpMM fp32, ogbn-products shape, d=128, hyb:c=1 (bounded row sample)",
                   "format": "hyb:c=1"},
        "cpu_baseline": {"value": round(gflops, 6), "unit": "GFLOP/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(gflops, 6), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "extra": extra,
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------
# device arm
# ---------------------------------------------------------------------------------------

def load_traffic(key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(key)
        except Exception:
            return None
    return None


def load_l2_peak():
    """Measured L2 read bandwidth (GB/s) of this B200 model: tools/peaks.cu (256-bit loads over
    an L2-resident buffer, every SM), committed as profiles/peaks.json.  None when absent."""
    p = os.path.join(ROOT, "profiles", "peaks.json")
    try:
        return float(json.load(open(p))["l2_read_peak_gbs"])
    except Exception:
        return None


def copy_bound_ms(torch, dev, host_in, host_out, reps=3):
    """The e2e path's floor on this box: the same pinned H2D and D2H byte counts issued
    concurrently on two streams (what strata_spmm_hyb_f32_host_batch overlaps), wall clock,
    best of `reps`."""
    d_in = torch.empty(host_in.shape, dtype=host_in.dtype, device=dev)
    d_out = torch.zeros(host_out.shape, dtype=host_out.dtype, device=dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = float("inf")
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s_in):
            d_in.copy_(host_in, non_blocking=True)
        with torch.cuda.stream(s_out):
            host_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    del d_in, d_out
    return best


def extra_reddit(S, torch, dev, stream, peak):
    """C2 (Reddit shape): hyb SpMM and CSR SDDMM, device-timed (informational)."""
    cfg = REDDIT
    l2_peak = load_l2_peak()
    m = S.generate_matrix(cfg["kind"], cfg["n"], cfg["m"], 0, 0, 0, cfg["avg"], cfg["seed"])
    d = cfg["d"]
    dcsr = m.to_device(dev)
    h = S.decompose_hyb(dcsr, 1, S.hyb_auto_k(m))
    X = torch.randint(-3, 4, (m.cols, d), device=dev, dtype=torch.float32)
    Y = torch.empty((m.rows, d), device=dev)
    Xs = torch.randint(-3, 4, (m.rows, d), device=dev, dtype=torch.float32)
    Yd = torch.randint(-3, 4, (d, m.cols), device=dev, dtype=torch.float32)
    B = torch.empty((m.nnz,), device=dev)
    out = {}
    for name, fn, flops, bytes_ in [
            ("reddit_hyb_spmm", lambda: S.spmm(h, X, Y), 2.0 * m.nnz * d, b_alg_spmm(m.nnz, m.rows, m.cols, d)),
            ("reddit_sddmm", lambda: S.sddmm(dcsr, Xs, Yd, B), 2.0 * m.nnz * d + m.nnz,
             b_alg_sddmm(m.nnz, m.rows, m.cols, d))]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = bytes_ / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 4), "gflops": round(flops / (ms * 1e-3) / 1e9, 2),
                     "b_alg_gbs": round(gbs, 1), "frac_of_hbm": round(gbs / peak, 3),
                     "note": "X is L2-resident (59.6 MB < 126 MB L2): frac is L2-assisted"}
        if l2_peak:  # the gathers' real ceiling: measured L2 read bandwidth
            out[name]["frac_of_l2_peak"] = round(gbs / l2_peak, 3)
        if name == "reddit_hyb_spmm":  # also B_min (X read once)
            out[name]["b_min_frac_of_hbm"] = round(
                b_min_spmm(m.nnz, m.rows, m.cols, d) / (ms * 1e-3) / 1e9 / peak, 3)
    out["reddit_nnz"] = m.nnz
    # Fused SDDMM -> edge softmax -> SpMM (GAT-style layer step), d = 64.
    plan = S.AttentionPlan(dcsr)
    Qa = torch.randn(m.rows, d, device=dev) * 0.1
    Ka = torch.randn(m.cols, d, device=dev) * 0.1
    Va = torch.randn(m.cols, d, device=dev)
    Za = torch.empty((m.rows, d), device=dev)
    ms_a = _time_ms(torch, stream, lambda: plan(Qa, Ka, Va, Za), reps=10)
    b_a = m.nnz * 8 + 2.0 * m.nnz * d * 4 + 2.0 * m.rows * d * 4 + (m.rows + 1) * 4
    out["reddit_fused_attention"] = {
        "ms": round(ms_a, 4), "gflops": round(4.0 * m.nnz * d / (ms_a * 1e-3) / 1e9, 1),
        "b_alg_gbs": round(b_a / (ms_a * 1e-3) / 1e9, 1),
        "note": "one pass (online softmax); K, V rows gathered per edge, L2-resident at C2"}
    if l2_peak:
        out["reddit_fused_attention"]["frac_of_l2_peak"] = round(b_a / (ms_a * 1e-3) / 1e9 / l2_peak, 3)
    if l2_peak:
        out["l2_read_peak_gbs"] = {"value": l2_peak, "source": "profiles/peaks.json (tools/peaks.cu)"}
    # The reference tuner's c-grid (tune.cpp:19-36) on the device: csr + hyb(c in 1..16) timed,
    # gated bitwise against the CSR format on integer operands.
    from paper_2207_04606_b200 import tune as T
    rep = T.run_trials("spmm", m, d, T.SearchSpace.hyb_c_grid(), repeats=5, warmup=2)
    out["reddit_tuner"] = {"best": rep.trials[rep.best].point.format,
                           "ms": {t.point.format: round(t.median_ns / 1e6, 4) for t in rep.trials},
                           "all_correct": all(t.correct for t in rep.trials)}
    return out


def extra_sddmm_sharded(S, torch, dist, dev, stream, rank, world, comm):
    """N > 1: BASELINE configs[1]'s SDDMM (C2, d = 64) row-sharded through the native plan —
    each rank computes its contiguous nnz range, then the ranges are all-gathered (grouped
    ncclBroadcast) so every rank holds B[nnz]; device time max over ranks."""
    from paper_2207_04606_b200.sharding import ShardPlan
    cfg = REDDIT
    m = S.generate_matrix(cfg["kind"], cfg["n"], cfg["m"], 0, 0, 0, cfg["avg"], cfg["seed"])
    d = cfg["d"]
    dcsr = m.to_device(dev)
    plan = ShardPlan(dcsr, rank, world, chunks=1, stream=stream)
    g = torch.Generator(device=dev)
    g.manual_seed(2)
    Xs = torch.randint(-3, 4, (m.rows, d), device=dev, dtype=torch.float32, generator=g)
    Yd = torch.randint(-3, 4, (d, m.cols), device=dev, dtype=torch.float32, generator=g)
    B = torch.empty((m.nnz,), device=dev)
    out = {}
    for name, gather in (("gathered", True), ("compute_only", False)):
        for _ in range(3):
            plan.sddmm(Xs, Yd, B, gather=gather, comm=comm, stream=stream)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):
            plan.sddmm(Xs, Yd, B, gather=gather, comm=comm, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        out[name + "_ms"] = round(ms, 4)
        out[name + "_gflops"] = round((2.0 * m.nnz * d + m.nnz) / (ms * 1e-3) / 1e9, 1)
    ref = S.sddmm(dcsr, Xs, Yd)
    plan.sddmm(Xs, Yd, B, gather=True, comm=comm, stream=stream)
    torch.cuda.synchronize()
    ok = torch.tensor([1 if torch.equal(B, ref) else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    out["equals_single_gpu"] = bool(int(ok[0]))
    out["nnz"] = m.nnz
    return out


def _time_ms(torch, stream, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _time_graph_ms(torch, fn, calls=20, reps=10):
    """Per-call device time of a launch-bound op replayed from a CUDA graph of `calls`
    back-to-back calls (captured on a side stream; CUDA events around `reps` replays)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(calls):
                fn()
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        s.synchronize()
    return e0.elapsed_time(e1) / (reps * calls)


def extra_gnn_layer(S, torch, dev, stream, h, X, nnz, spmm_ms):
    """GNN layer step Z = A @ X @ W at C5 shape (GraphSAGE/GCN layer):
    hyb SpMM + fp32 cuBLAS SGEMM (pedantic fp32), associated so the SpMM gathers the narrower
    rows.  Integer operands, so the layer is exact."""
    out = {}
    rows, d_in = h.rows, X.shape[1]
    for d_out in (128, 64):
        W = torch.randint(-3, 4, (d_in, d_out), device=dev).to(torch.float32)
        Z = torch.empty((rows, d_out), device=dev)
        work = torch.empty(max(S.gnn_layer_work_floats(h, d_in, d_out), 1), device=dev)
        ms = _time_ms(torch, stream, lambda: S.gnn_layer(h, X, W, Z, work, stream=stream))
        agg_d = d_out if d_out < d_in else d_in
        flops = 2.0 * nnz * agg_d + 2.0 * (h.cols if d_out < d_in else rows) * d_in * d_out
        out[f"c5_gnn_layer_{d_in}x{d_out}"] = {
            "ms": round(ms, 4), "gflops": round(flops / (ms * 1e-3) / 1e9, 1),
            "order": "A@(X@W)" if d_out < d_in else "(A@X)@W",
            "spmm_alone_ms_d128": round(spmm_ms, 4)}
        del W, Z, work
    return out


def extra_tensor_core(S, torch, dev, stream, hbm_peak, bf16_peak):
    """C3 (BSR sparse attention, bf16, tcgen05) and C4 (RGCN, AM shape, tcgen05)."""
    out = {}
    # C3: blocksparse 4096^2, b = 32, density 0.1, seed 1; head dim 64 (and a 12-head batch).
    m = S.generate_matrix("blocksparse", 4096, 4096, 0.1, 0, 32, 0, 1)
    bs = S.csr_to_bsr(m.to_device(dev), 32)
    d = 64
    X = torch.randint(-3, 4, (4096, d), device=dev).to(torch.bfloat16)
    Y = torch.empty((4096, d), device=dev)
    ms_loop = _time_ms(torch, stream, lambda: S.bsr_spmm(bs, X, Y))
    ms = _time_graph_ms(torch, lambda: S.bsr_spmm(bs, X, Y))
    flops = 2.0 * bs.nblocks * 32 * 32 * d
    b_alg = bs.nblocks * 32 * 32 * 2 + bs.nblocks * 4 + 129 * 4 + bs.nblocks * 32 * d * 2 + 4096 * d * 4
    out["c3_bsr_spmm"] = {"ms": round(ms, 5), "gflops": round(flops / (ms * 1e-3) / 1e9, 1),
                          "blocks": bs.nblocks, "tensor_frac": round(flops / (ms * 1e-3) / 1e12 / bf16_peak, 5),
                          "hbm_frac": round(b_alg / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                          "python_loop_ms": round(ms_loop, 5),
                          "timing": "CUDA graph of 20 back-to-back calls (launch-bound op); "
                                    "python_loop_ms = ctypes call per launch",
                          "note": "208 MFLOP over 10.8 MB: launch/latency-bound by construction"}
    # 12-head batched variant: heads share the mask, own values and features.
    H = 12
    Vh = torch.randint(1, 10, (H, bs.nblocks, 32, 32), device=dev).to(torch.bfloat16)
    Xh = torch.randint(-3, 4, (H, 4096, d), device=dev).to(torch.bfloat16)
    Yh = torch.empty((H, 4096, d), device=dev)
    msh = _time_graph_ms(torch, lambda: S.bsr_spmm_batched(bs, Vh, Xh, Yh))
    flops_h = H * flops
    # B_min: every head's block values, X and Y move once; the gather model charges a 32 x d
    # X tile per stored block, most of which are L2 re-reads (ncu: 45 MB DRAM per call).
    b_min_h = H * (bs.nblocks * 32 * 32 * 2 + 4096 * d * 2 + 4096 * d * 4) + bs.nblocks * 4 + 129 * 4
    b_alg_h = H * (bs.nblocks * 32 * 32 * 2 + bs.nblocks * 32 * d * 2 + 4096 * d * 4) + bs.nblocks * 4 + 129 * 4
    out["c3_bsr_spmm_12head"] = {"ms": round(msh, 5), "gflops": round(flops_h / (msh * 1e-3) / 1e9, 1),
                                 "tensor_frac": round(flops_h / (msh * 1e-3) / 1e12 / bf16_peak, 5),
                                 "hbm_frac": round(b_min_h / (msh * 1e-3) / 1e9 / hbm_peak, 4),
                                 "bytes_model": "B_min = heads*(blocks*2KB + 4096*d*2 + 4096*d*4)",
                                 "hbm_frac_gather_model_l2_assisted":
                                     round(b_alg_h / (msh * 1e-3) / 1e9 / hbm_peak, 4)}
    # 12-head block-sparse SDDMM (sparse-attention scores) on tcgen05, C3 mask.
    Qh = torch.randint(-3, 4, (H, 4096, d), device=dev).to(torch.bfloat16)
    Kh = torch.randint(-3, 4, (H, 4096, d), device=dev).to(torch.bfloat16)
    Sh = torch.empty((H, bs.nblocks, 32, 32), device=dev)
    ms_sd = _time_graph_ms(torch, lambda: S.bsr_sddmm(bs, Qh, Kh, Sh))
    fl_sd = H * bs.nblocks * 2.0 * 32 * 32 * d
    # B_min: the mask's block values (f32, shared by the heads) once, per head S out, Q and K
    # once; the gather model charges a 32 x d K tile per stored block (L2 re-reads).
    b_sd = bs.nblocks * 32 * 32 * 4 + H * (bs.nblocks * 32 * 32 * 4 + 2 * 4096 * d * 2)
    b_sd_g = bs.nblocks * 32 * 32 * 4 + H * (bs.nblocks * 32 * 32 * 4 + bs.nblocks * 32 * d * 2 + 4096 * d * 2)
    out["c3_bsr_sddmm_12head"] = {"ms": round(ms_sd, 5), "gflops": round(fl_sd / (ms_sd * 1e-3) / 1e9, 1),
                                  "tensor_frac": round(fl_sd / (ms_sd * 1e-3) / 1e12 / bf16_peak, 5),
                                  "hbm_frac": round(b_sd / (ms_sd * 1e-3) / 1e9 / hbm_peak, 4),
                                  "bytes_model": "B_min = blocks*4KB (A, shared) + heads*(blocks*4KB S out + 4096*d*2 Q + 4096*d*2 K)",
                                  "hbm_frac_gather_model_l2_assisted":
                                      round(b_sd_g / (ms_sd * 1e-3) / 1e9 / hbm_peak, 4),
                                  "timing": "CUDA graph of 20 calls"}
    # Pruned-weight formats: a 4096 x 4096 weight pruned
    # to 5 % density (unstructured, "random") as SR-BCRS(8, 32) and a 2 %-dense block mask as
    # DBSR(32), d = 128, tcgen05.
    wm = S.generate_matrix("random", 4096, 4096, 0.05, 0, 0, 0, 3)
    sr = S.csr_to_srbcrs(wm.to_device(dev), 8, 32)
    Xw = torch.randint(-3, 4, (4096, 128), device=dev).to(torch.bfloat16)
    Yw = torch.empty((sr.mb * 8, 128), device=dev)
    ms_sr = _time_graph_ms(torch, lambda: S.srbcrs_spmm(sr, Xw, Yw))
    slots = sr.groups * 32 * 8
    out["srbcrs_8_32_spmm"] = {"ms": round(ms_sr, 5), "nnz": wm.nnz, "stored_slots": slots,
                               "gflops_useful": round(2.0 * wm.nnz * 128 / (ms_sr * 1e-3) / 1e9, 1),
                               "tensor_tflops_issued": round(2.0 * sr.groups * 32 * 16 * 128 / (ms_sr * 1e-3) / 1e12, 2),
                               "timing": "CUDA graph of 20 calls"}
    bm = S.generate_matrix("blocksparse", 8192, 8192, 0.02, 0, 32, 0, 4)
    db = S.csr_to_dbsr(bm.to_device(dev), 32)
    Xd = torch.randint(-3, 4, (8192, 128), device=dev).to(torch.bfloat16)
    Yd2 = torch.empty((8192, 128), device=dev)
    ms_db = _time_graph_ms(torch, lambda: S.dbsr_spmm(db, Xd, Yd2))
    out["dbsr_32_spmm"] = {"ms": round(ms_db, 5), "blocks": db.nblocks, "stored_block_rows": db.nstored,
                           "block_rows": db.mb,
                           "gflops": round(2.0 * db.nblocks * 1024 * 128 / (ms_db * 1e-3) / 1e9, 1),
                           "timing": "CUDA graph of 20 calls"}
    # C4: AM-shaped power-law graph split into 133 relations, d_in = d_out = 32.
    g = S.generate_matrix("powerlaw", 1885136, 1885136, 0, 0, 0, 3.0051, 1)
    rel = S.split_relations(g, 133, 1).to_device(dev)
    t0 = time.time()
    plan = S.RgmsPlan(rel)
    torch.cuda.synchronize()
    plan_first_ms = (time.time() - t0) * 1e3  # includes lazy module loading / pool growth
    del plan
    t0 = time.time()
    plan = S.RgmsPlan(rel)
    torch.cuda.synchronize()
    plan_ms = (time.time() - t0) * 1e3
    Xr = torch.randint(-3, 4, (g.cols, 32), device=dev).to(torch.bfloat16)
    W = torch.randint(-3, 4, (133, 32, 32), device=dev).to(torch.bfloat16)
    Yr = torch.empty((g.rows, 32), device=dev)
    ms = _time_ms(torch, stream, lambda: plan.run(Xr, W, Yr), reps=10)
    flops = 2.0 * g.nnz * 32 * 32
    b_onchip = g.nnz * (4 + 4 + 2) + g.nnz * 32 * 2 + 133 * 32 * 32 * 2 + g.rows * 32 * 4
    # two-pass model actually executed: (src, pos, A) + X row gather + message-row write, then
    # message-row read + dptr + Y; message rows = the plan's (relation, destination) runs of
    # rows with >= 2 runs (a row's sole run goes to Y from pass 1: counted in m*d_out*4)
    runs = plan.message_rows
    b_2pass = g.nnz * 12 + g.nnz * 32 * 2 + runs * 32 * 4 * 2 + (g.rows + 1) * 4 + g.rows * 32 * 4
    out["c4_rgcn"] = {"ms": round(ms, 4), "gflops": round(flops / (ms * 1e-3) / 1e9, 1),
                      "nnz": g.nnz, "plan_ms": round(plan_ms, 1),
                      "plan_first_call_ms": round(plan_first_ms, 1),
                      "tensor_frac": round(flops / (ms * 1e-3) / 1e12 / bf16_peak, 5),
                      "hbm_frac_onchip_model": round(b_onchip / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                      "hbm_frac_two_pass_model": round(b_2pass / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                      "message_rows": runs,
                      "bytes_model": "on-chip: nnz*10 + nnz*d_in*2 + R*d_in*d_out*2 + m*d_out*4 "
                                     "(661 MB); two-pass: nnz*12 + nnz*d_in*2 + 2*runs*d_out*4 "
                                     "+ (m+1)*4 + m*d_out*4"}
    return out


def extra_mtx_ingest(S, torch, dev):
    """Device Matrix Market ingest: the C5 graph (61.9 M entries, values
    1..9 as the reference writer prints them) as text in host memory -> strata_mtx_parse
    (newline scan + per-line parse on the GPU) -> strata_csr_from_coo; wall clock, warm."""
    m = S.generate_matrix("powerlaw", 2449029, 2449029, 0, 0, 0, 25.3, 1)
    # entry lines "RRRRRRR CCCCCCC V\n": 7-digit zero-padded indices (istream reads leading
    # zeros as the same integer), built with vectorised digit arithmetic
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
    del rows, cols
    text = (f"%%MatrixMarket matrix coordinate real general\n{m.rows} {m.cols} {m.nnz}\n".encode()
            + lines.tobytes())
    del lines
    out = {"bytes": len(text), "entries": m.nnz}
    parse_s, csr_s = [], []
    for rep in range(4):  # first call warms the pinned ring and the pool; best of the rest
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mm = S.read_matrix_market(text)
        t1 = time.perf_counter()
        csr = mm.to_csr(dev)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if rep:
            parse_s.append(t1 - t0)
            csr_s.append(t2 - t1)
        ok = bool(torch.equal(csr.indptr.cpu(), torch.from_numpy(m.indptr))) and \
            bool(torch.equal(csr.indices.cpu(), torch.from_numpy(m.indices)))
        del mm, csr
    out.update({"parse_ms": round(min(parse_s) * 1e3, 1), "parse_ms_reps": [round(x * 1e3, 1) for x in parse_s],
                "csr_ms": round(min(csr_s) * 1e3, 1),
                "parse_gbs": round(len(text) / min(parse_s) / 1e9, 2), "csr_equals_generator": ok,
                "note": "text in pageable host memory: the H2D copy of the entry region is inside "
                        "(wall clock, best of 3 warm calls)"})
    # read_matrix_market_file (mmio.cpp:57-61): the same text from a file (page cache warm)
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".mtx", delete=False) as f:
        f.write(text)
        path = f.name
    try:
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mm = S.read_matrix_market_file(path)
            torch.cuda.synchronize()
            file_ms = (time.perf_counter() - t0) * 1e3
            del mm
        out["file_ms"] = round(file_ms, 1)
    finally:
        os.unlink(path)
    # The reference's parser (oracle/_ref: mmio.cpp:17-55, istream per line) on a 2M-line
    # prefix of the same text, one core: its line rate and the full-text estimate.
    try:
        from oracle import ref
        k = 2_000_000
        head = f"%%MatrixMarket matrix coordinate real general\n{m.rows} {m.cols} {k}\n".encode()
        body_off = text.index(b"\n", text.index(b"\n") + 1) + 1
        sample = head + text[body_off: body_off + 18 * k]
        t0 = time.perf_counter()
        coo = ref.Coo.read_matrix_market(sample)
        t_ref = time.perf_counter() - t0
        assert coo.nnz == k
        out["reference_sample"] = {"lines": k, "ms": round(t_ref * 1e3, 1), "cores": 1,
                                   "full_text_est_ms": round(t_ref * 1e3 * m.nnz / k, 0),
                                   "speedup_vs_parse_est": round(t_ref * 1e3 * m.nnz / k / out["parse_ms"], 1)}
    except Exception as e:  # informational only (no oracle/_ref on this box)
        out["reference_sample"] = {"unavailable": str(e)[:200]}
    return out


def extra_c1_same_config(S, torch, dev, stream):
    """BASELINE configs[0] (C1) end to end on both executors, same workload, same operands:
    power-law 65,536 nodes, avg 16, seed 1 (1,048,664 nnz), hyb:c=1 (k=5), d = 32, X from the
    tuner's seeding (tune.cpp:108-111).  Device: decompose + SpMM through the C ABI (kernel time
    by CUDA events; e2e with host X in / host Y out per call).  Reference: the unmodified
    interpreter (oracle/_ref) on one core, timed around interpret(); its Y is compared bitwise."""
    from oracle import ref
    d = 32
    m = S.generate_matrix("powerlaw", 65536, 65536, 0, 0, 0, 16.0, 1)
    h = S.decompose_hyb(m.to_device(dev), 1, S.hyb_auto_k(m))
    Xh = torch.from_numpy(S.dense_int((m.cols, d), 7)).pin_memory()
    X = Xh.to(dev)
    Y = torch.empty((m.rows, d), device=dev)
    ms = _time_ms(torch, stream, lambda: S.spmm(h, X, Y, stream=stream), reps=50)
    Yh = torch.empty((m.rows, d)).pin_memory()
    S.spmm_host(h, Xh, Yh, stream=stream)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        S.spmm_host(h, Xh, Yh, stream=stream)
    e2e_ms = (time.perf_counter() - t0) / reps * 1e3
    flops = 2.0 * m.nnz * d
    out = {"workload": "hyb SpMM fp32, power-law 65,536 nodes, avg 16, seed 1, d=32, hyb:c=1",
           "nnz": m.nnz, "device_ms": round(ms, 5), "device_gflops": round(flops / ms / 1e6, 2),
           "e2e_ms": round(e2e_ms, 4), "e2e_gflops": round(flops / e2e_ms / 1e6, 2),
           "e2e_path": "strata_spmm_hyb_f32_host (pinned X in, Y out, one call per step)",
           "same_config": True}
    if ref.available():
        t_ref, nnz_ref, y_ref = reference_c1_full(runs=1, X=Xh.numpy())
        out.update({"reference_ms": round(t_ref * 1e3, 2), "reference_cores": 1,
                    "reference_nnz": nnz_ref,
                    "ratio_device": round(t_ref * 1e3 / ms, 1),
                    "ratio_e2e": round(t_ref * 1e3 / e2e_ms, 1),
                    "bitwise_equal_to_reference": bool(np.array_equal(
                        Yh.numpy().ravel(), y_ref.astype(np.float32)))})
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:  # main() re-execs through torch.distributed.run; never relabel N
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    # STRATA_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 with a gloo group, so the
    # N > 1 code path (sharding, IPC peer stores, fallbacks) runs on a one-GPU box.
    share = os.environ.get("STRATA_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2207_04606_b200 as S

    hbm_peak, bf16_peak, peak_kind = load_peaks()
    cfg = PRODUCTS
    d = cfg["d"]
    t0 = time.time()
    m = S.generate_matrix(cfg["kind"], cfg["n"], cfg["m"], 0, 0, 0, cfg["avg"], cfg["seed"])
    gen_s = time.time() - t0
    k = S.hyb_auto_k(m)
    from paper_2207_04606_b200.sharding import NcclComm, PeerAllGather, RowShardPlan, ShardPlan
    # The native row-partitioned plan (strata_shard_plan_create): this rank's nnz-balanced row
    # range, cut into chunks, each decomposed to hyb on this GPU; X replicated, Y a full
    # replica on every rank.  N > 1 reassembly (--allgather):
    #   p2p (default)  strata_spmm_hyb_f32_sharded_p2p — the SpMM stores every finished row into
    #                  all ranks' replicas over NVLink (CUDA IPC), verified once against nccl;
    #   nccl           strata_spmm_hyb_f32_sharded with an NCCL communicator made by the C ABI —
    #                  per chunk a grouped ncclBroadcast from every owner (an uneven all-gather),
    #                  overlapping the next chunk's SpMM on the plan's stream.
    p2p = world > 1 and args.allgather == "p2p"
    chunks = 4 if (world > 1 and not p2p) else 1
    stream = torch.cuda.current_stream()
    t0 = time.time()
    dcsr = m.to_device(dev)  # the full CSR on every rank (the plan slices it)
    torch.cuda.synchronize()
    up_s = time.time() - t0
    t0 = time.time()
    plan = ShardPlan(dcsr, rank, world, chunks=chunks, c=1, k=k, stream=stream)
    torch.cuda.synchronize()
    plan_s = time.time() - t0
    r0, r1 = plan.rows_of(rank)
    shard = RowShardPlan(m, world).shard(rank)  # the same cuts, host copy for the byte model
    # The shard's decomposition alone, first and warm (second) call, for the plan-cost record.
    dsh = shard.to_device(dev)
    torch.cuda.synchronize()
    t0 = time.time()
    h = S.decompose_hyb(dsh, 1, k)
    torch.cuda.synchronize()
    decomp_s = time.time() - t0
    h_warm = S.decompose_hyb(dsh, 1, k)  # second plan beside the first (fresh allocations)
    torch.cuda.synchronize()
    h_warm.close()
    torch.cuda.synchronize()
    t0 = time.time()  # rebuild after release: the warm plan cost
    h_warm = S.decompose_hyb(dsh, 1, k)
    torch.cuda.synchronize()
    decomp_warm_s = time.time() - t0
    del h_warm, dsh
    sched = h.schedule_info()
    launches_per_step = sched["launches_per_spmm"] * chunks

    # X replicated on every rank (BASELINE: "dense features replicated"); integer operands in
    # [-3, 3] like the reference tuner's (tune.cpp:108-111).
    gx = torch.Generator(device=dev)
    gx.manual_seed(1)
    X = torch.randint(-3, 4, (m.cols, d), device=dev, dtype=torch.float32, generator=gx)
    Yrep = torch.empty((m.rows, d), device=dev, dtype=torch.float32)
    # NCCL refuses two ranks on one device: the shared-GPU test mode runs p2p only.
    comm, comm_note = None, None
    if world > 1 and not share:
        try:
            comm = NcclComm(rank, world)
        except Exception as e:  # noqa: BLE001 — p2p still runs; its check uses a local SpMM
            comm_note = f"NCCL communicator unavailable ({e})"
    if comm is None and world > 1 and not p2p:
        print(f"bench.py: --allgather nccl needs an NCCL communicator ({comm_note or 'shared GPU'})",
              file=sys.stderr)
        return 2

    pag, p2p_note = None, None
    if p2p:
        try:
            pag = PeerAllGather(Yrep, rank, world)
            # one-time check against the NCCL path (bitwise), then fall back if it differs
            Ychk = torch.empty_like(Yrep)
            if comm is not None:
                plan.spmm(X, Ychk, comm, stream=stream)
            else:  # shared-GPU test mode: the single-GPU SpMM of the whole graph
                S.spmm(S.decompose_hyb(dcsr, 1, k), X, Ychk, stream=stream)
            plan.spmm_p2p(X, pag.dsts(0), d, stream=stream)
            pag.fence()
            torch.cuda.synchronize()
            ok = torch.tensor([1 if torch.equal(Yrep, Ychk) else 0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            del Ychk
            if int(ok[0]) != 1:
                raise RuntimeError("peer all-gather differs from the NCCL all-gather")
        except Exception as e:  # noqa: BLE001 — fall back to the NCCL collective
            p2p_note = f"p2p unavailable ({e}); NCCL all-gather used"
            pag = None
            p2p = False

    def step():
        if pag is not None:
            plan.spmm_p2p(X, pag.dsts(0), d, stream=stream)
            pag.fence()
        else:
            plan.spmm(X, Yrep, comm, stream=stream)

    def compute_only():  # the same kernels, no reassembly (this rank's rows)
        plan.spmm(X, Yrep, None, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_start.record(stream)
    for i in range(args.steps):
        step()
    e_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = e_start.elapsed_time(e_end)
    # compute-only launches, CUDA events around each (the kernel time of the roofline)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for a_, b_ in ev:
        a_.record(stream)
        compute_only()
        b_.record(stream)
    torch.cuda.synchronize()
    spmm_ms = float(np.mean([a_.elapsed_time(b_) for a_, b_ in ev]))
    t = torch.tensor([total_ms, spmm_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, spmm_ms_max = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    flops = 2.0 * m.nnz * d
    gflops = flops / (ms_per_step * 1e-3) / 1e9
    sddmm_sharded = None
    if comm is not None and not args.no_extra:
        try:
            sddmm_sharded = extra_sddmm_sharded(S, torch, dist, dev, stream, rank, world, comm)
        except Exception as e:  # informational only
            sddmm_sharded = {"error": str(e)}

    # roofline of the dominant kernel on this rank's shard
    b_alg = b_alg_spmm(shard.nnz, shard.rows, m.cols, d)
    achieved = b_alg / (spmm_ms * 1e-3) / 1e9
    traffic = load_traffic(f"products_spmm_n{world}")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
            "peak_kind": peak_kind, "kernel": "spmm_hyb_kernel (+ split-run fix-up)",
            "kernel_ms": round(spmm_ms, 4),
            "algorithmic_bytes_per_launch": int(b_alg),
            "bytes_model": "nnz*8 + (m+1)*4 + nnz*d*4 (one X row per non-zero) + m*d*4",
            # B_min (X read once): how far the step is from perfect X reuse, which at C5 (X
            # 1.25 GB, 10x L2) no schedule can approach
            "b_min_bytes": int(b_min_spmm(shard.nnz, shard.rows, m.cols, d)),
            "b_min_frac": round(b_min_spmm(shard.nnz, shard.rows, m.cols, d) / (spmm_ms * 1e-3) / 1e9 / hbm_peak, 4)}
    if traffic:  # measured DRAM bytes (ncu, profiles/) over the same launch time: frac > 1 on
        # the algorithmic model means L2 served part of the X gathers (~10 % at C5)
        roof["dram_traffic_frac"] = round(traffic / 1e9 / (spmm_ms * 1e-3) / hbm_peak, 4)

    # e2e: same metric through the C ABI with host buffers (pinned), copies inside the region:
    # strata_spmm_hyb_f32_host = H2D of X, the shard SpMM, D2H of this rank's rows.
    h_e2e = h  # this rank's shard as one hyb
    # Batched form (strata_spmm_hyb_f32_host_batch): e2e_steps independent feature matrices,
    # each copied in from pinned host memory and its Y copied back; copy-in of step b+1 and
    # copy-out of step b-1 overlap step b's SpMM.  Two host buffer pairs alternate.
    Xh = [X.cpu().pin_memory() for _ in range(2)]
    Yh = [torch.empty((r1 - r0, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    # the same K steps as the device-timed region (pipeline fill/drain amortised over K)
    e2e_steps = max(2, min(args.steps, 64))
    xs = [Xh[b % 2] for b in range(e2e_steps)]
    ys = [Yh[b % 2] for b in range(e2e_steps)]
    S.spmm_host_batch(h_e2e, xs[:2], ys[:2], stream=stream)  # warm staging buffers
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    S.spmm_host_batch(h_e2e, xs, ys, stream=stream)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # unpipelined single call for reference
    t0 = time.perf_counter()
    S.spmm_host(h_e2e, Xh[0], Yh[0], stream=stream)
    single_ms = (time.perf_counter() - t0) * 1e3
    floor_ms = copy_bound_ms(torch, dev, Xh[0], Yh[1])
    e2e = {"value": round(flops / float(te[0]) / 1e9, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(Xh[0].numel() * 4), "d2h_bytes_per_step": int(Yh[0].numel() * 4),
           "ms_per_step": round(float(te[0]) * 1e3, 3), "steps": e2e_steps,
           "single_call_ms": round(single_ms, 3),
           "copy_bound_ms": round(floor_ms, 3),
           "frac_of_copy_bound": round(floor_ms / (float(te[0]) * 1e3), 4),
           "copy_bound_note": "the same pinned H2D + D2H bytes issued concurrently on two "
                              "streams, no compute (the link's bidirectional floor)",
           "path": "strata_spmm_hyb_f32_host_batch (pinned host X in, host Y rows out, per "
                   "step; copy-in/compute/copy-out pipelined across steps, wall clock)"}
    del Xh, Yh

    cpu = None
    extra = {"generate_s": round(gen_s, 2), "csr_upload_ms": round(up_s * 1e3, 1),
             "shard_plan_ms": round(plan_s * 1e3, 1),
             "decompose_ms": round(decomp_s * 1e3, 1),
             "decompose_warm_ms": round(decomp_warm_s * 1e3, 1),
             "hyb_parts_rows": [P.nrows for P in h.parts],
             "padding_ratio": round(h.padding_ratio, 5),
             "schedule": sched, "spmm_ms_max_over_ranks": round(spmm_ms_max, 4),
             "allgather_exposed_ms": round(ms_per_step - spmm_ms_max, 4) if world > 1 else 0.0,
             "chunks_per_rank": chunks,
             "allgather": ("none" if world == 1 else ("p2p" if pag is not None else "nccl")),
             "allgather_note": p2p_note or comm_note,
             "compute_only_gflops": round(flops / (spmm_ms_max * 1e-3) / 1e9, 2),
             "frac_of_8tbs_nameplate": round(achieved / 8000.0, 4)}
    if sddmm_sharded is not None:
        extra["sddmm_sharded_c2"] = sddmm_sharded
    if rank == 0 and world == 1 and not args.no_extra:
        try:
            extra.update(extra_reddit(S, torch, dev, stream, hbm_peak))
        except Exception as e:  # informational only
            extra["reddit_error"] = str(e)
        try:
            extra.update(extra_gnn_layer(S, torch, dev, stream, h, X, m.nnz, spmm_ms))
        except Exception as e:  # informational only
            extra["gnn_layer_error"] = str(e)
        try:
            extra.update(extra_tensor_core(S, torch, dev, stream, hbm_peak, bf16_peak))
        except Exception as e:  # informational only
            extra["tensor_core_error"] = str(e)
    if rank == 0 and world == 1 and not args.no_extra:
        try:
            extra["c1_same_config"] = extra_c1_same_config(S, torch, dev, stream)
        except Exception as e:  # informational only
            extra["c1_error"] = str(e)
        try:
            extra["c5_mtx_ingest"] = extra_mtx_ingest(S, torch, dev)
        except Exception as e:  # informational only
            extra["mtx_error"] = str(e)
    if rank == 0 and not args.no_cpu_baseline:  # every N: the other ranks wait at the barrier
        try:
            cpu = cpu_baseline_single(m, d)
        except Exception as e:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}"}
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generator: powerlaw, seed 1; X integer in [-3,3])",
            "config": {"workload": "hyb SpMM fp32, ogbn-products shape (n=2,449,029, "
                                   "nnz=61,943,588, d=128), hyb:c=1,k=5",
                       "format": f"hyb:c=1,k={k}", "nnz": m.nnz, "rows": m.rows, "d": d,
                       "parallelism": ("single GPU" if world == 1 else
                                       f"row-sharded x{world} (nnz-balanced) + " +
                                       ("fused peer-store all-gather (NVLink, CUDA IPC)" if pag is not None
                                        else "NCCL grouped-broadcast all-gather (4 chunks overlapped)")),
                       "l2": "no flush: inputs larger than L2 (X 1.25 GB, ELL 0.57 GB)"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks, "extra": extra,
        }
        print(json.dumps(line))
    if pag is not None:
        pag.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--allgather", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 reassembly of Y: fused peer stores (p2p) or NCCL all-gather")
    args = ap.parse_args()
    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        return 2
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # One process per GPU: re-launch this command under torch.distributed.run so that
        # `python bench.py --gpus N` really runs N ranks (never a 1-GPU run labelled N).
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
