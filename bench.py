"""Benchmark: full RQA of the N = 2^20 uniform series (config C3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C3] [--no-cpu-baseline]

One step = one complete analysis of the configured workload: the recurrence
test over all N^2 cells, diagonal / vertical / white-vertical line
extraction, cross-band (and, for N > 1 GPUs, cross-stripe) stitching and the
histogram reduction.  ``value`` is whole-job recurrence cells per second
with the series resident in HBM (CUDA events on the launching stream, max
over ranks); ``e2e`` is the same metric through the public API with the
host series copied in and the histograms copied out every step.
``--impl reference`` times the CPU restatement of the reference algorithm
(oracle/, all host threads) on a bounded prefix sample of the same workload.
Prints one JSON line on rank 0.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "recurrence cells/sec & full-RQA wall time, N=2^20, at 1/2/4/8 B200 vs CPU ref"
UNIT = "cells/s"


def ops_per_cell(settings) -> int:
    """Algorithmic FP64 ops per cell of the reference formulation."""
    m = settings.embedding_dimension
    if m == 1:
        return 2
    return 3 * m if settings.metric == "l2" else 2 * m


def executed_ops_per_cell(settings, evaluation="fp64", candidates=None) -> float:
    """FP64 ops per evaluated cell the chosen kernel issues.

    fp64: term reuse (App. A.3/A.4); fp64-prefilter: for m <= 4 the component
    predicate runs in packed float32 (no FP64), for m >= 5 the pair predicate
    issues 2 DADD + DADD + DSETP (+ 2 DMUL for L2) per cell; plus the full
    3m (L2) / 2m (L1) sum for the sampled candidate fraction (the component
    fraction, an upper bound for the pair predicate)."""
    m = settings.embedding_dimension
    if evaluation == "fp64-prefilter" and candidates is not None and candidates >= 0:
        per_cell = 0 if m <= 4 else (4 if settings.metric == "l1" else 6)
        return per_cell + candidates * ops_per_cell(settings)
    if m == 1 or settings.metric == "linf":
        return 2
    return m + 2 if settings.metric == "l2" else m + 1


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) == 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_model() -> str:
    """`lscpu` model name of the host (BASELINE.md's CPU-baseline record)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


CPU_PREFIX = 131_072  # vectors of the CPU sample, the same in both arms


def cpu_reference(settings, series_full, n_full, prefix=CPU_PREFIX, threads=None):
    """Time the oracle port (C restatement of tiledrqa's run_analysis, all
    host threads) on the first ``prefix`` vectors of the same series.

    Both bench arms (this line's cpu_baseline and ``--impl reference``) use
    this function with the same prefix, so their CPU numbers are comparable.
    """
    from oracle.oracle import oracle_histograms

    threads = threads or len(os.sched_getaffinity(0))
    m, tau = settings.embedding_dimension, settings.time_delay
    span = (m - 1) * tau
    n = min(prefix, n_full)
    s = series_full[: n + span]
    t0 = time.perf_counter()
    oracle_histograms(s, m, tau, settings.metric, settings.radius, settings.theiler_window,
                      tile_size=1024, workers=threads)
    dt = time.perf_counter() - t0
    return {"value": n * n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "threads": threads,
            "sample": f"prefix of {n} vectors ({n * n:.3e} cells) of the same series, "
                      f"{dt:.2f} s, oracle/rqa_oracle.c tiled port (tile 1024, "
                      f"{threads} threads)"}


def golden_parity(workload, hist_np, points):
    """Compare the final histograms with tests/golden/full_<workload>.json
    (made by tests/golden/make_full_golden.py from the pinned oracle)."""
    path = os.path.join(REPO, "tests", "golden", f"full_{workload}.json")
    if not os.path.exists(path):
        return "no golden"
    with open(path) as fh:
        fx = json.load(fh)
    res = fx["result"]
    n = res["n_vectors"]
    if hist_np.shape[1] != n + 1:
        return "mismatch (size)"
    if int(points) != int(res["recurrence_points"]):
        return "mismatch (points)"
    for row, key in enumerate(("diagonal", "vertical", "white_vertical")):
        want = np.zeros(n + 1, np.int64)
        for k, v in res[key].items():
            want[int(k)] = v
        if not np.array_equal(hist_np[row], want):
            return f"mismatch ({key})"
    return "exact"


def flush_l2(buf):
    buf.add_(1)  # 256 MiB write > 126 MB L2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-prefix", type=int, default=CPU_PREFIX)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    args = ap.parse_args()

    from paper_2402_16853_b200.workloads import WORKLOADS, series_sha256

    wl = WORKLOADS[args.workload]
    settings = wl.settings
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": f"{wl.name}: {wl.description}", "n_vectors": wl.n_vectors(),
              "m": settings.embedding_dimension, "tau": settings.time_delay,
              "metric": settings.metric, "radius": settings.radius,
              "theiler": settings.theiler_window, "parallelism": f"row stripes x{args.gpus}",
              "l2_between_steps": "flushed (256 MiB write) before every timed step"}

    if args.impl == "reference":
        if rank != 0:
            return
        series = wl.series()
        n_full = wl.n_vectors()
        per_step = []
        info = None
        for i in range(args.warmup + args.steps):
            info = cpu_reference(settings, series, n_full, prefix=args.cpu_prefix)
            if i >= args.warmup:
                per_step.append(info["value"])
        val = float(np.median(per_step))
        out = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference",
               "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": 1e3 * (wl.n_vectors() ** 2) / val, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded, sha256 " + series_sha256(series)[:16] + ")",
               "config": config,
               "cpu_baseline": {"value": val, "unit": UNIT, "cores": info["cores"],
                                "kind": "port", "sample": info["sample"],
                                "cpu_model": info["cpu_model"], "threads": info["threads"]},
               "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0},
               "note": "ms_per_step is the N^2-extrapolated wall of the full workload"}
        print(json.dumps(out))
        return

    import torch

    from paper_2402_16853_b200 import _native, embed, run_analysis
    from paper_2402_16853_b200.device import (MODE_FINAL, MODE_STRIPE, StripeOutputs, band_rows,
                                              run_rows_device, stitch_device)
    from paper_2402_16853_b200.distributed import all_reduce, exchange, reduce_sum, stripe_bounds

    # RQA_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 over gloo
    shared = os.environ.get("RQA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t_init0 = time.perf_counter()
    lib = _native.lib()
    lib.rqa_device_count()
    torch.zeros(1, device=dev)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t_init0  # driver context, library load (excluded from steps)
    series_np = wl.series()
    n = wl.n_vectors()
    series = torch.from_numpy(series_np).to(dev)
    hist = torch.zeros(3, n + 1, dtype=torch.int64, device=dev)
    points = torch.zeros(1, dtype=torch.int64, device=dev)
    prec = args.precision
    mism = torch.zeros(1, dtype=torch.int64, device=dev) if prec == "fp32" else None
    so = StripeOutputs.empty(n, dev) if world > 1 else None
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    bounds = stripe_bounds(n, world, band_rows(settings, n))
    lo, hi = bounds[rank], bounds[rank + 1]

    def step():
        hist.zero_()
        points.zero_()
        if mism is not None:
            mism.zero_()
        if world == 1:
            run_rows_device(series, settings, 0, n, MODE_FINAL, hist, points, stream=stream,
                            precision=prec, mismatches=mism)
        else:
            so.rowlead.zero_()
            run_rows_device(series, settings, lo, hi, MODE_STRIPE, hist, points, so,
                            stream=stream, precision=prec, mismatches=mism)
            gathered = exchange(so, world)
            reduce_sum(hist, 0)
            reduce_sum(points, 0)
            if rank == 0:
                stitch_device(gathered, bounds, n, hist)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # kernel-level timing of the dominant (band) kernel: one isolated launch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times = []
    launches0 = lib.rqa_launch_counter()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(flush)
            barrier()
            ev[0].record(stream)
            step()
            ev[1].record(stream)
            barrier()
            times.append(ev[0].elapsed_time(ev[1]) * 1e-3)
    launches = lib.rqa_launch_counter() - launches0
    # parity self-check of the last timed step (untimed): bit-exact against
    # the full-size golden of tests/golden (fp64) ...
    parity = None
    if rank == 0 and prec == "fp64":
        parity = golden_parity(args.workload, hist.cpu().numpy(), int(points.item()))
    t_step = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device=dev)
        all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    cells = float(n) * float(n)
    value = cells / t_step

    # band kernel alone (no fold) on this rank for the roofline
    hist.zero_()
    points.zero_()
    barrier()
    kern_times = []
    for _ in range(3):
        flush_l2(flush)
        torch.cuda.synchronize()
        ev[0].record(stream)
        if mism is not None:
            mism.zero_()
        run_rows_device(series, settings, lo, hi, MODE_FINAL if world == 1 else MODE_STRIPE,
                        hist, points, so, stream=stream, precision=prec, mismatches=mism)
        ev[1].record(stream)
        torch.cuda.synchronize()
        kern_times.append(ev[0].elapsed_time(ev[1]) * 1e-3)
    t_kern = float(np.min(kern_times))

    # e2e through the public API: host series in, histograms out, every step
    e2e_val = None
    e2e_timing = {}
    h2d = series_np.nbytes
    d2h = 3 * (n + 1) * 8 + 8
    full_rqa = None
    if world == 1:
        # full RQA through the public API every step: embed + H2D + kernels +
        # D2H + compute_measures (SURVEY 8d "full-RQA wall")
        from paper_2402_16853_b200 import analyze

        emb = embed(series_np, settings.embedding_dimension, settings.time_delay)
        dev_index = torch.cuda.current_device()
        _, e2e_timing = run_analysis(emb, settings, device=dev_index, precision=prec)
        e2e_t = []
        for _ in range(max(1, args.steps)):
            flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            analyze(series_np, settings, device=dev_index, precision=prec)
            e2e_t.append(time.perf_counter() - t0)
        e2e_val = cells / float(np.mean(e2e_t))
        # results come back as device-compacted nonzero bins (16 B each) plus
        # the counter and the point count (run_analysis, RQA_FLAG_OUT_ZEROED)
        res_h = analyze(series_np, settings, device=dev_index, precision=prec).histograms
        nnz = sum(int(np.count_nonzero(a)) for a in (res_h.diagonal, res_h.vertical,
                                                     res_h.white_vertical))
        d2h = 16 * nnz + 8 + 8
        full_rqa = {"median_s": float(np.median(e2e_t)), "min_s": float(np.min(e2e_t)),
                    "max_s": float(np.max(e2e_t)), "runs": len(e2e_t), "init_s": init_s,
                    "api": "paper_2402_16853_b200.analyze (embed -> run_analysis -> "
                           "compute_measures), host series in, RQAResult out"}
    else:
        from paper_2402_16853_b200.distributed import run_analysis_distributed

        emb = embed(series_np, settings.embedding_dimension, settings.time_delay)
        run_analysis_distributed(emb, settings, device=dev)
        barrier()
        t0 = time.perf_counter()
        run_analysis_distributed(emb, settings, device=dev)
        barrier()
        e2e_val = cells / (time.perf_counter() - t0)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    dadd = ctypes.c_double()
    dmul = ctypes.c_double()
    err = ctypes.create_string_buffer(256)
    lib.rqa_fp64_peak(local, ctypes.byref(dadd), ctypes.byref(dmul), err, 256)
    peak = min(dadd.value, dmul.value)
    # cells of the full matrix that this rank's stripe accounts for (upper
    # triangle rows [lo, hi) stand for their mirrored lower-triangle cells
    # too) and the cells its kernel actually evaluates (the upper triangle)
    local_cells = float(n - lo + n - hi) * float(hi - lo)
    evaluated_cells = float(n - lo + n - hi + 1) * float(hi - lo) / 2.0
    alg_ops = local_cells * ops_per_cell(settings)
    achieved = alg_ops / t_kern
    evaluation = e2e_timing.get("evaluation", "fp64") if world == 1 else "fp64"
    cand = e2e_timing.get("prefilter_candidates") if world == 1 else None
    # dram bytes per launch of the dominant kernel from the committed ncu capture
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(args.workload)
        if tr and world == 1:
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            traffic_src = "profiles/ncu_traffic.json (" + tr["kernel"] + ", ncu --set full)"
    except (OSError, ValueError, KeyError):
        tr = None
    # issue roofline of the dominant kernel: its ncu warp-instruction count over
    # the live kernel time vs 4 warp-instructions / clk / SM at the sampled clock
    issue = None
    sm_mhz = clocks.summary().get("sm_mhz")
    if tr and world == 1 and tr.get("warp_instructions") and sm_mhz:
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        ipeak = 4.0 * sms * sm_mhz * 1e6
        t_unit = t_kern * tr["gpu_time_ms"] / (tr["gpu_time_ms"] + sum(
            f["gpu_time_ms"] for f in tr.get("folds", {}).values()))
        ia = tr["warp_instructions"] / t_unit
        issue = {"unit": "warp-inst/s", "achieved": ia, "peak": ipeak, "frac": ia / ipeak,
                 "source": "warp instructions per launch from profiles/ncu_traffic.json, "
                           "kernel share of the timed band+fold span"}
    roofline = {
        "bound": "fp64", "unit": "FP64 op/s",
        "achieved": achieved, "peak": peak, "frac": achieved / peak if peak else None,
        "peak_source": "measured in-run: rqa_fp64_peak DADD/DMUL microbenchmark (not in "
                       "MEASURED_PEAKS.json, which has only HBM and bf16)",
        "traffic": traffic,
        "traffic_source": traffic_src,
        "kernel": "unit_kernel (fused test + runs + histograms) + folds, one launch triple",
        "kernel_s": t_kern,
        "algorithmic_ops_per_cell": ops_per_cell(settings),
        "evaluation": evaluation,
        "frac_full_matrix": achieved / peak if peak else None,
        "frac_per_evaluated_cell": evaluated_cells * ops_per_cell(settings) / t_kern / peak
        if peak else None,
        "evaluated_cells": evaluated_cells,
        "executed_fp64_ops_per_evaluated_cell": executed_ops_per_cell(settings, evaluation, cand),
        "executed_frac": evaluated_cells * executed_ops_per_cell(settings, evaluation, cand)
        / t_kern / peak if peak else None,
        "note": "frac = frac_full_matrix: SURVEY 8d algorithmic ops over all N^2 cells; "
                "the kernel evaluates only the upper triangle (R = R^T exactly), so "
                "frac_per_evaluated_cell is the same ops over the cells evaluated; "
                "executed_frac counts the FP64 ops the chosen kernel really issues",
    }
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, sha256 " + series_sha256(series_np)[:16] + ")",
           "config": config,
           "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h},
           "gpu_launches": int(launches),
           "roofline": roofline,
           "issue_roofline": issue,
           "clocks": clocks.summary(),
           "full_rqa_wall_s": cells / e2e_val if e2e_val else None,
           "full_rqa": full_rqa,
           "parity": parity,
           "precision": prec}
    if prec == "fp32" and world == 1:
        from paper_2402_16853_b200 import compare_precision

        rep = compare_precision(series_np, settings, device=dev_index)
        out["fp32_mode"] = {"mismatched_cells": rep["mismatched_cells"],
                            "mismatch_fraction": rep["mismatched_cells"] / rep["cells"],
                            "max_rel_error": rep["max_rel_error"],
                            "rel_error": rep["rel_error"],
                            "evaluation": rep["fp32_evaluation"]}
        out["dtype"] = "f32"
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_reference(settings, series_np, n, prefix=args.cpu_prefix)
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
