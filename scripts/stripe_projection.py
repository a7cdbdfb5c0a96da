"""Projected strong scaling of C3 over G GPUs, measured on ONE B200.

Every stripe of a G-way split (bench.py's equal-area row stripes) is run on
its own, timed with CUDA events, and the cross-stripe stitch is timed on the
gathered summaries.  The projection for G GPUs is the slowest stripe plus the
stitch plus the NCCL exchange at NVLink rate (summaries 16 B/column/rank
gathered to rank 0, 24 MiB histograms reduced); it ignores everything the one-GPU
measurement cannot see (NCCL latency, clock differences between GPUs).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_16853_b200.device import (MODE_FINAL, MODE_STRIPE, StripeOutputs,  # noqa: E402
                                          band_rows, run_rows_device, stitch_device)
from paper_2402_16853_b200.distributed import stripe_bounds  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
st = wl.settings
s_np = wl.series()
n = wl.n_vectors()
dev = torch.device("cuda", 0)
s = torch.from_numpy(s_np).to(dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=2):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) * 1e-3
        best = t if best is None else min(best, t)
    return best


h = torch.zeros(3, n + 1, dtype=torch.int64, device=dev)
p = torch.zeros(1, dtype=torch.int64, device=dev)
ref_h = torch.zeros_like(h)
ref_p = torch.zeros_like(p)
run_rows_device(s, st, 0, n, MODE_FINAL, ref_h, ref_p)
t1 = timed(lambda: run_rows_device(s, st, 0, n, MODE_FINAL, h.zero_(), p.zero_()))
out = {"workload": wl.name, "n": n, "one_gpu_s": t1, "nvlink_GBps": 900.0, "splits": {}}
band = band_rows(st, n)
for g in (2, 4, 8):
    bounds = stripe_bounds(n, g, band)
    gathered = StripeOutputs.empty(n, dev, rows=g)
    hh = torch.zeros_like(h)
    pp = torch.zeros_like(p)
    times = []
    for q in range(g):
        so = StripeOutputs(gathered.prefix[q], gathered.suffix[q], gathered.col[q],
                           gathered.rowlead)
        times.append(timed(lambda: run_rows_device(s, st, bounds[q], bounds[q + 1],
                                                   MODE_STRIPE, hh, pp, so), reps=1))
    t_stitch = timed(lambda: stitch_device(gathered, bounds, n, hh), reps=1)
    torch.cuda.synchronize()
    exact = bool(torch.equal(hh, ref_h) and torch.equal(pp, ref_p))
    xbytes = g * 16 * n + 3 * (n + 1) * 8            # all-gather + histogram reduce into rank 0
    t_x = xbytes / 900e9
    proj = max(times) + t_stitch + t_x
    out["splits"][g] = {"stripe_s": times, "max_stripe_s": max(times), "stitch_s": t_stitch,
                        "exchange_s_at_nvlink": t_x, "projected_s": proj,
                        "projected_speedup": t1 / proj, "stitched_result_exact": exact}
    print(g, json.dumps(out["splits"][g]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/stripe_projection.json", "w"), indent=1)
