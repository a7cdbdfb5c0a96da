"""Time the band+fold kernels for each benchmark configuration (one GPU)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_16853_b200.device import MODE_FINAL, run_rows_device  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS  # noqa: E402

out = {}
for name in (sys.argv[1:] or ["C1", "C2", "C3", "P", "C4", "C5"]):
    wl = WORKLOADS[name]
    series = wl.series()
    n = wl.n_vectors()
    s = torch.from_numpy(series).cuda()
    h = torch.zeros(3, n + 1, dtype=torch.int64, device="cuda")
    p = torch.zeros(1, dtype=torch.int64, device="cuda")
    run_rows_device(s, wl.settings, 0, n, MODE_FINAL, h, p)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(3):
        h.zero_(); p.zero_()
        ev[0].record()
        run_rows_device(s, wl.settings, 0, n, MODE_FINAL, h, p)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
    t = min(ts)
    out[name] = {"n": n, "seconds": t, "cells_per_s": n * n / t, "points": int(p.item())}
    print(name, json.dumps(out[name]), flush=True)
json.dump(out, open("gpurun_out/configs.json", "w"), indent=1)
