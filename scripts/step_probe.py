"""Step-time probe: device time of run_rows_device (C3, series resident) per
call, with and without bench.py's nvidia-smi clock sampler running."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_16853_b200.device import MODE_FINAL, run_rows_device  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
s = torch.from_numpy(wl.series()).cuda()
n = wl.n_vectors()
h = torch.zeros(3, n + 1, dtype=torch.int64, device="cuda")
p = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def run(k):
    out = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record(st)
        run_rows_device(s, wl.settings, 0, n, MODE_FINAL, h, p, stream=st)
        ev[1].record(st)
        torch.cuda.synchronize()
        out.append((ev[0].elapsed_time(ev[1]), (time.perf_counter() - t0) * 1e3))
    return out


run(2)
a = run(12)
with bench.ClockSampler(0):
    b = run(6)
c = run(6)
for name, r in (("plain", a), ("sampler", b), ("plain2", c)):
    d = [x[0] for x in r]
    w = [x[1] for x in r]
    print(f"{name:8s} device ms mean {np.mean(d):.2f} min {np.min(d):.2f} max {np.max(d):.2f}"
          f"  wall ms mean {np.mean(w):.2f}  all {[round(x, 1) for x in d]}")
