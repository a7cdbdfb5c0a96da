"""One analysis on cuda:0 (warm-up + profiled launch) for ncu captures.

usage: python scripts/profile_once.py [WORKLOAD] [REPEATS] [PREFIX_SAMPLES]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_16853_b200.device import MODE_FINAL, run_rows_device  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prefix = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = WORKLOADS[name]
series = wl.series(prefix)
s = torch.from_numpy(series).cuda()
n = series.shape[0] - (wl.settings.embedding_dimension - 1) * wl.settings.time_delay
h = torch.zeros(3, n + 1, dtype=torch.int64, device="cuda")
p = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(reps):
    run_rows_device(s, wl.settings, 0, n, MODE_FINAL, h, p)
torch.cuda.synchronize()
print("n", n, "points", int(p.item()) // reps)
