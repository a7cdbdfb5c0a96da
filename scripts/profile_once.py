"""One C3 analysis on cuda:0 (warm-up + profiled launch) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_16853_b200.workloads import WORKLOADS
from paper_2402_16853_b200.device import run_rows_device, MODE_FINAL
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
wl = WORKLOADS[name]
s = torch.from_numpy(wl.series()).cuda()
n = wl.n_vectors()
h = torch.zeros(3, n + 1, dtype=torch.int64, device="cuda")
p = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    run_rows_device(s, wl.settings, 0, n, MODE_FINAL, h, p)
torch.cuda.synchronize()
print("points", int(p.item()))
