import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_16853_b200 import embed, run_analysis
from paper_2402_16853_b200.workloads import WORKLOADS
wl = WORKLOADS["C3"]
e = embed(wl.series(), 3, 1)
for i in range(4):
    t0 = time.perf_counter()
    h, t = run_analysis(e, wl.settings, device=0)
    w = time.perf_counter() - t0
    print(f"wall {w*1e3:.1f} ms  h2d {t['h2d']*1e3:.1f} kern {t['create_recurrence_matrix']*1e3:.1f} fold {t['fold']*1e3:.1f} d2h {t['d2h']*1e3:.1f} dev {t['device_total']*1e3:.1f} eval {t['evaluation']}", flush=True)
from paper_2402_16853_b200 import analyze, compute_measures
s = wl.series()
for i in range(3):
    t0 = time.perf_counter()
    e = embed(s, 3, 1)
    t1 = time.perf_counter()
    h, t = run_analysis(e, wl.settings, device=0)
    t2 = time.perf_counter()
    r = compute_measures(h, wl.settings)
    t3 = time.perf_counter()
    print(f"embed {1e3*(t1-t0):.2f} run_analysis {1e3*(t2-t1):.2f} (device_total {1e3*t['device_total']:.2f}) measures {1e3*(t3-t2):.2f} ms")
