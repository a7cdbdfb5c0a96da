"""In-process multi-stripe path on one GPU: run_analysis(devices=[0]*G) vs device=0 (C3)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_16853_b200 import embed, run_analysis  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
e = embed(wl.series(), wl.settings.embedding_dimension, wl.settings.time_delay)
ref, _ = run_analysis(e, wl.settings, device=0)
for G in (1, 2, 4, 8):
    devs = [0] * G
    run_analysis(e, wl.settings, devices=devs)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        h, t = run_analysis(e, wl.settings, devices=devs)
        ts.append(time.perf_counter() - t0)
    same = h == ref
    print(f"G={G} wall {min(ts)*1e3:.1f} ms  kernels(max stripe) {t['create_recurrence_matrix']*1e3:.1f} "
          f"stitch {t['fold']*1e3:.1f} exact={same}", flush=True)
