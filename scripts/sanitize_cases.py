"""Small parity cases for compute-sanitizer runs (memcheck / racecheck /
synccheck / initcheck): every kernel family once (fp64 term reuse, L-inf AND,
prefilter with the packed float32 predicate, prefilter with the cell list,
f32 filter / fp32 mode, direct kernel, multi-stripe stitch, plot, tile scan),
each checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import oracle_histograms, oracle_histograms_prec  # noqa: E402
from paper_2402_16853_b200 import AnalysisSettings, embed, run_analysis  # noqa: E402

rng = np.random.default_rng(99)
n_len = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
cases = [("l2", 3, 1, 0.1, 0, "fp64"), ("linf", 3, 2, 0.05, 1, "fp64"), ("l1", 2, 2, 0.1, 0, "fp64"),
         ("l2", 10, 5, 0.9, 10, "fp64"), ("l1", 10, 5, 1.5, 10, "fp64"), ("l2", 7, 3, 0.5, 0, "fp64"),
         ("l2", 2, 1, 0.05, 0, "fp32"), ("linf", 2, 1, 0.05, 0, "fp32")]
bad = 0
for metric, m, tau, r, w, prec in cases:
    s = rng.uniform(0, 1, n_len)
    st = AnalysisSettings(m, tau, metric, r, theiler_corrector=w)
    for devices in ([0], [0, 0]):
        h, t = run_analysis(embed(s, m, tau), st, devices=devices, precision=prec)
        d, v, wh, p, mm = oracle_histograms_prec(s, m, tau, metric, r, w,
                                                 precision=64 if prec == "fp64" else 32,
                                                 tile_size=256)
        ok = (h.recurrence_points == p and (h.diagonal == d).all() and (h.vertical == v).all()
              and (h.white_vertical == wh).all())
        if prec == "fp32":
            ok = ok and t["mismatched_cells"] == mm
        bad += not ok
        print(metric, m, tau, w, prec, devices, t["evaluation"], "ok" if ok else "MISMATCH", flush=True)
from paper_2402_16853_b200 import compute_plot  # noqa: E402

s = rng.uniform(0, 1, 300)
compute_plot(embed(s, 2, 1), AnalysisSettings(2, 1, "l2", 0.1), 2)
print("plot ok")
print("FAILURES", bad)
sys.exit(1 if bad else 0)
