"""Randomised parity sweep of the CUDA path against the C oracle (one B200).

Draws random (family, n, m, tau, metric, radius quantile, Theiler window,
precision, device list) cases, runs run_analysis and the oracle on the same
series, and requires bit-identical histograms and point counts (and, for
fp32 mode, the same mismatch count).  Usage: python scripts/fuzz_parity.py [CASES] [SEED] [MAX_LEN]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import oracle_histograms_prec  # noqa: E402
from paper_2402_16853_b200 import AnalysisSettings, distance, embed, run_analysis  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2026)
max_len = int(sys.argv[3]) if len(sys.argv) > 3 else 6000  # series length bound
fails, t0, stats = [], time.time(), {}
for i in range(cases):
    fam = rng.choice(["uniform", "sine", "ar1", "offset", "grid"])
    n_len = int(rng.integers(20, max_len))
    m = int(rng.choice([1, 2, 3, 4, 5, 6, 10]))
    tau = int(rng.choice([1, 2, 3, 5]))
    if n_len <= (m - 1) * tau + 1:
        n_len = (m - 1) * tau + 2 + int(rng.integers(0, 100))
    metric = str(rng.choice(["l1", "l2", "linf"]))
    if fam == "uniform":
        s = rng.uniform(0, 1, n_len)
    elif fam == "sine":
        s = np.sin(np.linspace(0, rng.uniform(5, 200), n_len)) + 0.1 * rng.normal(size=n_len)
    elif fam == "ar1":
        e = rng.normal(size=n_len)
        s = np.empty(n_len)
        s[0] = 0
        for k in range(1, n_len):
            s[k] = 0.95 * s[k - 1] + 0.3 * e[k]
    elif fam == "offset":
        s = 1e3 + rng.uniform(0, 1e-2, n_len)
    else:
        s = np.round(rng.uniform(0, 6, n_len)) * 0.5
    n = n_len - (m - 1) * tau
    idx = rng.integers(0, n, (300, 2))
    d = [distance(s[a:a + (m - 1) * tau + 1:tau], s[b:b + (m - 1) * tau + 1:tau], metric)
         for a, b in idx]
    q = float(rng.choice([0.0, 0.001, 0.01, 0.05, 0.2, 0.6, 1.0]))
    radius = float(np.quantile(d, q))
    w = int(rng.choice([0, 0, 1, 2, 7]))
    prec = "fp32" if rng.random() < 0.2 else "fp64"
    devs = [0] * int(rng.choice([1, 1, 1, 2, 3]))
    st = AnalysisSettings(m, tau, metric, radius, theiler_corrector=w)
    h, t = run_analysis(embed(s, m, tau), st, devices=devs, precision=prec)
    dd, vv, ww, pp, mm = oracle_histograms_prec(s, m, tau, metric, radius, w,
                                                precision=32 if prec == "fp32" else 64,
                                                tile_size=256)
    ok = (h.recurrence_points == pp and np.array_equal(h.diagonal, dd)
          and np.array_equal(h.vertical, vv) and np.array_equal(h.white_vertical, ww)
          and (prec == "fp64" or t["mismatched_cells"] == mm))
    key = f"{t['evaluation']}"
    stats[key] = stats.get(key, 0) + 1
    if not ok:
        fails.append(dict(i=i, fam=str(fam), n_len=n_len, m=m, tau=tau, metric=metric,
                          radius=radius, w=w, prec=prec, devices=devs))
        print("FAIL", fails[-1], flush=True)
out = {"cases": cases, "failures": fails, "paths": stats, "seconds": time.time() - t0}
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fuzz_parity.json", "w"), indent=1)
