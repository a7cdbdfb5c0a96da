"""Precision paths of the CUDA engine (rqa_run_prec, SURVEY.md 8b `precision=`).

* fp32 mode: histograms bit-identical to the oracle's float32 restatement
  (numpy float32 semantics, oracle/rqa_oracle.c recurrence_tile32) and the
  mismatched-cell count identical to the oracle's cell-by-cell comparison of
  the float32 and float64 matrices.
* fp64 through the f32 filter (float32 evaluation inside a certified band,
  float64 re-evaluation of every word with a cell near the threshold): the
  histograms must be bit-identical to the float64 oracle, including inputs
  that make the band wide (forced with RQA_FILTER=2 in a subprocess).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from fixtures import assert_same

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpu_available():
    try:
        from paper_2402_16853_b200 import _native

        return _native.lib().rqa_device_count() > 0
    except Exception:
        return False


if not _gpu_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_16853_b200 import AnalysisSettings, embed, run_analysis  # noqa: E402


def _series(kind, length, rng):
    if kind == "uniform":
        return rng.uniform(0, 1, length)
    if kind == "offset":   # float32 rounding of the samples decides many cells
        return 100.0 + rng.uniform(0, 1e-3, length)
    if kind == "sine":
        return np.sin(np.linspace(0, 40 * np.pi, length)) + 0.05 * rng.normal(size=length)
    if kind == "nan":
        s = rng.uniform(0, 1, length)
        s[[3, length // 2, length // 2 + 1]] = np.nan
        return s
    if kind == "huge":     # beyond the certifiable band: every word re-evaluated
        return rng.uniform(0, 1, length) * 1e17
    raise ValueError(kind)


FP32_CASES = [
    # (kind, length, m, tau, metric, radius, theiler)
    ("uniform", 3000, 3, 1, "l2", 0.1, 0),        # packed f32x2 L2 reuse
    ("uniform", 2500, 3, 2, "l1", 0.3, 1),        # packed L1 reuse
    ("sine", 2200, 2, 1, "l2", 0.2, 0),
    ("sine", 3001, 10, 5, "l1", 2.0, 10),         # packed, one slot pair (large window)
    ("uniform", 2000, 1, 1, "l2", 0.01, 0),       # direct f32 (m = 1)
    ("uniform", 2100, 3, 1, "linf", 0.1, 0),      # direct f32 L-inf
    ("uniform", 1900, 6, 3, "l2", 0.6, 2),        # direct f32, runtime (m, tau)
    ("offset", 2600, 2, 1, "l2", 2e-4, 0),        # many fp32/fp64 mismatches
    ("offset", 2600, 3, 1, "l1", 4e-4, 0),
    ("offset", 2600, 3, 1, "linf", 2e-4, 1),
    ("nan", 1500, 3, 1, "l2", 0.2, 0),            # non-finite: all words re-evaluated
    ("huge", 1200, 2, 1, "l2", 2e16, 0),
]


@pytest.mark.parametrize("case", FP32_CASES,
                         ids=[f"{c[0]}-{c[1]}-m{c[2]}t{c[3]}-{c[4]}" for c in FP32_CASES])
def test_fp32_mode_matches_oracle(case, oracle_lib):
    kind, length, m, tau, metric, radius, w = case
    rng = np.random.default_rng(length + 7 * m)
    s = _series(kind, length, rng)
    st = AnalysisSettings(m, tau, metric, radius, theiler_corrector=w)
    h, timing = run_analysis(embed(s, m, tau), st, precision="fp32")
    d, v, wh, p, mism = oracle_lib.oracle_histograms_prec(s, m, tau, metric, radius, w,
                                                          precision=32, tile_size=256)
    assert_same((h.diagonal, h.vertical, h.white_vertical, h.recurrence_points),
                (d, v, wh, p), str(case))
    assert timing["evaluation"] == "fp32"
    assert timing["mismatched_cells"] == mism, (case, timing["mismatched_cells"], mism)
    if kind == "offset":
        assert mism > 0  # the case must exercise the mismatch count


def test_fp32_mode_known_answers():
    """Exact data (small integers): float32 and float64 agree everywhere."""
    s = np.arange(400, dtype=np.float64) % 17
    st = AnalysisSettings(2, 1, "l2", 3.0)
    h32, t32 = run_analysis(embed(s, 2, 1), st, precision="fp32")
    h64, _ = run_analysis(embed(s, 2, 1), st)
    assert t32["mismatched_cells"] == 0
    assert h32 == h64


def test_default_fp64_path_is_float64():
    rng = np.random.default_rng(5)
    s = rng.uniform(0, 1, 5000)
    _, timing = run_analysis(embed(s, 3, 1), AnalysisSettings(3, 1, "l2", 0.1))
    assert timing["evaluation"] in ("fp64", "f32-filter", "fp64-prefilter")
    if "RQA_FILTER" not in os.environ:
        assert timing["evaluation"] != "f32-filter"


_CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2402_16853_b200 import AnalysisSettings, embed, run_analysis
from oracle.oracle import oracle_histograms
out = []
rng = np.random.default_rng(17)
for kind, m, tau, metric, r in (("offset", 2, 1, "l2", 2e-4), ("offset", 3, 2, "l1", 5e-4),
                                ("uniform", 3, 1, "l2", 0.1), ("uniform", 4, 1, "l1", 0.4),
                                ("uniform", 10, 5, "l2", 1.2)):
    s = 100.0 + rng.uniform(0, 1e-3, 2400) if kind == "offset" else rng.uniform(0, 1, 2400)
    h, t = run_analysis(embed(s, m, tau), AnalysisSettings(m, tau, metric, r))
    d, v, w, p = oracle_histograms(s, m, tau, metric, r, 0, tile_size=512)
    ok = (h.recurrence_points == p and (h.diagonal == d).all() and (h.vertical == v).all()
          and (h.white_vertical == w).all())
    out.append([kind, m, tau, metric, bool(ok), t["evaluation"]])
print(json.dumps(out))
"""


@pytest.mark.parametrize("mode,expect", [("2", "f32-filter"), ("0", "fp64"), ("1", None)])
def test_filter_modes_in_subprocess(mode, expect):
    """RQA_FILTER=1 uses the filter for narrow bands, 2 for every certifiable
    band, 0 never; every path must reproduce the float64 oracle bit for bit."""
    env = dict(os.environ, RQA_FILTER=mode)
    out = subprocess.run([sys.executable, "-c", _CHILD, REPO], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    rows = json.loads(out.stdout.strip().splitlines()[-1])
    for kind, m, tau, metric, ok, ev in rows:
        assert ok, (kind, m, tau, metric, ev)
        want = expect or ("f32-filter" if kind == "uniform" else "fp64")
        if want == "fp64":
            assert ev in ("fp64", "fp64-prefilter"), (kind, m, tau, metric, ev)
        else:
            assert ev == want, (kind, m, tau, metric, ev)


_CHILD_PRE = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2402_16853_b200 import AnalysisSettings, embed, run_analysis
from oracle.oracle import oracle_histograms
out = []
rng = np.random.default_rng(23)
for kind, m, tau, metric, r, w in (("uniform", 3, 1, "l2", 0.1, 0), ("uniform", 2, 3, "l2", 0.05, 1),
                                   ("sine", 2, 1, "l2", 0.5, 0), ("uniform", 5, 1, "l2", 0.3, 2),
                                   ("uniform", 3, 1, "l1", 0.2, 0), ("sine", 2, 2, "l1", 1.0, 0),
                                   ("uniform", 4, 2, "l2", 0.25, 0), ("sine", 10, 5, "l1", 3.0, 10),
                                   ("sine", 5, 5, "l2", 0.8, 1),
                                   # long windows use the component-PAIR predicate: ties at
                                   # the radius on integer data, dense and sparse radii
                                   ("grid", 10, 5, "l1", 4.0, 0), ("grid", 5, 5, "l2", 3.0, 0),
                                   ("grid", 10, 5, "l2", 6.0, 3), ("sine", 5, 5, "l1", 2.5, 0),
                                   ("uniform", 10, 5, "l1", 1.5, 0)):
    n = 3100
    if kind == "uniform":
        s = rng.uniform(0, 1, n)
    elif kind == "grid":
        s = rng.integers(0, 3, n).astype(np.float64)
    else:
        s = np.sin(np.linspace(0, 60, n)) + 0.1 * rng.normal(size=n)
    s[100] = np.nan
    h, t = run_analysis(embed(s, m, tau), AnalysisSettings(m, tau, metric, r, theiler_corrector=w))
    d, v, wh, p = oracle_histograms(s, m, tau, metric, r, w, tile_size=512)
    ok = (h.recurrence_points == p and (h.diagonal == d).all() and (h.vertical == v).all()
          and (h.white_vertical == wh).all())
    out.append([kind, m, tau, metric, bool(ok), t["evaluation"]])
print(json.dumps(out))
"""


@pytest.mark.parametrize("mode,expect", [("1", "fp64-prefilter"), ("0", "fp64")])
def test_prefilter_modes_in_subprocess(mode, expect):
    """RQA_PREFILTER=1 forces the sparse prefilter (also on dense data), 0 disables
    it; both must reproduce the float64 oracle bit for bit (NaN included)."""
    env = dict(os.environ, RQA_PREFILTER=mode)
    out = subprocess.run([sys.executable, "-c", _CHILD_PRE, REPO], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    rows = json.loads(out.stdout.strip().splitlines()[-1])
    for kind, m, tau, metric, ok, ev in rows:
        assert ok, (kind, m, tau, metric, ev)
        assert ev == expect, (kind, m, tau, metric, ev)


def test_prefilter_chosen_for_sparse_c3_like(oracle_lib):
    rng = np.random.default_rng(8)
    s = rng.uniform(0, 1, 40000)   # >= 2^15 vectors: the prefilter is sampled
    st = AnalysisSettings(3, 1, "l2", 0.1)
    h, timing = run_analysis(embed(s, 3, 1), st)
    if "RQA_PREFILTER" not in os.environ:
        assert timing["evaluation"] == "fp64-prefilter"
    want = oracle_lib.oracle_histograms(s, 3, 1, "l2", 0.1, 0, tile_size=512)
    assert_same((h.diagonal, h.vertical, h.white_vertical, h.recurrence_points), want, "C3-like")


def test_fp32_stripes_then_stitch_equal_single_run():
    """fp32 mode through the device-resident stripe path (multi-GPU building
    blocks): histograms and the summed mismatch counts equal the single run."""
    import torch

    from paper_2402_16853_b200.device import (MODE_FINAL, MODE_STRIPE, StripeOutputs,
                                              band_rows, run_rows_device, stitch_device)
    from paper_2402_16853_b200.distributed import stripe_bounds

    rng = np.random.default_rng(31)
    s = 100.0 + rng.uniform(0, 1e-3, 7000)
    st = AnalysisSettings(2, 1, "l2", 2e-4)
    n = 7000 - 1
    dev = torch.device("cuda", 0)
    sd = torch.from_numpy(s).to(dev)
    ref_h = torch.zeros(3, n + 1, dtype=torch.int64, device=dev)
    ref_p = torch.zeros(1, dtype=torch.int64, device=dev)
    ref_m = torch.zeros(1, dtype=torch.int64, device=dev)
    run_rows_device(sd, st, 0, n, MODE_FINAL, ref_h, ref_p, precision="fp32", mismatches=ref_m)
    for g in (2, 3):
        bounds = stripe_bounds(n, g, band_rows(st, n))
        h = torch.zeros_like(ref_h)
        p = torch.zeros_like(ref_p)
        mm = torch.zeros_like(ref_m)
        gathered = StripeOutputs.empty(n, dev, rows=g)
        for q in range(g):
            so = StripeOutputs(gathered.prefix[q], gathered.suffix[q], gathered.col[q],
                               gathered.rowlead)
            run_rows_device(sd, st, bounds[q], bounds[q + 1], MODE_STRIPE, h, p, so,
                            precision="fp32", mismatches=mm)
        stitch_device(gathered, bounds, n, h)
        torch.cuda.synchronize()
        assert torch.equal(h, ref_h) and torch.equal(p, ref_p) and torch.equal(mm, ref_m), g
    assert int(ref_m.item()) > 0


ENTROPIES = ("L_entr", "V_entr", "W_entr")


@pytest.mark.parametrize("tag,length", [("C1", None), ("C2", None), ("C3", 65_538)])
def test_fp32_mode_measures_relative_error(tag, length):
    """north_star: fp32 mode reports its mismatched cells and its derived
    measures against fp64 (measures.py:90-139).  On C1, C2 and the C3 prefix
    every ratio measure (RR, DET, L, LAM, TT, W, DIV) is within 1e-6
    relative and the maxima are equal; the entropies move more (a mismatched
    cell shifts one count between two bins) and are within 1e-5.  Measured
    on every workload by scripts/fp32_report.py (profiles/r02_fp32_report.json)."""
    from paper_2402_16853_b200 import compare_precision
    from paper_2402_16853_b200.workloads import WORKLOADS

    wl = WORKLOADS[tag]
    rep = compare_precision(wl.series(length), wl.settings, device=0)
    assert rep["mismatched_cells"] >= 0
    for k, e in rep["rel_error"].items():
        bound = 1e-5 if k in ENTROPIES else 1e-6
        assert e <= bound, (tag, k, e, rep["mismatched_cells"])
    for k in ("L_max", "V_max", "W_max"):
        assert rep["measures_fp32"][k] == rep["measures_fp64"][k], k


_CHILD_FLUSH = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2402_16853_b200 import AnalysisSettings, embed, run_analysis
from oracle.oracle import oracle_histograms
out = []
rng = np.random.default_rng(5)
for kind, m, tau, metric, r, w in (("uniform", 3, 1, "l2", 0.15, 0), ("sine", 2, 2, "l2", 0.5, 1),
                                   ("sine", 10, 5, "l1", 3.0, 10), ("uniform", 3, 2, "linf", 0.1, 0)):
    n = 9000
    s = rng.uniform(0, 1, n) if kind == "uniform" else np.sin(np.linspace(0, 90, n)) + 0.1 * rng.normal(size=n)
    st = AnalysisSettings(m, tau, metric, r, theiler_corrector=w)
    for devices in ([0], [0, 0]):
        h, t = run_analysis(embed(s, m, tau), st, devices=devices)
        d, v, wh, p = oracle_histograms(s, m, tau, metric, r, w, tile_size=512)
        ok = (h.recurrence_points == p and (h.diagonal == d).all() and (h.vertical == v).all()
              and (h.white_vertical == wh).all())
        out.append([kind, m, metric, len(devices), bool(ok)])
print(json.dumps(out))
"""


def test_shared_bin_flush_every_two_iterations_in_subprocess():
    """RQA_FLUSH_EVERY=2: the band kernel empties its 32-bit shared bins into
    the 64-bit histogram every second iteration (by default every 4096, which
    only units of C5-size runs reach); every result must stay exact."""
    env = dict(os.environ, RQA_FLUSH_EVERY="2", RQA_PREFILTER="1")
    out = subprocess.run([sys.executable, "-c", _CHILD_FLUSH, REPO], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    for kind, m, metric, g, ok in json.loads(out.stdout.strip().splitlines()[-1]):
        assert ok, (kind, m, metric, g)
