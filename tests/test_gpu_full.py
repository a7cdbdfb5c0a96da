"""Bit-exact parity at the benchmark sizes (north_star: "full RQA of a
2^20-point embedded series ... with bit-exact histograms vs the CPU
reference").

The goldens tests/golden/full_<C>.json hold the sparse histograms of the full
configurations C3 (N = 2^20), P (999,999), C4 (500,000, Theiler 10) and C5
(N = 2^22), made by tests/golden/make_full_golden.py with the C oracle
(oracle/rqa_oracle.c, pinned bit-exact to tiledrqa by test_oracle_golden.py)
together with the SHA-256 of the input series.  The GPU run must reproduce
every bin and the point count exactly; C5 also exercises the single-device
path at the largest size and C3 the multi-stripe path (devices=[0, 0, 0]).
"""

import os

import numpy as np
import pytest

from fixtures import GOLDEN, assert_same, result_arrays

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _gpu_available():
    try:
        from paper_2402_16853_b200 import _native

        return _native.lib().rqa_device_count() > 0
    except Exception:
        return False


if not _gpu_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import json  # noqa: E402

from paper_2402_16853_b200 import compute_measures, embed, run_analysis  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS, series_sha256  # noqa: E402

FULL = sorted(f[len("full_"):-len(".json")] for f in os.listdir(GOLDEN)
              if f.startswith("full_") and f.endswith(".json"))
_SERIES = {}


def _load(tag):
    with open(os.path.join(GOLDEN, f"full_{tag}.json")) as fh:
        fx = json.load(fh)
    if tag not in _SERIES:
        _SERIES[tag] = WORKLOADS[fx["workload"]].series()
    s = _SERIES[tag]
    assert series_sha256(s) == fx["sha256"], "input series differs from the golden's"
    return fx, s


def test_full_goldens_present():
    assert {"C3", "C4", "P"} <= set(FULL), FULL


@pytest.mark.parametrize("tag", FULL)
def test_full_size_bit_exact(tag):
    fx, s = _load(tag)
    st = WORKLOADS[fx["workload"]].settings
    assert st.theiler_window == (fx["settings"].get("theiler_corrector")
                                 if fx["settings"].get("theiler_corrector") is not None
                                 else (0 if fx["settings"]["include_main_diagonal"] else 1))
    h, timing = run_analysis(embed(s, st.embedding_dimension, st.time_delay), st, device=0)
    got = (h.diagonal, h.vertical, h.white_vertical, h.recurrence_points)
    assert_same(got, result_arrays(fx["result"]), f"full {tag}")
    if "measures" in fx:  # tiledrqa.compute_measures on the golden histograms
        m = compute_measures(h, st).measures_dict()
        for k, v in fx["measures"].items():
            if v is None:
                assert m[k] is None, k
            else:
                assert m[k] == pytest.approx(v, rel=1e-12, abs=0), k


@pytest.mark.parametrize("tag", [t for t in FULL if t in ("C3", "P", "C5")])
def test_full_size_multi_stripe(tag):
    """Three stripes on one GPU (rqa_run_multi: device-side reduction + stitch)."""
    fx, s = _load(tag)
    st = WORKLOADS[fx["workload"]].settings
    h, timing = run_analysis(embed(s, st.embedding_dimension, st.time_delay), st,
                             devices=[0, 0, 0])
    got = (h.diagonal, h.vertical, h.white_vertical, h.recurrence_points)
    assert_same(got, result_arrays(fx["result"]), f"full {tag} x3")
    assert timing["bands"] == 3


_CHILD_LONG_UNITS = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_2402_16853_b200 import embed, run_analysis
from paper_2402_16853_b200.workloads import WORKLOADS
wl = WORKLOADS["C3"]
st = wl.settings
e = embed(wl.series(), st.embedding_dimension, st.time_delay)
out = []
for _ in range(3):
    h, t = run_analysis(e, st, device=0)
    out.append([int(h.recurrence_points), {str(k): int(v) for k, v in enumerate(h.diagonal) if v},
                {str(k): int(v) for k, v in enumerate(h.vertical) if v},
                {str(k): int(v) for k, v in enumerate(h.white_vertical) if v}])
print(json.dumps(out))
"""


def test_long_work_units_in_subprocess():
    """RQA_WAVES=1: one wave of units, each > 4096 iterations, so every unit
    empties its 32-bit shared bins into the 64-bit histogram mid-run (the
    path C5 takes by default; a missing barrier there lost a few diagonal
    runs nondeterministically).  Three runs of full C3 must equal the golden."""
    import subprocess
    import sys

    fx, _ = _load("C3")
    env = dict(os.environ, RQA_WAVES="1")
    out = subprocess.run([sys.executable, "-c", _CHILD_LONG_UNITS, REPO], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    want = fx["result"]
    for pts, d, v, w in json.loads(out.stdout.strip().splitlines()[-1]):
        assert pts == want["recurrence_points"]
        assert d == want["diagonal"] and v == want["vertical"] and w == want["white_vertical"]
