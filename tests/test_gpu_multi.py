"""Single-process multi-device path (rqa_run_multi, run_analysis(devices=...)).

On a one-GPU box the device list repeats device 0: every stripe still runs on
its own host thread, stream and workspace, and the stripes are gathered by
peer copies and stitched exactly as with distinct GPUs.  The results must be
identical to the single-device run and to the oracle for every list.
"""

import json
import subprocess
import sys

import numpy as np
import pytest

from fixtures import assert_same

pytestmark = pytest.mark.gpu


def _gpu_available():
    try:
        from paper_2402_16853_b200 import _native

        return _native.lib().rqa_device_count() > 0
    except Exception:
        return False


if not _gpu_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_16853_b200 import AnalysisSettings, embed, run_analysis  # noqa: E402


def _h(h):
    return h.diagonal, h.vertical, h.white_vertical, h.recurrence_points


CASES = [
    ("l2", 3, 1, 0.1, 0, 9000),
    ("linf", 2, 2, 0.15, 1, 7001),
    ("l1", 1, 1, 0.01, 0, 5003),
    ("l1", 6, 2, 0.6, 3, 4100),      # direct kernel
    ("l2", 10, 5, 1.3, 10, 6100),    # one-slot large-window kernel
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-m{c[1]}t{c[2]}" for c in CASES])
def test_device_lists_match_oracle(case, oracle_lib):
    metric, m, tau, r, w, length = case
    rng = np.random.default_rng(length)
    s = np.sin(np.linspace(0, 25 * np.pi, length)) + 0.3 * rng.uniform(-1, 1, length)
    st = AnalysisSettings(m, tau, metric, r, theiler_corrector=w)
    want = oracle_lib.oracle_histograms(s, m, tau, metric, r, w, tile_size=512)
    e = embed(s, m, tau)
    for devs in ([0], [0, 0], [0, 0, 0], [0] * 5, [0] * 8):
        h, t = run_analysis(e, st, devices=devs)
        assert_same(_h(h), want, f"{case} devices={devs}")
        assert t["devices"] == devs


def test_multi_device_fp32_mismatches(oracle_lib):
    rng = np.random.default_rng(3)
    s = 100.0 + rng.uniform(0, 1e-3, 6000)
    st = AnalysisSettings(2, 1, "l2", 2e-4)
    d, v, wh, p, mism = oracle_lib.oracle_histograms_prec(s, 2, 1, "l2", 2e-4, 0, precision=32,
                                                          tile_size=512)
    for devs in ([0], [0, 0, 0]):
        h, t = run_analysis(embed(s, 2, 1), st, devices=devs, precision="fp32")
        assert_same(_h(h), (d, v, wh, p), f"fp32 devices={devs}")
        assert t["mismatched_cells"] == mism


def test_cli_devices_and_precision(tmp_path):
    rng = np.random.default_rng(4)
    path = tmp_path / "x.csv"
    np.savetxt(path, rng.uniform(0, 1, 3000))
    outs = []
    for extra in ([], ["--devices", "0,0"], ["--precision", "fp32"]):
        out = subprocess.run([sys.executable, "-m", "paper_2402_16853_b200", "rqa", "--input",
                              str(path), "--embedding", "3", "--radius", "0.1", *extra],
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(json.loads(out.stdout))
    assert outs[0]["histograms"] == outs[1]["histograms"]
    assert outs[0]["recurrence_points"] == outs[1]["recurrence_points"]
    assert outs[1]["timing"]["devices"] == [0, 0]
    assert "mismatched_cells" in outs[2]["timing"]
