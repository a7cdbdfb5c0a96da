"""GPU recurrence_block / recurrence plots vs the oracle matrix (bit-exact)."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpu_available():
    try:
        from paper_2402_16853_b200 import _native

        return _native.lib().rqa_device_count() > 0
    except Exception:
        return False


if not _gpu_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_16853_b200 import (AnalysisSettings, compute_plot, embed,  # noqa: E402
                                   read_pbm, recurrence_block, render)


@pytest.mark.parametrize("metric,m,tau,w", [("l2", 3, 1, 0), ("l1", 2, 3, 1), ("linf", 4, 2, 3),
                                            ("l2", 1, 1, 0), ("l1", 10, 5, 0)])
def test_recurrence_block_matches_oracle(oracle_lib, metric, m, tau, w):
    rng = np.random.default_rng(m * 7 + tau)
    s = np.sin(np.linspace(0, 20, 300)) + 0.3 * rng.normal(size=300)
    r = {"l1": 1.0, "l2": 0.6, "linf": 0.4}[metric]
    mat = oracle_lib.oracle_matrix(s, m, tau, metric, r, w)
    n = mat.shape[0]
    st = AnalysisSettings(m, tau, metric, r, theiler_corrector=w)
    e = embed(s, m, tau)
    assert np.array_equal(recurrence_block(e, st, 0, n, 0, n), mat)
    for r0, r1, c0, c1 in ((3, 77, 40, 201), (0, 1, 0, n), (n - 5, n, 0, 9), (10, 10, 0, 5)):
        assert np.array_equal(recurrence_block(e, st, r0, r1, c0, c1), mat[r0:r1, c0:c1])


def _or_reduce(mat, b):
    n = mat.shape[0]
    size = -(-n // b)
    pad = np.zeros((size * b, size * b), bool)
    pad[:n, :n] = mat
    return pad.reshape(size, b, size, b).any(axis=(1, 3))


@pytest.mark.parametrize("b", [1, 2, 3, 4, 16])
def test_plot_or_reduction(oracle_lib, tmp_path, b):
    rng = np.random.default_rng(b)
    s = rng.uniform(0, 1, 250)
    mat = oracle_lib.oracle_matrix(s, 2, 1, "l2", 0.1, 0)
    st = AnalysisSettings(2, 1, "euclidean", 0.1)
    plot = render(embed(s, 2, 1), st, reduction_factor=b, out=tmp_path / "p.pbm")
    want = _or_reduce(mat, b)
    assert np.array_equal(plot.matrix(), want)
    assert np.array_equal(read_pbm(tmp_path / "p.pbm")[::-1], want)   # bottom-left origin


def test_plot_spec_examples():
    """identity-only 3x3 and all-ones 8x8 at b=4."""
    p = compute_plot(embed(np.array([0.0, 10.0, 20.0]), 1, 1), AnalysisSettings(1, 1, "l2", 0.5))
    assert np.array_equal(p.matrix(), np.eye(3, dtype=bool))
    p = compute_plot(embed(np.zeros(8), 1, 1), AnalysisSettings(1, 1, "l2", 0.0), 4)
    assert p.size == 2 and p.matrix().all()


def test_cli_rqa_json(tmp_path):
    from paper_2402_16853_b200.cli import main

    out = tmp_path / "r.json"
    assert main(["rqa", "--synthetic-sine", "2001", "--x-end-pi-multiples", "2",
                 "--embedding", "2", "--delay", "2", "--radius", "1.0", "--output", str(out)]) == 0
    d = json.loads(out.read_text())
    assert set(d) == {"settings", "n_vectors", "recurrence_points", "measures", "histograms",
                      "timing"}
    assert d["n_vectors"] == 1999 and 0 < d["measures"]["RR"] <= 1
    assert main(["plot", "--synthetic-sine", "300", "--radius", "0.1",
                 "--output", str(tmp_path / "p.pbm")]) == 0
