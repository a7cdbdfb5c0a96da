"""Host-side API (no GPU): settings, measures, PBM I/O, CLI parsing, ingest."""

import math

import numpy as np
import pytest

from paper_2402_16853_b200 import (AnalysisSettings, InvalidArgument, LineHistograms, PlotTooLarge,
                                   RecurrencePlot, compute_measures, embed, generate_sine, merge,
                                   normalize_metric, read_column, read_pbm, write_pbm)
from paper_2402_16853_b200.cli import build_parser, main, settings_from


def test_metric_aliases_and_validation():
    assert normalize_metric("Manhattan") == "l1" and normalize_metric("chebyshev") == "linf"
    with pytest.raises(InvalidArgument):
        normalize_metric("cosine")
    for bad in (dict(embedding_dimension=0), dict(time_delay=0), dict(radius=-1.0),
                dict(radius=float("nan")), dict(min_diagonal_line_length=0),
                dict(theiler_corrector=-1)):
        with pytest.raises(InvalidArgument):
            AnalysisSettings(**bad)


def test_theiler_extension_semantics():
    s = AnalysisSettings(radius=1.0)
    assert s.theiler_window == 0 and "theiler_corrector" not in s.to_dict()
    s = AnalysisSettings(radius=1.0, include_main_diagonal=False)
    assert s.theiler_window == 1 and s.excluded_cells(10) == 10
    s = AnalysisSettings(radius=1.0, theiler_corrector=3)
    assert not s.include_main_diagonal and s.excluded_cells(10) == 10 + 2 * (9 + 8)
    assert s.to_dict()["theiler_corrector"] == 3


def test_measures_known_answer_all_ones_7x7():
    """all-ones 7x7 -> DET 47/49, L_max 7, DIV 1/7, LAM 1, TT 7."""
    n = 7
    h = LineHistograms(n, recurrence_points=n * n)
    h.diagonal[1:n] = 2
    h.diagonal[n] = 1
    h.vertical[n] = n
    r = compute_measures(h, AnalysisSettings(radius=0.0))
    assert r.rr == 1.0 and r.det == pytest.approx(47 / 49) and r.l_max == 7
    assert r.div == pytest.approx(1 / 7) and r.lam == 1.0 and r.tt == 7.0
    assert r.w_mean is None and r.w_max is None and r.w_entr is None


def test_measures_empty_and_point_mass():
    h = LineHistograms(5)
    r = compute_measures(h, AnalysisSettings(radius=0.0))
    assert r.det is None and r.l_mean is None and r.l_max is None and r.div is None
    h.diagonal[5] = 3
    assert compute_measures(h, AnalysisSettings(radius=0.0)).l_entr == 0.0


def test_merge_commutes():
    a = LineHistograms(4, 3)
    a.vertical[2] = 1
    b = LineHistograms(4, 5)
    b.white_vertical[4] = 2
    assert merge(a, b) == merge(b, a)


def test_pbm_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    mat = rng.uniform(size=(13, 13)) < 0.3
    plot = RecurrencePlot(13, 1, 13, np.packbits(mat, axis=1))
    path = tmp_path / "p.pbm"
    write_pbm(plot, path)
    img = read_pbm(path)
    assert np.array_equal(img[::-1], mat)      # row 0 is the bottom image row
    assert plot.matrix().tolist() == mat.tolist()


def test_cli_argument_errors_exit_2():
    assert main(["rqa", "--synthetic-sine", "100"]) == 2       # --radius required
    assert main(["plot", "--radius", "1"]) == 2                 # no input source


def test_cli_settings_mapping():
    args = build_parser().parse_args(["rqa", "--synthetic-sine", "10", "--radius", "0.5",
                                      "--embedding", "2", "--delay", "3", "--metric", "maximum",
                                      "--main-diagonal", "exclude"])
    st = settings_from(args)
    assert (st.embedding_dimension, st.time_delay, st.metric, st.theiler_window) == (2, 3, "linf", 1)


def test_ingest_spec_examples(tmp_path):
    p = tmp_path / "a.csv"
    p.write_text("a,1\nb,2\nc,3")
    assert read_column(p, ",", 1, 1).values.tolist() == [2.0, 3.0]
    s = generate_sine(3, math.pi)
    assert s.values[0] == 0.0 and s.values[1] == 1.0 and abs(s.values[2]) < 1e-12
    assert embed(np.arange(10.0), 2, 3).n_vectors == 7


def test_measures_from_golden_histograms_are_bit_identical():
    """compute_measures (sparse formulation) on the reference's own histograms
    reproduces the reference's measures exactly (measures.py:73-139)."""
    from fixtures import load_cases, result_arrays, settings_obj

    from paper_2402_16853_b200 import LineHistograms, compute_measures

    for series, st, res, meta in load_cases("small_cases"):
        s = settings_obj(st)
        d, v, w, p = result_arrays(res)
        n = d.shape[0] - 1
        got = compute_measures(LineHistograms(n, p, d, v, w), s).measures_dict()
        for k, want in meta["measures"].items():
            assert got[k] == want, (meta["id"], k, got[k], want)
