"""The CPU oracle (oracle/rqa_oracle.c) is pinned to the reference.

Every golden fixture was produced by tiledrqa itself
(tests/golden/make_golden.py); the oracle must reproduce each one exactly,
at several tile sizes and worker counts (tiling/worker invariance,
SPEC.md:239-240).
"""

import numpy as np
import pytest

from fixtures import assert_same, config_tags, load_cases, load_config, result_arrays, theiler_of

SMALL = load_cases("small_cases")
THEILER = load_cases("theiler_cases")


def test_small_case_count():
    assert len(SMALL) >= 200  # SPEC.md:465 acceptance criterion 1


@pytest.mark.parametrize("tile,workers", [(1, 1), (7, 2), (64, 8), (100000, 3)])
def test_oracle_small_cases(oracle_lib, tile, workers):
    for series, st, res, meta in SMALL:
        if tile == 1 and res["n_vectors"] > 120:
            continue
        got = oracle_lib.oracle_histograms(series, st["embedding_dimension"], st["time_delay"],
                                           st["metric"], st["radius"], theiler_of(st),
                                           tile_size=tile, workers=workers)
        assert_same(got, result_arrays(res), f"case {meta['id']} tile {tile}")


def test_oracle_theiler_cases(oracle_lib):
    for series, st, res, meta in THEILER:
        got = oracle_lib.oracle_histograms(series, st["embedding_dimension"], st["time_delay"],
                                           st["metric"], st["radius"], theiler_of(st),
                                           tile_size=37, workers=4)
        assert_same(got, result_arrays(res), f"theiler case {meta['id']}")


@pytest.mark.parametrize("tag", config_tags())
def test_oracle_config_fixtures(oracle_lib, tag):
    from paper_2402_16853_b200.workloads import WORKLOADS, series_sha256

    fx = load_config(tag)
    wl = WORKLOADS[fx["workload"]]
    series = wl.series(fx["samples"] if fx["prefix"] else None)
    assert series_sha256(series) == fx["sha256"]
    st = fx["settings"]
    got = oracle_lib.oracle_histograms(series, st["embedding_dimension"], st["time_delay"],
                                       st["metric"], st["radius"], theiler_of(st),
                                       tile_size=1024)
    assert_same(got, result_arrays(fx["result"]), tag)


def test_oracle_matrix_symmetric_and_brute_force(oracle_lib):
    """Bit level: R = R^T and agreement with scalar distances."""
    from paper_2402_16853_b200 import distance

    rng = np.random.default_rng(5)
    for metric in ("l1", "l2", "linf"):
        for m, tau in ((1, 1), (3, 2), (5, 1)):
            s = rng.uniform(-3, 3, 70)
            n = 70 - (m - 1) * tau
            vec = [s[i: i + (m - 1) * tau + 1: tau] for i in range(n)]
            r = float(np.median([distance(vec[0], v, metric) for v in vec]))
            mat = oracle_lib.oracle_matrix(s, m, tau, metric, r)
            assert np.array_equal(mat, mat.T)
            brute = np.array([[distance(vec[i], vec[j], metric) <= r for j in range(n)]
                              for i in range(n)])
            assert np.array_equal(mat, brute)


@pytest.mark.parametrize("metric", ["l1", "l2", "linf"])
def test_oracle_fp32_mode_matches_numpy_float32(metric, oracle_lib):
    """The fp32-mode restatement (recurrence_tile32) is numpy's float32
    evaluation of embedding.py:137-156: samples, ufuncs and radius in float32."""
    rng = np.random.default_rng(11)
    for m, tau, kind in ((1, 1, "u"), (3, 2, "u"), (4, 1, "o"), (2, 3, "o")):
        s = rng.uniform(0, 1, 300) if kind == "u" else 100 + rng.uniform(0, 1e-3, 300)
        r = 0.3 if kind == "u" else 3e-4
        n = len(s) - (m - 1) * tau
        s32 = s.astype(np.float32)
        acc = None
        for k in range(m):
            d = s32[k * tau:k * tau + n][:, None] - s32[k * tau:k * tau + n][None, :]
            t = d * d if (metric == "l2" and m > 1) else np.abs(d)
            acc = t if k == 0 else (np.maximum(acc, t) if metric == "linf" else acc + t)
        if metric == "l2" and m > 1:
            acc = np.sqrt(acc)
        want = acc <= np.float32(r)
        got = oracle_lib.oracle_matrix(s, m, tau, metric, r, 0, precision=32)
        assert np.array_equal(got, want), (metric, m, tau, kind)
        d, v, w, p, mism = oracle_lib.oracle_histograms_prec(s, m, tau, metric, r, 0,
                                                             precision=32, tile_size=64)
        m64 = oracle_lib.oracle_matrix(s, m, tau, metric, r, 0)
        assert p == int(want.sum()) and mism == int((m64 != want).sum())
