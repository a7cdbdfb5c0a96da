"""Parity of the CUDA path with the reference (through the C-ABI).

Golden fixtures come from tiledrqa itself; larger random cases are checked
against the C oracle (pinned to the reference by test_oracle_golden.py); at
full benchmark size the checks are size-independent identities.  Integer
results must be bit-identical.
"""

import numpy as np
import pytest

from fixtures import (assert_same, config_tags, load_cases, load_config, result_arrays,
                      settings_obj, theiler_of)

pytestmark = pytest.mark.gpu


def _gpu_available():
    try:
        from paper_2402_16853_b200 import _native

        return _native.lib().rqa_device_count() > 0
    except Exception:
        return False


if not _gpu_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_16853_b200 import (AnalysisSettings, compute_measures, embed,  # noqa: E402
                                   run_analysis)


def gpu_hist(series, settings):
    e = embed(series, settings.embedding_dimension, settings.time_delay)
    h, _ = run_analysis(e, settings)
    return h.diagonal, h.vertical, h.white_vertical, h.recurrence_points


def test_small_golden_cases():
    fails = []
    for series, st, res, meta in load_cases("small_cases"):
        try:
            assert_same(gpu_hist(series, settings_obj(st)), result_arrays(res), f"case {meta['id']}")
        except AssertionError as exc:
            fails.append(str(exc))
    assert not fails, f"{len(fails)} failures: {fails[:5]}"


def test_small_golden_measures():
    for series, st, res, meta in load_cases("small_cases")[:60]:
        s = settings_obj(st)
        e = embed(series, s.embedding_dimension, s.time_delay)
        h, _ = run_analysis(e, s)
        got = compute_measures(h, s).measures_dict()
        for k, v in meta["measures"].items():
            if v is None:
                assert got[k] is None, (meta["id"], k)
            else:
                assert got[k] == pytest.approx(v, rel=1e-12, abs=0), (meta["id"], k)


def test_theiler_golden_cases():
    for series, st, res, meta in load_cases("theiler_cases"):
        assert_same(gpu_hist(series, settings_obj(st)), result_arrays(res),
                    f"theiler case {meta['id']}")


@pytest.mark.parametrize("tag", config_tags())
def test_config_fixtures(tag):
    from paper_2402_16853_b200.workloads import WORKLOADS, series_sha256

    fx = load_config(tag)
    wl = WORKLOADS[fx["workload"]]
    series = wl.series(fx["samples"] if fx["prefix"] else None)
    assert series_sha256(series) == fx["sha256"]
    assert_same(gpu_hist(series, settings_obj(fx["settings"])), result_arrays(fx["result"]), tag)


CASES = [
    # (family, length, m, tau, metric, quantile, theiler)
    ("uniform", 3000, 3, 1, "l2", 0.01, 0),
    ("uniform", 4097, 3, 2, "linf", 0.02, 0),
    ("sine", 5000, 2, 2, "l2", 0.4, 0),
    ("sine", 2500, 1, 1, "l1", 0.05, 1),
    ("ar1", 3333, 4, 1, "l1", 0.1, 1),
    ("ar1", 2049, 5, 1, "linf", 0.3, 3),
    ("uniform", 2111, 6, 3, "l2", 0.2, 0),      # direct (runtime m, tau) kernel
    ("sine", 3001, 10, 5, "l1", 0.3, 10),       # C4 shape, direct kernel
    ("uniform", 1800, 7, 1, "linf", 0.5, 2),    # direct Linf
    ("sine", 6000, 2, 3, "l1", 0.9, 0),         # dense
    ("uniform", 40, 3, 1, "l2", 1.0, 0),        # all ones
    ("uniform", 33, 1, 1, "l2", 0.0, 0),        # only the main diagonal
]


def _series(family, length, rng):
    if family == "uniform":
        return rng.uniform(0, 1, length)
    if family == "sine":
        return np.sin(np.linspace(0, 40 * np.pi, length)) + 0.05 * rng.normal(size=length)
    x = np.empty(length)
    x[0] = 0.0
    eps = rng.normal(size=length)
    for i in range(1, length):
        x[i] = 0.9 * x[i - 1] + 0.3 * eps[i]
    return x


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-m{c[2]}t{c[3]}-{c[4]}" for c in CASES])
def test_random_cases_vs_oracle(case, oracle_lib):
    fam, length, m, tau, metric, q, w = case
    rng = np.random.default_rng(length * 31 + m)
    s = _series(fam, length, rng)
    n = length - (m - 1) * tau
    # radius from the quantile of sampled distances
    from paper_2402_16853_b200 import distance

    idx = rng.integers(0, n, (400, 2))
    d = [distance(s[i: i + (m - 1) * tau + 1: tau], s[j: j + (m - 1) * tau + 1: tau], metric)
         for i, j in idx]
    radius = float(np.quantile(d, q)) if q > 0 else 0.0
    st = AnalysisSettings(m, tau, metric, radius, theiler_corrector=w)
    want = oracle_lib.oracle_histograms(s, m, tau, metric, radius, w, tile_size=512)
    assert_same(gpu_hist(s, st), want, str(case))


def test_nan_in_raw_array_matches_reference_semantics(oracle_lib):
    """A raw ndarray is not finite-checked (embedding.py:59-60): NaN cells are 0."""
    rng = np.random.default_rng(9)
    s = rng.uniform(0, 1, 700)
    s[[5, 300, 301, 650]] = np.nan
    for metric in ("l1", "l2", "linf"):
        for m, tau in ((1, 1), (3, 1), (2, 2), (6, 2)):
            want = oracle_lib.oracle_histograms(s, m, tau, metric, 0.2, 0, tile_size=64)
            assert_same(gpu_hist(s, AnalysisSettings(m, tau, metric, 0.2)), want,
                        f"nan {metric} m{m} t{tau}")


def test_spec_known_answers():
    """SPEC.md examples: all-ones and identity-only matrices."""
    for n in (3, 4, 7, 50, 1000):
        s = np.zeros(n)
        d, v, w, p = gpu_hist(s, AnalysisSettings(1, 1, "l2", 0.0))
        assert p == n * n
        want_d = np.zeros(n + 1, np.int64)
        want_d[1:n] = 2
        want_d[n] = 1
        assert np.array_equal(d, want_d)
        assert v[n] == n and v.sum() == n
        assert w.sum() == 0
    h = gpu_hist(np.arange(5.0), AnalysisSettings(1, 1, "l2", 0.5, include_main_diagonal=False))
    assert h[3] == 0 and h[2][5] == 5 and h[2].sum() == 5
    res = compute_measures(
        run_analysis(embed(np.zeros(7), 1, 1), AnalysisSettings(1, 1, "l2", 0.0))[0],
        AnalysisSettings(1, 1, "l2", 0.0))
    assert res.det == pytest.approx(47 / 49) and res.l_max == 7 and res.lam == 1.0
    assert res.tt == 7.0 and res.div == pytest.approx(1 / 7)


def test_stripes_then_stitch_equal_single_run():
    """Multi-GPU decomposition, emulated on one device: G stripes + stitch."""
    import torch

    from paper_2402_16853_b200.device import (MODE_FINAL, MODE_STRIPE, StripeOutputs, band_rows,
                                              run_rows_device, stitch_device)
    from paper_2402_16853_b200.distributed import stripe_bounds

    rng = np.random.default_rng(11)
    for metric, m, tau, r, length in (("l2", 3, 1, 0.12, 9000), ("linf", 2, 2, 0.3, 7001),
                                      ("l1", 1, 1, 0.02, 5000), ("l1", 6, 2, 0.5, 4100)):
        s = np.sin(np.linspace(0, 30 * np.pi, length)) + 0.2 * rng.uniform(-1, 1, length)
        st = AnalysisSettings(m, tau, metric, r)
        n = length - (m - 1) * tau
        dev = torch.device("cuda", 0)
        sd = torch.from_numpy(s).to(dev)
        ref_h = torch.zeros(3, n + 1, dtype=torch.int64, device=dev)
        ref_p = torch.zeros(1, dtype=torch.int64, device=dev)
        run_rows_device(sd, st, 0, n, MODE_FINAL, ref_h, ref_p)
        band = band_rows(st, n)
        for g in (1, 2, 3, 5):
            bounds = stripe_bounds(n, g, band)
            h = torch.zeros(3, n + 1, dtype=torch.int64, device=dev)
            p = torch.zeros(1, dtype=torch.int64, device=dev)
            gathered = StripeOutputs.empty(n, dev, rows=g)
            for q in range(g):
                so = StripeOutputs(gathered.prefix[q], gathered.suffix[q], gathered.col[q],
                                   gathered.rowlead)
                run_rows_device(sd, st, bounds[q], bounds[q + 1], MODE_STRIPE, h, p, so)
            stitch_device(gathered, bounds, n, h)
            torch.cuda.synchronize()
            assert torch.equal(h, ref_h), (metric, g)
            assert torch.equal(p, ref_p)


def test_full_size_identities():
    """C3 at full size (N = 2^20): conservation identities.
    Bit-exact parity at this size is tests/test_gpu_full.py (full goldens)."""
    from paper_2402_16853_b200.workloads import WORKLOADS

    wl = WORKLOADS["C3"]
    s = wl.series()
    d, v, w, p = gpu_hist(s, wl.settings)
    n = wl.n_vectors()
    lengths = np.arange(n + 1, dtype=np.int64)
    assert int((lengths * d).sum()) == p
    assert int((lengths * v).sum()) == p
    assert int((lengths * v).sum() + (lengths * w).sum()) == n * n


@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 255, 257, 1023, 1025])
def test_tiny_and_boundary_sizes(n, oracle_lib):
    """n around warp / slot / band boundaries, every metric, both kernel families."""
    rng = np.random.default_rng(n)
    for metric, m, tau, r in (("l2", 3, 1, 0.3), ("l1", 2, 2, 0.2), ("linf", 1, 1, 0.1),
                              ("l2", 6, 2, 0.6)):
        s = rng.uniform(0, 1, n + (m - 1) * tau)
        for w in (0, 1, 3):
            st = AnalysisSettings(m, tau, metric, r, theiler_corrector=w)
            want = oracle_lib.oracle_histograms(s, m, tau, metric, r, w, tile_size=64)
            assert_same(gpu_hist(s, st), want, f"n={n} {metric} m{m} t{tau} w{w}")


def test_largest_embedding_window(oracle_lib):
    """(m - 1) * tau = 4096 (the direct kernel's largest window)."""
    rng = np.random.default_rng(4)
    for m, tau in ((2, 4096), (4097, 1)):
        s = rng.uniform(0, 1, 4096 + 300)
        r = 0.5 if m == 2 else 30.0
        st = AnalysisSettings(m, tau, "l1", r)
        want = oracle_lib.oracle_histograms(s, m, tau, "l1", r, 0, tile_size=128)
        assert_same(gpu_hist(s, st), want, f"m{m} t{tau}")


def test_c_abi_dense_and_sparse_outputs_agree(oracle_lib):
    """rqa_run (dense copy-back, the reference binding of INTEGRATION.md) and
    rqa_run_prec with RQA_FLAG_OUT_ZEROED (device-compacted bins) agree with
    the oracle; garbage in the output arrays is overwritten by rqa_run."""
    import ctypes

    from paper_2402_16853_b200 import _native

    rng = np.random.default_rng(12)
    s = rng.uniform(0, 1, 3000)
    n = 3000 - 2
    want = oracle_lib.oracle_histograms(s, 3, 1, "l2", 0.15, 1, tile_size=256)
    p64 = ctypes.POINTER(ctypes.c_int64)
    pd = ctypes.POINTER(ctypes.c_double)
    d, v, w = (np.full(n + 1, 77, np.int64) for _ in range(3))
    pts = np.zeros(1, np.int64)
    tim = np.zeros(_native.TIMING_SLOTS)
    _native.call("rqa_run", s.ctypes.data_as(pd), s.shape[0], 3, 1, 1, 0.15, 1, 0,
                 d.ctypes.data_as(p64), v.ctypes.data_as(p64), w.ctypes.data_as(p64),
                 pts.ctypes.data_as(p64), tim.ctypes.data_as(pd))
    assert_same((d, v, w, int(pts[0])), want, "rqa_run dense")
    d2, v2, w2 = (np.zeros(n + 1, np.int64) for _ in range(3))
    pts2 = np.zeros(1, np.int64)
    mism = np.zeros(1, np.int64)
    _native.call("rqa_run_prec", s.ctypes.data_as(pd), s.shape[0], 3, 1, 1, 0.15, 1, 64, 0, 1,
                 d2.ctypes.data_as(p64), v2.ctypes.data_as(p64), w2.ctypes.data_as(p64),
                 pts2.ctypes.data_as(p64), mism.ctypes.data_as(p64), tim.ctypes.data_as(pd))
    assert_same((d2, v2, w2, int(pts2[0])), want, "rqa_run_prec sparse")


ADVERSARIAL = [
    # (name, series builder, m, tau, metric, radius)
    ("grid-ties-l2", lambda r: np.round(r.uniform(0, 8, 1500)) * 0.25, 2, 1, "l2", 0.25 * 2 ** 0.5),
    ("grid-ties-l1", lambda r: np.round(r.uniform(0, 8, 1500)) * 0.5, 3, 1, "l1", 1.0),
    ("grid-ties-linf", lambda r: np.round(r.uniform(0, 8, 1500)) * 0.5, 3, 2, "linf", 0.5),
    ("radius-zero", lambda r: np.round(r.uniform(0, 3, 1200)), 2, 1, "l2", 0.0),
    ("denormals", lambda r: r.uniform(0, 1, 1300) * 5e-324 * 1000, 3, 1, "l2", 5e-322),
    ("tiny-radius-l2", lambda r: r.uniform(0, 1, 1300) * 1e-160, 3, 1, "l2", 1e-161),
    ("huge-overflow", lambda r: r.uniform(-1, 1, 1300) * 1e300, 3, 1, "l2", 1e300),
    ("huge-radius", lambda r: r.uniform(-1, 1, 1300) * 1e300, 2, 1, "l2", 1.7e308),
    ("inf-radius", lambda r: r.uniform(-1, 1, 900), 3, 1, "l1", float("inf")),
    ("signed-zeros", lambda r: np.where(r.random(1000) < 0.5, -0.0, 0.0), 3, 1, "linf", 0.0),
    ("constant", lambda r: np.full(1100, 3.25), 4, 2, "l2", 0.0),
    ("nan-and-inf", lambda r: np.where(r.random(1200) < 0.02, np.inf,
                                       np.where(r.random(1200) < 0.02, np.nan,
                                                r.uniform(0, 1, 1200))), 3, 1, "l2", 0.3),
]


@pytest.mark.parametrize("case", ADVERSARIAL, ids=[c[0] for c in ADVERSARIAL])
def test_adversarial_inputs_vs_oracle(case, oracle_lib):
    """Ties exactly at the radius, denormals, overflowing squares, radius 0 /
    huge / inf, signed zeros, non-finite samples: bit-exact on every path."""
    name, build, m, tau, metric, radius = case
    s = build(np.random.default_rng(len(name)))
    for w in (0, 1):
        st = AnalysisSettings(m, tau, metric, radius, theiler_corrector=w)
        want = oracle_lib.oracle_histograms(s, m, tau, metric, radius, w, tile_size=128)
        assert_same(gpu_hist(s, st), want, f"{name} w{w}")


@pytest.mark.parametrize("case", ADVERSARIAL, ids=[c[0] for c in ADVERSARIAL])
def test_adversarial_inputs_fp32_mode(case, oracle_lib):
    """The same inputs in fp32 mode: float32 histograms and the exact
    fp32/fp64 mismatch count (band certification off for most of them)."""
    name, build, m, tau, metric, radius = case
    s = build(np.random.default_rng(len(name)))
    st = AnalysisSettings(m, tau, metric, radius)
    h, t = run_analysis(embed(s, m, tau), st, precision="fp32")
    d, v, w, p, mism = oracle_lib.oracle_histograms_prec(s, m, tau, metric, radius, 0,
                                                         precision=32, tile_size=128)
    assert_same((h.diagonal, h.vertical, h.white_vertical, h.recurrence_points), (d, v, w, p),
                f"fp32 {name}")
    assert t["mismatched_cells"] == mism, (name, t["mismatched_cells"], mism)
