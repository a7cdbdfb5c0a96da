"""Generate golden fixtures from the reference implementation (tiledrqa).

Run IN THE BUILD CONTAINER ONLY (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py [--skip-large]

Outputs (committed):
  tests/golden/small_cases.npz / small_cases.json
      >= 200 random cases in the SPEC.md:465 matrix (families uniform /
      sine_noise / ar1, m 1..5, tau 1..5, all metrics, radii from sparse to
      dense, main diagonal on/off), results of tiledrqa.oracle_analyze,
      cross-checked against tiledrqa.run_analysis at two tile sizes.
  tests/golden/theiler_cases.npz / theiler_cases.json
      Theiler window w > 1 (extension, not expressible in the reference):
      results of an extended copy of oracle_analyze whose only change is the
      generalised zeroing |i-j| < w (embedding.py:158-171 generalised).
  tests/golden/config_<name>.json
      Reference run_analysis on the benchmark workloads (full C1, C2 and
      prefix samples of C3, C4, C5 and the paper sine), with the SHA-256 of
      the input bytes.
"""

import argparse
import json
import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
COPY = "/tmp/tiledrqa_ref_copy"


def import_reference():
    """Import tiledrqa from a scratch copy (the reference tree is read-only)."""
    if not os.path.isdir(COPY):
        shutil.copytree(REF_SRC, os.path.join(COPY, "src"))
        shutil.copytree(REF_TESTS, os.path.join(COPY, "tests"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(COPY, "src"))
    sys.path.insert(0, os.path.join(COPY, "tests"))
    import helpers  # noqa: E402  (reference tests/helpers.py)
    import tiledrqa  # noqa: E402
    return tiledrqa, helpers


def hist_to_json(h):
    d = h.to_dicts()
    return {"n_vectors": int(h.n_vectors), "recurrence_points": int(h.recurrence_points),
            "diagonal": {str(k): v for k, v in d["diagonal"].items()},
            "vertical": {str(k): v for k, v in d["vertical"].items()},
            "white_vertical": {str(k): v for k, v in d["white_vertical"].items()}}


def measures_to_json(res):
    return {k: (None if v is None else float(v)) for k, v in res.measures_dict().items()}


def small_cases(t, helpers, count=240, seed=20260417):
    rng = np.random.default_rng(seed)
    metrics = ["l1", "l2", "linf"]
    quantiles = [0.0, 0.02, 0.1, 0.3, 0.6, 0.9, 1.0]
    edge_lengths = [33, 40, 64, 65, 96, 97, 128, 129, 160, 257, 300, 511, 520]
    series, meta = {}, []
    for i in range(count):
        fam = helpers.FAMILIES[i % 3]
        length = int(edge_lengths[i % len(edge_lengths)] if i % 4 == 0 else rng.integers(50, 501))
        m = int(rng.integers(1, 6))
        tau = int(rng.integers(1, 6))
        if (m - 1) * tau >= length - 8:
            tau = 1
        metric = metrics[(i // 3) % 3]
        q = float(quantiles[int(rng.integers(0, len(quantiles)))])
        incl = bool(rng.integers(0, 2))
        data = helpers.make_series(rng, fam, length)
        emb = t.embed(data, m, tau)
        radius = helpers.radius_for_quantile(rng, emb, metric, q)
        st = t.AnalysisSettings(embedding_dimension=m, time_delay=tau, metric=metric,
                                radius=radius, include_main_diagonal=incl)
        h, _ = t.oracle_analyze(emb, st)
        for tile in (7, 64):
            h2, _ = t.run_analysis(emb, st, tile_size=tile, workers=2)
            assert h2 == h, f"reference self-check failed for case {i}"
        series[f"s{i}"] = np.asarray(data, np.float64)
        meta.append({"id": i, "family": fam, "settings": st.to_dict(),
                     "quantile": q, "result": hist_to_json(h),
                     "measures": measures_to_json(t.compute_measures(h, st))})
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **series)
    with open(os.path.join(HERE, "small_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "tiledrqa 0.1.0",
                   "cases": meta}, fh)
    print(f"small cases: {len(meta)}")


def extended_oracle(t, emb, settings, w):
    """tiledrqa.oracle_analyze with the zeroing generalised to |i-j| < w."""
    n = emb.n_vectors
    base = t.AnalysisSettings(embedding_dimension=settings.embedding_dimension,
                              time_delay=settings.time_delay, metric=settings.metric,
                              radius=settings.radius, include_main_diagonal=True)
    matrix = t.recurrence_block(emb, base, 0, n, 0, n)
    ii, jj = np.indices((n, n))
    matrix[np.abs(ii - jj) < w] = False
    h = t.LineHistograms(n, recurrence_points=int(matrix.sum()))
    for k in range(-(n - 1), n):
        for length in t.run_lengths(np.diagonal(matrix, offset=k)):
            h.diagonal[length] += 1
    for j in range(n):
        col = matrix[:, j]
        for length in t.run_lengths(col):
            h.vertical[length] += 1
        for length in t.run_lengths(~col):
            h.white_vertical[length] += 1
    return h


def theiler_cases(t, helpers, count=36, seed=77):
    rng = np.random.default_rng(seed)
    series, meta = {}, []
    for i in range(count):
        fam = helpers.FAMILIES[i % 3]
        length = int(rng.integers(60, 400))
        m = int(rng.integers(1, 5))
        tau = int(rng.integers(1, 4))
        metric = ["l1", "l2", "linf"][i % 3]
        w = [2, 3, 5, 10, 33][i % 5]
        data = helpers.make_series(rng, fam, length)
        emb = t.embed(data, m, tau)
        radius = helpers.radius_for_quantile(rng, emb, metric, float(rng.choice([0.05, 0.3, 0.8])))
        st = t.AnalysisSettings(embedding_dimension=m, time_delay=tau, metric=metric,
                                radius=radius)
        h = extended_oracle(t, emb, st, w)
        if i < 6:  # w = 1 must coincide with the reference's own exclusion
            st1 = t.AnalysisSettings(embedding_dimension=m, time_delay=tau, metric=metric,
                                     radius=radius, include_main_diagonal=False)
            assert extended_oracle(t, emb, st, 1) == t.oracle_analyze(emb, st1)[0]
        s = st.to_dict()
        s["theiler_corrector"] = w
        series[f"s{i}"] = np.asarray(data, np.float64)
        meta.append({"id": i, "settings": s, "result": hist_to_json(h)})
    np.savez_compressed(os.path.join(HERE, "theiler_cases.npz"), **series)
    with open(os.path.join(HERE, "theiler_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "extended copy of tiledrqa.oracle_analyze (Theiler w > 1)",
                   "cases": meta}, fh)
    print(f"theiler cases: {len(meta)}")


def config_fixture(t, name, length=None, theiler_override=None):
    sys.path.insert(0, REPO)
    from paper_2402_16853_b200.workloads import WORKLOADS, series_sha256

    wl = WORKLOADS[name]
    data = wl.series(length)
    s = wl.settings
    incl = s.include_main_diagonal if theiler_override is None else theiler_override == 0
    st = t.AnalysisSettings(embedding_dimension=s.embedding_dimension, time_delay=s.time_delay,
                            metric=s.metric, radius=s.radius, include_main_diagonal=incl)
    emb = t.embed(data, st.embedding_dimension, st.time_delay)
    t0 = time.perf_counter()
    h, timing = t.run_analysis(emb, st, tile_size=4096, workers=len(os.sched_getaffinity(0)))
    wall = time.perf_counter() - t0
    out = {"workload": name, "samples": int(data.shape[0]), "prefix": length is not None,
           "sha256": series_sha256(data), "settings": st.to_dict(),
           "result": hist_to_json(h), "measures": measures_to_json(t.compute_measures(h, st)),
           "reference_wall_s": wall, "reference_workers": len(os.sched_getaffinity(0))}
    tag = name if length is None else f"{name}_{emb.n_vectors}"
    with open(os.path.join(HERE, f"config_{tag}.json"), "w") as fh:
        json.dump(out, fh)
    print(f"config {tag}: n={emb.n_vectors} points={h.recurrence_points} wall={wall:.1f}s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-large", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    t, helpers = import_reference()
    only = set(args.only.split(",")) if args.only else None
    if only is None or "small" in only:
        small_cases(t, helpers)
    if only is None or "theiler" in only:
        theiler_cases(t, helpers)
    if only is None or "C1" in only:
        config_fixture(t, "C1")
    if args.skip_large:
        return
    if only is None or "C5" in only:
        config_fixture(t, "C5", 32_770)
    if only is None or "C4" in only:
        config_fixture(t, "C4", 16_429, theiler_override=1)
    if only is None or "P" in only:
        config_fixture(t, "P", 20_002)
    if only is None or "C3" in only:
        config_fixture(t, "C3", 65_538)
    if only is None or "C2" in only:
        config_fixture(t, "C2")


if __name__ == "__main__":
    main()
