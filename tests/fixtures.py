"""Loading of the golden fixtures (tests/golden/, made by make_golden.py)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def dense(sparse: dict, n: int) -> np.ndarray:
    out = np.zeros(n + 1, np.int64)
    for k, v in sparse.items():
        out[int(k)] = v
    return out


def load_cases(name: str):
    """[(series, settings_dict, result_dict, meta)] of small_cases / theiler_cases."""
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)["cases"]
    arrays = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return [(arrays[f"s{c['id']}"], c["settings"], c["result"], c) for c in meta]


def load_config(tag: str):
    with open(os.path.join(GOLDEN, f"config_{tag}.json")) as fh:
        return json.load(fh)


def config_tags():
    return sorted(f[len("config_"):-len(".json")] for f in os.listdir(GOLDEN)
                  if f.startswith("config_") and f.endswith(".json"))


def theiler_of(settings: dict) -> int:
    if settings.get("theiler_corrector") is not None:
        return int(settings["theiler_corrector"])
    return 0 if settings["include_main_diagonal"] else 1


def result_arrays(result: dict):
    n = result["n_vectors"]
    return (dense(result["diagonal"], n), dense(result["vertical"], n),
            dense(result["white_vertical"], n), int(result["recurrence_points"]))


def settings_obj(settings: dict):
    from paper_2402_16853_b200 import AnalysisSettings

    kw = dict(settings)
    return AnalysisSettings(**kw)


def assert_same(got, want, label=""):
    """got/want: (diag, vert, white, points)."""
    gd, gv, gw, gp = got
    wd, wv, ww, wp = want
    assert gp == wp, f"{label}: points {gp} != {wp}"
    for name, a, b in (("diagonal", gd, wd), ("vertical", gv, wv), ("white", gw, ww)):
        if not np.array_equal(a, b):
            idx = np.flatnonzero(a != b)[:8]
            raise AssertionError(f"{label}: {name} differs at lengths {idx.tolist()}: "
                                 f"got {a[idx].tolist()} want {b[idx].tolist()}")
