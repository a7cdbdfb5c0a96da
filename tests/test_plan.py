"""Host-side work-unit plan of the band kernel (rqa_capi.cu plan_units via the
rqa_plan_units diagnostic): CPU only, no device.

The plan replaces the reference's tile partition (engine.py:86-126) as the
unit of scheduling; the kernel's correctness relies on three invariants
checked here: every band's diagonal sweep [0, X_b) is covered exactly once
in order, every unit spans >= R iterations (a diagonal's band segment, R
consecutive iterations, is then cut by at most one unit boundary -- the
fix_diag_pieces contract), and X_b = ceil(rows_left / D) + R - 1.
"""

import ctypes

import numpy as np
import pytest

from paper_2402_16853_b200 import _native


def plan(n, lo, hi, slot_rows=256, r=4, slots=296):
    lib = _native.lib()
    count = ctypes.c_int64()
    assert lib.rqa_plan_units(n, lo, hi, slot_rows, r, slots, None, 0, ctypes.byref(count)) == 0
    buf = np.zeros(3 * count.value, np.int32)
    p32 = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    assert lib.rqa_plan_units(n, lo, hi, slot_rows, r, slots, p32, count.value,
                              ctypes.byref(count)) == 0
    return buf.reshape(-1, 3)


CASES = [(1_999, 0, 1_999), (99_996, 0, 99_996), (1 << 20, 0, 1 << 20),
         (1 << 20, 0, 136_192), (1 << 20, 650_240, 1 << 20), (500_000, 0, 500_000),
         (4_194_304, 0, 4_194_304), (1_025, 0, 1_025), (1, 0, 1), (5_000, 1_024, 3_000)]


@pytest.mark.parametrize("n,lo,hi", CASES)
def test_plan_covers_every_band_sweep_once(n, lo, hi):
    D, R = 256, 4
    H = D * R
    u = plan(n, lo, hi)
    nb = (hi - lo + H - 1) // H
    assert sorted(set(u[:, 0].tolist())) == list(range(nb))
    for b in range(nb):
        ub = u[u[:, 0] == b]
        X = (n - (lo + b * H) + D - 1) // D + R - 1
        assert ub[0, 1] == 0 and ub[-1, 2] == X, (b, ub[0], ub[-1], X)
        assert (ub[1:, 1] == ub[:-1, 2]).all()        # contiguous, in order
        lens = ub[:, 2] - ub[:, 1]
        assert (lens >= R).all(), (b, lens.min())       # >= R iterations per unit


def test_plan_balances_and_ends_with_small_units():
    u = plan(1 << 20, 0, 1 << 20)
    lens = u[:, 2] - u[:, 1]
    total = int(lens.sum())
    # waves = 16 (T / 887)^(1/3) = 32 waves of 296 resident CTAs (±50 %)
    assert 0.5 * 32 * 296 < len(u) < 1.5 * 32 * 296
    # the longest bands are cut into double-size units first and half-size
    # units in the last quarter of their sweep (short launch tail)
    b0 = u[u[:, 0] == 0]
    l0 = b0[:, 2] - b0[:, 1]
    assert l0[0] > 3 * l0[-1]
    assert total == sum((((1 << 20) - b * 1024 + 255) // 256 + 3)
                        for b in range(1024))


def test_plan_per_stripe_uses_fewer_waves():
    whole = plan(1 << 20, 0, 1 << 20)
    # an eighth of the triangle's area: 16 waves of smaller units
    stripe = plan(1 << 20, 0, 68_608)
    assert len(stripe) < len(whole) / 2


def test_plan_rejects_bad_arguments():
    lib = _native.lib()
    c = ctypes.c_int64()
    assert lib.rqa_plan_units(0, 0, 0, 256, 4, 296, None, 0, ctypes.byref(c)) != 0
    assert lib.rqa_plan_units(100, 50, 20, 256, 4, 296, None, 0, ctypes.byref(c)) != 0
    assert lib.rqa_plan_units(100, 0, 100, 100, 4, 296, None, 0, ctypes.byref(c)) != 0
    assert lib.rqa_plan_units(100, 0, 100, 256, 4, 0, None, 0, ctypes.byref(c)) != 0


def _unit_count_in_subprocess(env_extra):
    """Unit count of the full 2^20 plan in a fresh process (knobs are read once)."""
    import os
    import subprocess
    import sys

    code = ("import ctypes, sys; sys.path.insert(0, '.');"
            "from paper_2402_16853_b200 import _native; lib = _native.lib();"
            "c = ctypes.c_int64();"
            "assert lib.rqa_plan_units(1 << 20, 0, 1 << 20, 256, 4, 296, None, 0, ctypes.byref(c)) == 0;"
            "print(c.value)")
    env = dict(os.environ)
    for k in ("RQA_WAVES", "RQA_TAIL_FRAC", "RQA_MIN_UNIT"):
        env.pop(k, None)
    env.update(env_extra)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, check=True)
    return int(out.stdout.strip())


def test_empty_knobs_mean_default():
    # RQA_WAVES= (empty) used to parse as 0 -> one wave: a 2 % slower plan
    base = _unit_count_in_subprocess({})
    assert _unit_count_in_subprocess({"RQA_WAVES": "", "RQA_TAIL_FRAC": "",
                                      "RQA_MIN_UNIT": ""}) == base
    assert _unit_count_in_subprocess({"RQA_WAVES": "8"}) < base
