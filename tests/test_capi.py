"""The C-ABI library loads and exports every symbol of include/rqa_b200.h.

These tests make no compute calls that need a GPU; without a device the
compute entry points must fail loudly (no CPU fallback).
"""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2402_16853_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "rqa_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+\*?(rqa_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_symbols():
    syms = header_symbols()
    assert "rqa_run" in syms and "rqa_run_device" in syms and "rqa_stitch_device" in syms
    assert set(syms) == set(_native.SYMBOLS), "ctypes table and header disagree"


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_version_and_counter():
    lib = _native.lib()
    assert lib.rqa_version() == 10000
    assert lib.rqa_launch_counter() >= 0


def _thr(metric, m, r):
    out = ctypes.c_double()
    assert _native.lib().rqa_threshold(metric, m, r, ctypes.byref(out)) == 0
    return out.value


def test_exact_threshold_brackets_sqrt():
    """T* = max{x : RN(sqrt(x)) <= eps}."""
    rng = np.random.default_rng(3)
    radii = list(rng.uniform(0, 10, 300)) + list(10.0 ** rng.uniform(-150, 150, 300))
    radii += [0.0, 5e-324, 1.0, 0.1, 1e154, 1.3407807929942596e154, 1e200, 1.7976931348623157e308]
    for eps in radii:
        t = _thr(1, 3, eps)
        assert math.sqrt(t) <= eps
        nxt = math.nextafter(t, math.inf)
        assert math.isinf(nxt) or math.sqrt(nxt) > eps
    assert _thr(1, 3, math.inf) == math.inf
    # L1 / Linf / m == 1 use the radius itself
    assert _thr(0, 3, 0.25) == 0.25 and _thr(2, 3, 0.25) == 0.25 and _thr(1, 1, 0.25) == 0.25


def test_eps_squared_is_not_the_threshold():
    """The naive eps*eps differs from T* for a large share of radii."""
    rng = np.random.default_rng(4)
    radii = rng.uniform(0, 1, 2000)
    differ = sum(_thr(1, 2, float(e)) != float(e) * float(e) for e in radii)
    assert differ > 200


def test_band_rows():
    h = ctypes.c_int64()
    r = ctypes.c_int32()
    lib = _native.lib()
    assert lib.rqa_band_rows(1, 3, 1, 1 << 20, ctypes.byref(h), ctypes.byref(r)) == 0
    assert h.value == 1024 and r.value == 1
    assert lib.rqa_band_rows(1, 3, 1, 100000, ctypes.byref(h), ctypes.byref(r)) == 0
    assert h.value == 1024 and r.value == 1           # work units balance any n
    assert lib.rqa_band_rows(0, 10, 5, 500000, ctypes.byref(h), ctypes.byref(r)) == 0
    assert r.value == 1                               # C4 has a reuse variant
    assert lib.rqa_band_rows(0, 17, 3, 500000, ctypes.byref(h), ctypes.byref(r)) == 0
    assert r.value == 0                               # runtime (m, tau) kernel
    assert lib.rqa_band_rows(5, 3, 1, 1000, ctypes.byref(h), ctypes.byref(r)) != 0


def test_invalid_arguments_map_to_reference_errors():
    from paper_2402_16853_b200 import AnalysisSettings, InvalidArgument, SeriesTooShort, embed
    from paper_2402_16853_b200.engine import run_analysis

    e = embed(np.arange(10.0), 2, 3)
    with pytest.raises(InvalidArgument):
        run_analysis(e, AnalysisSettings(2, 3, radius=1.0), workers=0)
    with pytest.raises(InvalidArgument):
        run_analysis(e, AnalysisSettings(2, 3, radius=1.0), tile_size=0)
    with pytest.raises(SeriesTooShort):
        embed(np.arange(4.0), 3, 2)


@pytest.mark.skipif(_native.lib().rqa_device_count() > 0, reason="a GPU is present")
def test_no_cpu_fallback_without_gpu():
    from paper_2402_16853_b200 import AnalysisSettings, DeviceError, embed
    from paper_2402_16853_b200.engine import run_analysis

    e = embed(np.sin(np.arange(100.0)), 2, 1)
    with pytest.raises(DeviceError):
        run_analysis(e, AnalysisSettings(2, 1, radius=0.5))
