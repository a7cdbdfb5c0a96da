"""ctypes wrapper of the CPU oracle (oracle/rqa_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
(paper_2402_16853_b200) never imports this module.

The oracle restates tiledrqa's run_analysis (engine.py:215-280) tile by tile
in C; its parity against the reference is pinned by tests/golden/ fixtures
generated from tiledrqa itself (tests/golden/make_golden.py).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

METRICS = {"l1": 0, "l2": 1, "linf": 2}


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH)
            < os.path.getmtime(os.path.join(_HERE, "rqa_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_run.argtypes = [
            ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int32,
            ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_int32, i64p, i64p, i64p, i64p]
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run_prec.argtypes = [
            ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int32,
            ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, i64p, i64p, i64p, i64p, i64p]
        lib.oracle_run_prec.restype = ctypes.c_int
        lib.oracle_matrix_prec.argtypes = [
            ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int32,
            ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int64,
            ctypes.c_int32, ctypes.POINTER(ctypes.c_uint8)]
        lib.oracle_matrix_prec.restype = ctypes.c_int
        lib.oracle_matrix.argtypes = [
            ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int32,
            ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_uint8)]
        lib.oracle_matrix.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def oracle_histograms(values, m, tau, metric, radius, theiler=0,
                      tile_size=512, workers=None):
    """Run the C restatement; returns (diag, vert, white, points).

    theiler: 0 keeps the main diagonal (reference default), 1 is the
    reference's include_main_diagonal=False, w>1 zeroes |i-j| < w.
    """
    lib = _load()
    s = np.ascontiguousarray(values, dtype=np.float64)
    n = s.shape[0] - (m - 1) * tau
    if n < 1:
        raise ValueError("series too short")
    if workers is None:
        workers = len(os.sched_getaffinity(0))
    diag = np.zeros(n + 1, np.int64)
    vert = np.zeros(n + 1, np.int64)
    white = np.zeros(n + 1, np.int64)
    pts = np.zeros(1, np.int64)
    rc = lib.oracle_run(_ptr(s, ctypes.c_double), s.shape[0], m, tau,
                        METRICS[metric], float(radius), int(theiler),
                        int(tile_size), int(workers),
                        _ptr(diag, ctypes.c_int64), _ptr(vert, ctypes.c_int64),
                        _ptr(white, ctypes.c_int64), _ptr(pts, ctypes.c_int64))
    if rc != 0:
        raise RuntimeError(f"oracle_run failed with {rc}")
    return diag, vert, white, int(pts[0])


def oracle_histograms_prec(values, m, tau, metric, radius, theiler=0,
                           precision=64, tile_size=512, workers=None):
    """As oracle_histograms, with precision 64 or 32 (fp32 mode extension);
    returns (diag, vert, white, points, mismatched_cells), the last being the
    number of cells of the full N x N matrix whose fp32 decision differs from
    the float64 one (0 for precision 64)."""
    lib = _load()
    s = np.ascontiguousarray(values, dtype=np.float64)
    n = s.shape[0] - (m - 1) * tau
    if n < 1:
        raise ValueError("series too short")
    if workers is None:
        workers = len(os.sched_getaffinity(0))
    diag = np.zeros(n + 1, np.int64)
    vert = np.zeros(n + 1, np.int64)
    white = np.zeros(n + 1, np.int64)
    pts = np.zeros(1, np.int64)
    mism = np.zeros(1, np.int64)
    rc = lib.oracle_run_prec(_ptr(s, ctypes.c_double), s.shape[0], m, tau,
                             METRICS[metric], float(radius), int(theiler),
                             int(tile_size), int(workers), int(precision),
                             _ptr(diag, ctypes.c_int64), _ptr(vert, ctypes.c_int64),
                             _ptr(white, ctypes.c_int64), _ptr(pts, ctypes.c_int64),
                             _ptr(mism, ctypes.c_int64))
    if rc != 0:
        raise RuntimeError(f"oracle_run_prec failed with {rc}")
    return diag, vert, white, int(pts[0]), int(mism[0])


def oracle_matrix(values, m, tau, metric, radius, theiler=0, precision=64):
    """Full recurrence matrix (bool N x N) for small N."""
    lib = _load()
    s = np.ascontiguousarray(values, dtype=np.float64)
    n = s.shape[0] - (m - 1) * tau
    out = np.zeros((n, n), np.uint8)
    rc = lib.oracle_matrix_prec(_ptr(s, ctypes.c_double), s.shape[0], m, tau,
                                METRICS[metric], float(radius), int(theiler),
                                int(precision), _ptr(out, ctypes.c_uint8))
    if rc != 0:
        raise RuntimeError(f"oracle_matrix failed with {rc}")
    return out.astype(bool)


def theiler_of(settings) -> int:
    """Map settings (reference include_main_diagonal / extension) to w."""
    w = getattr(settings, "theiler_corrector", None)
    if w is not None:
        return int(w)
    return 0 if settings.include_main_diagonal else 1
