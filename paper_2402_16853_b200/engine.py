"""The drop-in boundary: run_analysis (mirror of tiledrqa engine.py:215-280).

``run_analysis(embedded, settings, tile_size, workers)`` keeps the
reference's signature, validation and return value ``(LineHistograms,
timing)``.  The work runs in librqa_b200.so on a B200 (csrc/): one fused
kernel evaluates the neighbourhood test, bit-packs rows with warp-level
transposes and extracts diagonal, vertical and white-vertical runs with
carries; a fold kernel stitches runs across band edges.  ``tile_size`` and
``workers`` are validated exactly as before and, like in the reference,
cannot change the integer result (engine.py:226-227); the device geometry is
chosen by the library.
"""

import ctypes
import os
import time

import numpy as np

from . import _native
from .embedding import EmbeddedSeries
from .errors import InvalidArgument
from .histograms import LineHistograms
from .settings import METRIC_CODES, AnalysisSettings

from .operators import (CarryoverBuffers, Tile, TileGrid, create_recurrence_matrix,  # noqa: E402,F401
                        detect_diagonal_lines, detect_vertical_lines, flush_carryovers,
                        partition)

__all__ = ["DEFAULT_TILE_SIZE", "TileGrid", "Tile", "CarryoverBuffers", "partition",
           "create_recurrence_matrix", "detect_diagonal_lines", "detect_vertical_lines",
           "flush_carryovers", "run_analysis", "default_workers", "device_count",
           "exact_threshold"]

DEFAULT_TILE_SIZE = 4096  # engine.py:44 (accepted, validated, geometry is device-chosen)


def default_workers() -> int:
    """engine.py:47-52: execution contexts when none are requested."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# precision keyword -> C-ABI code (rqa_run_prec); evaluation path reported in timing
PRECISIONS = {"fp64": 64, "fp32": 32}
FLAG_OUT_ZEROED = 1  # rqa_run_prec flags (include/rqa_b200.h)
# below this many vectors the default device list is one GPU: a stripe would be
# smaller than a few waves of work units and the gather/stitch would dominate
MULTI_DEVICE_MIN_VECTORS = 1 << 16
EVALUATION_PATHS = {-1: "fp64", 0: "f32-filter", 1: "fp32", 2: "fp64-prefilter"}


def device_count() -> int:
    return int(_native.lib().rqa_device_count())


def exact_threshold(metric: str, m: int, radius: float) -> float:
    """The kernels' threshold: T* for L2 with m > 1 (sqrt-free, exact), else radius."""
    out = ctypes.c_double()
    rc = _native.lib().rqa_threshold(METRIC_CODES[metric], m, float(radius), ctypes.byref(out))
    if rc != 0:
        raise InvalidArgument("invalid threshold arguments")
    return out.value


def _series_array(embedded: EmbeddedSeries) -> np.ndarray:
    return np.ascontiguousarray(embedded.values, dtype=np.float64)


def run_analysis(embedded: EmbeddedSeries, settings: AnalysisSettings,
                 tile_size: int = DEFAULT_TILE_SIZE, workers: int | None = None, *,
                 device: int | None = None, devices=None, precision: str = "fp64"):
    """Full analysis on the B200s of this process; returns (LineHistograms, timing).

    Mirrors run_analysis (engine.py:215-280): same arguments and validation;
    tile_size / workers do not change the results (as in the reference).
    ``devices``: CUDA device ids to split the rows over (one host thread per
    device, stripes stitched on the first; a device may repeat); default: the
    single ``device`` if given, else every visible GPU (one GPU below
    MULTI_DEVICE_MIN_VECTORS vectors).  Results do not depend on the device
    list.
    ``precision``: "fp64" (default) is bit-exact against the float64
    reference; "fp32" evaluates with float32 samples, arithmetic and radius
    and reports ``timing["mismatched_cells"]``, the number of cells of the
    full N x N matrix whose decision differs from the float64 one.

    timing keeps the reference keys (create_recurrence_matrix holds the fused
    kernel time, the two detector phases are fused into it and report 0.0)
    and adds h2d, fold, d2h, device_total, cells_per_second, band_rows,
    bands, evaluation ("fp64", "f32-filter" or "fp32"), f32_band.
    Multi-GPU runs go through ``paper_2402_16853_b200.distributed``.
    """
    if workers is None:
        workers = default_workers()
    if workers < 1:
        raise InvalidArgument("workers must be >= 1")  # engine.py:231-232
    if tile_size < 1:
        raise InvalidArgument("tile_size must be >= 1")  # engine.py:123-124
    if precision not in PRECISIONS:
        raise InvalidArgument(f"precision must be one of {sorted(PRECISIONS)}")
    # like the reference, the embedding parameters come from the embedded
    # series (recurrence_block reads embedded.embedding_dimension / time_delay,
    # embedding.py:137-143); settings' m / tau are not consulted here
    m, tau = embedded.embedding_dimension, embedded.time_delay
    if devices is None:
        if device is not None:
            devices = [device]
        else:  # every visible GPU, except for matrices too small to split usefully
            devices = list(range(max(1, device_count())))
            if embedded.n_vectors < MULTI_DEVICE_MIN_VECTORS:
                devices = devices[:1]
    devices = [int(d) for d in devices]
    if not devices:
        raise InvalidArgument("devices must not be empty")
    started = time.perf_counter()
    s = _series_array(embedded)
    n = embedded.n_vectors
    diag = np.zeros(n + 1, np.int64)
    vert = np.zeros(n + 1, np.int64)
    white = np.zeros(n + 1, np.int64)
    pts = np.zeros(1, np.int64)
    mism = np.zeros(1, np.int64)
    tim = np.zeros(_native.TIMING_SLOTS, np.float64)
    p64 = ctypes.POINTER(ctypes.c_int64)
    args = (s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), s.shape[0], m, tau,
            METRIC_CODES[settings.metric], float(settings.radius),
            settings.theiler_window, PRECISIONS[precision])
    outs = (diag.ctypes.data_as(p64), vert.ctypes.data_as(p64), white.ctypes.data_as(p64),
            pts.ctypes.data_as(p64), mism.ctypes.data_as(p64),
            tim.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if len(devices) == 1:  # outputs are fresh np.zeros: only nonzero bins come back
        _native.call("rqa_run_prec", *args, devices[0], FLAG_OUT_ZEROED, *outs)
    else:
        dv = (ctypes.c_int32 * len(devices))(*devices)
        _native.call("rqa_run_multi", *args, dv, len(devices), FLAG_OUT_ZEROED, *outs)
    hist = LineHistograms(n, int(pts[0]), diag, vert, white)
    timing = {
        "create_recurrence_matrix": float(tim[1]),
        "detect_diagonal_lines": 0.0,
        "detect_vertical_lines": 0.0,
        "h2d": float(tim[0]),
        "fold": float(tim[2]),
        "d2h": float(tim[3]),
        "device_total": float(tim[4]),
        "cells_per_second": float(tim[5]),
        "band_rows": int(tim[6]),
        "bands": int(tim[7]),
        "evaluation": EVALUATION_PATHS.get(int(tim[8]), "fp64"),
        "devices": devices,
        "f32_band": float(tim[9]),
        "prefilter_candidates": float(tim[10]),
        "total": time.perf_counter() - started,
    }
    if precision == "fp32":
        timing["mismatched_cells"] = int(mism[0])
    return hist, timing
