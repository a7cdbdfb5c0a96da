"""Device-resident entry points over torch CUDA tensors.

torch is used only as plumbing here (device memory and streams); the work is
done by librqa_b200.so through the C-ABI (rqa_run_device / rqa_stitch_device).
"""

import ctypes

from . import _native
from .settings import METRIC_CODES, AnalysisSettings

__all__ = ["band_rows", "run_rows_device", "stitch_device", "MODE_FINAL", "MODE_STRIPE"]

MODE_FINAL = 0
MODE_STRIPE = 1


def band_rows(settings: AnalysisSettings) -> int:
    """Rows per CTA band of the kernel variant chosen for these settings."""
    h = ctypes.c_int64()
    r = ctypes.c_int32()
    rc = _native.lib().rqa_band_rows(METRIC_CODES[settings.metric], settings.embedding_dimension,
                                     settings.time_delay, ctypes.byref(h), ctypes.byref(r))
    if rc != 0:
        raise ValueError("no kernel variant for these settings")
    return int(h.value)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def run_rows_device(series, settings: AnalysisSettings, row_lo: int, row_hi: int, mode: int,
                    hist, points, stripe_prefix=None, stripe_suffix=None, stream=None) -> None:
    """Enqueue the band + fold kernels for rows [row_lo, row_hi) on ``stream``.

    series: float64 CUDA tensor of samples; hist: int64 CUDA tensor [3, n+1]
    and points: int64 CUDA tensor [1], both accumulated into.
    """
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(series.device)
    _native.call("rqa_run_device", _ptr(series), series.numel(),
                 settings.embedding_dimension, settings.time_delay,
                 METRIC_CODES[settings.metric], float(settings.radius),
                 settings.theiler_window, int(row_lo), int(row_hi), int(mode),
                 _ptr(hist), _ptr(points), _ptr(stripe_prefix), _ptr(stripe_suffix),
                 ctypes.c_void_p(stream.cuda_stream))


def stitch_device(prefix, suffix, bounds, n: int, hist, stream=None) -> None:
    """Fold the gathered stripe summaries ([G, n] int32 CUDA) into hist."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(prefix.device)
    b = (ctypes.c_int64 * len(bounds))(*[int(x) for x in bounds])
    _native.call("rqa_stitch_device", _ptr(prefix), _ptr(suffix), b, len(bounds) - 1, int(n),
                 _ptr(hist), ctypes.c_void_p(stream.cuda_stream))
