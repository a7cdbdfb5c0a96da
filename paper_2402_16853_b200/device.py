"""Device-resident entry points over torch CUDA tensors.

torch is used only as plumbing here (device memory and streams); the work is
done by librqa_b200.so through the C-ABI (rqa_run_device / rqa_stitch_device).
"""

import ctypes
from dataclasses import dataclass

from . import _native
from .settings import METRIC_CODES, AnalysisSettings

PRECISIONS = {"fp64": 64, "fp32": 32}

__all__ = ["band_rows", "run_rows_device", "stitch_device", "StripeOutputs", "MODE_FINAL",
           "MODE_STRIPE"]

MODE_FINAL = 0
MODE_STRIPE = 1


def band_rows(settings: AnalysisSettings, n: int) -> int:
    """Rows per CTA band of the kernel variant chosen for these settings and n vectors."""
    h = ctypes.c_int64()
    r = ctypes.c_int32()
    rc = _native.lib().rqa_band_rows(METRIC_CODES[settings.metric], settings.embedding_dimension,
                                     settings.time_delay, int(n), ctypes.byref(h), ctypes.byref(r))
    if rc != 0:
        raise ValueError("no kernel variant for these settings")
    return int(h.value)


@dataclass
class StripeOutputs:
    """Per-stripe summaries of a multi-GPU run (see include/rqa_b200.h)."""

    prefix: object   # int32 [n]
    suffix: object   # int32 [n]
    col: object      # int32 [2n] (uint32 bit patterns): column part (first, last run)
    rowlead: object  # int32 [2n] (uint32 bit patterns): row part (first, last), zero-init

    @staticmethod
    def empty(n: int, device, rows: int = 1):
        import torch

        shape = (rows, n) if rows > 1 else (n,)
        cshape = (rows, 2 * n) if rows > 1 else (2 * n,)
        return StripeOutputs(torch.zeros(shape, dtype=torch.int32, device=device),
                             torch.zeros(shape, dtype=torch.int32, device=device),
                             torch.zeros(cshape, dtype=torch.int32, device=device),
                             torch.zeros(2 * n, dtype=torch.int32, device=device))


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def run_rows_device(series, settings: AnalysisSettings, row_lo: int, row_hi: int, mode: int,
                    hist, points, stripe: StripeOutputs | None = None, stream=None,
                    precision: str = "fp64", mismatches=None) -> None:
    """Enqueue the band + fold kernels for rows [row_lo, row_hi) on ``stream``.

    series: float64 CUDA tensor of samples; hist: int64 CUDA tensor [3, n+1]
    and points: int64 CUDA tensor [1], both accumulated into.  precision
    "fp32" needs ``mismatches`` (int64 CUDA tensor [1], accumulated into).
    """
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(series.device)
    so = stripe if stripe is not None else StripeOutputs(None, None, None, None)
    _native.call("rqa_run_device_prec", _ptr(series), series.numel(),
                 settings.embedding_dimension, settings.time_delay,
                 METRIC_CODES[settings.metric], float(settings.radius),
                 settings.theiler_window, PRECISIONS[precision], int(row_lo), int(row_hi),
                 int(mode), _ptr(hist), _ptr(points), _ptr(mismatches), _ptr(so.prefix),
                 _ptr(so.suffix), _ptr(so.col), _ptr(so.rowlead),
                 ctypes.c_void_p(stream.cuda_stream))


def stitch_device(gathered: StripeOutputs, bounds, n: int, hist, stream=None) -> None:
    """Fold the gathered stripe summaries ([G, n] / [G, 2n] / summed rowlead) into hist."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(gathered.prefix.device)
    b = (ctypes.c_int64 * len(bounds))(*[int(x) for x in bounds])
    _native.call("rqa_stitch_device", _ptr(gathered.prefix), _ptr(gathered.suffix),
                 _ptr(gathered.col), _ptr(gathered.rowlead), b, len(bounds) - 1, int(n),
                 _ptr(hist), ctypes.c_void_p(stream.cuda_stream))
