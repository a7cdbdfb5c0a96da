"""Recurrence plots as binary PBM (mirror of tiledrqa plotting.py:1-159).

The bits come from the GPU (rqa_block, csrc/rqa_plot.cu): each pixel is the
OR of a b x b block of matrix cells evaluated with the reference's
arithmetic, so a plot at reduction factor 1 is the analysed matrix bit for
bit.  Image orientation follows the recurrence-plot convention: matrix row 0
is the bottom image row.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .embedding import EmbeddedSeries
from .engine import DEFAULT_TILE_SIZE
from .errors import InvalidArgument, PlotTooLarge
from .settings import METRIC_CODES, AnalysisSettings

__all__ = ["MAX_PLOT_SIZE", "RecurrencePlot", "compute_plot", "write_pbm", "read_pbm", "render",
           "device_block"]

MAX_PLOT_SIZE = 65_536  # plotting.py:26


@dataclass(frozen=True)
class RecurrencePlot:
    """A possibly OR-reduced recurrence matrix, bit-packed row by row."""

    n_vectors: int
    reduction_factor: int
    size: int
    row_bits: np.ndarray

    def matrix(self) -> np.ndarray:
        """(size, size) bool matrix in matrix orientation."""
        return np.unpackbits(self.row_bits, axis=1, count=self.size).view(bool)


def device_block(embedded: EmbeddedSeries, settings: AnalysisSettings, row0: int, row1: int,
                 col0: int, col1: int, factor: int = 1, device: int = 0) -> np.ndarray:
    """Packed rows (uint8, MSB-first) of an OR-reduced matrix block, computed on the GPU."""
    s = np.ascontiguousarray(embedded.values, dtype=np.float64)
    rows = -(-(row1 - row0) // factor)
    cols = -(-(col1 - col0) // factor)
    out = np.zeros((rows, -(-cols // 8)), np.uint8)
    _native.call("rqa_block", s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), s.shape[0],
                 settings.embedding_dimension, settings.time_delay, METRIC_CODES[settings.metric],
                 float(settings.radius), settings.theiler_window, int(row0), int(row1), int(col0),
                 int(col1), int(factor), int(device),
                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    return out


def compute_plot(embedded: EmbeddedSeries, settings: AnalysisSettings, reduction_factor: int = 1,
                 tile_size: int = DEFAULT_TILE_SIZE, workers: int | None = None) -> RecurrencePlot:
    """The recurrence matrix reduced to plot resolution (plotting.py:48-90)."""
    if reduction_factor < 1:
        raise InvalidArgument("reduction_factor must be >= 1")
    if tile_size < 1:
        raise InvalidArgument("tile_size must be >= 1")
    if workers is not None and workers < 1:
        raise InvalidArgument("workers must be >= 1")
    n = embedded.n_vectors
    size = -(-n // reduction_factor)
    if size > MAX_PLOT_SIZE:
        raise PlotTooLarge(f"{size} pixels per side exceeds the {MAX_PLOT_SIZE} limit; "
                           "increase the reduction factor")
    bits = device_block(embedded, settings, 0, n, 0, n, reduction_factor)
    return RecurrencePlot(n, reduction_factor, size, bits)


def write_pbm(plot: RecurrencePlot, path) -> None:
    """Binary PBM (P4); matrix row 0 is written last (bottom of the image)."""
    with open(path, "wb") as fh:
        fh.write(f"P4\n{plot.size} {plot.size}\n".encode("ascii"))
        fh.write(plot.row_bits[::-1].tobytes())


def read_pbm(path) -> np.ndarray:
    """Parse a binary PBM into a bool array in image orientation (row 0 = top)."""
    with open(path, "rb") as fh:
        data = fh.read()
    fields, pos = [], 0
    while len(fields) < 3:
        end = data.index(b"\n", pos)
        line = data[pos:end].strip()
        pos = end + 1
        if not line or line.startswith(b"#"):
            continue
        fields.extend(line.split())
    if fields[0] != b"P4":
        raise InvalidArgument(f"not a binary PBM file: magic {fields[0]!r}")
    width, height = int(fields[1]), int(fields[2])
    row_bytes = -(-width // 8)
    raster = np.frombuffer(data[pos: pos + height * row_bytes], dtype=np.uint8)
    return np.unpackbits(raster.reshape(height, row_bytes), axis=1, count=width).view(bool)


def render(embedded: EmbeddedSeries, settings: AnalysisSettings, reduction_factor: int = 1,
           out="recurrence.pbm", tile_size: int = DEFAULT_TILE_SIZE,
           workers: int | None = None) -> RecurrencePlot:
    """Compute the plot and write it to a PBM file (plotting.py:151-159)."""
    plot = compute_plot(embedded, settings, reduction_factor, tile_size, workers)
    write_pbm(plot, out)
    return plot
