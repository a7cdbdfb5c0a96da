"""The reference's per-tile operator API (tiledrqa engine.py:55-212), GPU-backed.

``run_analysis`` never materialises tiles (the fused kernel keeps the bits in
registers), but callers that drive the tiled engine themselves -- partition
the matrix, fill tiles, scan them in wave order with carry-over buffers and
flush -- find the same objects and functions here:

* ``Tile``, ``TileGrid``, ``partition``, ``CarryoverBuffers``: host geometry
  and state, identical fields and checks (engine.py:55-153);
* ``create_recurrence_matrix``: the tile's bits from the GPU (rqa_block,
  csrc/rqa_plot.cu), packed like ``np.packbits(block)`` (engine.py:156-164);
* ``detect_diagonal_lines`` / ``detect_vertical_lines``: the scans on the GPU
  (rqa_tile_scan, csrc/rqa_tiles.cu, one thread per diagonal / column) with
  the reference's dependency checks on the host (engine.py:167-192,
  322-433);
* ``flush_carryovers``: closes the open runs (engine.py:195-212).

Results are identical to the reference operators for every tile size.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .embedding import EmbeddedSeries
from .errors import DependencyViolation, InvalidArgument
from .histograms import LineHistograms
from .settings import AnalysisSettings

__all__ = ["Tile", "TileGrid", "partition", "CarryoverBuffers", "create_recurrence_matrix",
           "detect_diagonal_lines", "detect_vertical_lines", "flush_carryovers"]


@dataclass
class Tile:
    """One sub-matrix; ``bits`` is row-major, MSB-first, ceil(h*w/8) bytes (engine.py:55-83)."""

    row_offset: int
    col_offset: int
    height: int
    width: int
    bits: np.ndarray | None = None

    def matrix(self) -> np.ndarray:
        if self.bits is None:
            raise DependencyViolation(
                "tile bits are absent; run create_recurrence_matrix first")
        flat = np.unpackbits(self.bits, count=self.height * self.width)
        return flat.reshape(self.height, self.width).view(bool)

    def count_points(self) -> int:
        if self.bits is None:
            raise DependencyViolation(
                "tile bits are absent; run create_recurrence_matrix first")
        return int(np.unpackbits(self.bits, count=self.height * self.width).sum())


@dataclass(frozen=True)
class TileGrid:
    """Tile (r, c) covers rows [r*T, min((r+1)*T, N)) x the same columns (engine.py:86-116)."""

    n_vectors: int
    tile_size: int
    rows_of_tiles: int
    cols_of_tiles: int

    def tile(self, r: int, c: int) -> Tile:
        if not (0 <= r < self.rows_of_tiles and 0 <= c < self.cols_of_tiles):
            raise InvalidArgument(f"tile ({r}, {c}) outside the grid")
        n, t = self.n_vectors, self.tile_size
        return Tile(r * t, c * t, min((r + 1) * t, n) - r * t, min((c + 1) * t, n) - c * t)

    def waves(self):
        """Anti-diagonal waves {(r, s - r)} in dependency order (engine.py:111-116)."""
        for s in range(self.rows_of_tiles + self.cols_of_tiles - 1):
            r_lo = max(0, s - self.cols_of_tiles + 1)
            r_hi = min(self.rows_of_tiles - 1, s)
            yield [(r, s - r) for r in range(r_lo, r_hi + 1)]


def partition(n_vectors: int, tile_size: int) -> TileGrid:
    """engine.py:119-126."""
    if n_vectors < 1:
        raise InvalidArgument("n_vectors must be >= 1")
    if tile_size < 1:
        raise InvalidArgument("tile_size must be >= 1")
    blocks = -(-n_vectors // tile_size)
    return TileGrid(n_vectors, tile_size, blocks, blocks)


class CarryoverBuffers:
    """Open-run lengths per diagonal k + N - 1 and per column, plus scan progress
    (engine.py:129-153)."""

    def __init__(self, n_vectors: int):
        if n_vectors < 1:
            raise InvalidArgument("n_vectors must be >= 1")
        n = n_vectors
        self.n_vectors = n
        self.diagonal = np.zeros(2 * n - 1, dtype=np.int64)
        self.vertical = np.zeros(n, dtype=np.int64)
        self.white_vertical = np.zeros(n, dtype=np.int64)
        k = np.arange(2 * n - 1) - (n - 1)
        self.diagonal_progress = np.maximum(0, -k)
        self.vertical_progress = np.zeros(n, dtype=np.int64)


def create_recurrence_matrix(tile: Tile, embedded: EmbeddedSeries,
                             settings: AnalysisSettings, *, device: int = 0) -> Tile:
    """Fill the tile's bits on the GPU (engine.py:156-164)."""
    from .plotting import device_block

    packed = device_block(embedded, settings, tile.row_offset, tile.row_offset + tile.height,
                          tile.col_offset, tile.col_offset + tile.width, 1, device=device)
    rows = np.unpackbits(packed, axis=1, count=tile.width)
    tile.bits = np.packbits(rows)  # row-major flat layout of the reference
    return tile


def _ptr(a, ctype=ctypes.c_int64):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _tile_bits(tile: Tile) -> np.ndarray:
    if tile.bits is None:
        raise DependencyViolation("tile bits are absent; run create_recurrence_matrix first")
    return np.ascontiguousarray(tile.bits, dtype=np.uint8)


def detect_diagonal_lines(tile: Tile, carryover: CarryoverBuffers,
                          histograms: LineHistograms, *, device: int = 0) -> None:
    """Diagonal runs of the tile with carries (engine.py:167-172, 398-433)."""
    bits = _tile_bits(tile)
    h, w, n = tile.height, tile.width, carryover.n_vectors
    offsets = np.arange(-(h - 1), w)
    seg_start = np.maximum(0, -offsets)
    seg_end = np.minimum(h, w - offsets)
    ids = (tile.col_offset - tile.row_offset) + offsets + (n - 1)
    if not np.array_equal(carryover.diagonal_progress[ids], tile.row_offset + seg_start):
        raise DependencyViolation(
            f"diagonal detection of tile at ({tile.row_offset}, {tile.col_offset}) ran before "
            f"an earlier tile on one of its diagonals finished")
    lo = int(ids[0])
    carry = np.ascontiguousarray(carryover.diagonal[lo: lo + h + w - 1])
    _native.call("rqa_tile_scan", _ptr(bits, ctypes.c_uint8), h, w, n, 0, _ptr(carry), None,
                 _ptr(histograms.diagonal), None, int(device))
    carryover.diagonal[lo: lo + h + w - 1] = carry
    carryover.diagonal_progress[ids] = tile.row_offset + seg_end


def detect_vertical_lines(tile: Tile, carryover: CarryoverBuffers,
                          histograms: LineHistograms, *, device: int = 0) -> None:
    """Vertical runs of ones and zeroes with carries (engine.py:175-192, 338-361)."""
    bits = _tile_bits(tile)
    h, w = tile.height, tile.width
    cols = slice(tile.col_offset, tile.col_offset + w)
    if not (carryover.vertical_progress[cols] == tile.row_offset).all():
        raise DependencyViolation(
            f"vertical detection of tile at ({tile.row_offset}, {tile.col_offset}) ran before "
            f"the tile above finished")
    cv = np.ascontiguousarray(carryover.vertical[cols])
    cw = np.ascontiguousarray(carryover.white_vertical[cols])
    _native.call("rqa_tile_scan", _ptr(bits, ctypes.c_uint8), h, w, carryover.n_vectors, 1,
                 _ptr(cv), _ptr(cw), _ptr(histograms.vertical), _ptr(histograms.white_vertical),
                 int(device))
    carryover.vertical[cols] = cv
    carryover.white_vertical[cols] = cw
    carryover.vertical_progress[cols] = tile.row_offset + h


def flush_carryovers(carryover: CarryoverBuffers, histograms: LineHistograms) -> LineHistograms:
    """Count every still-open run at its truncated length and zero the buffers
    (engine.py:195-212)."""
    for buffer, counts in ((carryover.diagonal, histograms.diagonal),
                           (carryover.vertical, histograms.vertical),
                           (carryover.white_vertical, histograms.white_vertical)):
        open_lengths = buffer[buffer > 0]
        if open_lengths.size:
            binned = np.bincount(open_lengths)
            counts[: binned.size] += binned
        buffer[:] = 0
    return histograms
