"""The reference's per-tile operator API (operators.py) on the GPU.

Driving partition -> waves -> create_recurrence_matrix -> detect_*_lines ->
flush_carryovers exactly like tiledrqa's run_analysis (engine.py:215-280)
must reproduce the reference's own results (golden fixtures) for every tile
size, and the dependency checks must fire like the reference's.
"""

import numpy as np
import pytest

from fixtures import assert_same, load_cases, result_arrays, settings_obj

pytestmark = pytest.mark.gpu


def _gpu_available():
    try:
        from paper_2402_16853_b200 import _native

        return _native.lib().rqa_device_count() > 0
    except Exception:
        return False


if not _gpu_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_16853_b200 import (CarryoverBuffers, DependencyViolation,  # noqa: E402
                                   LineHistograms, create_recurrence_matrix,
                                   detect_diagonal_lines, detect_vertical_lines, embed,
                                   flush_carryovers, partition, recurrence_block)


def tiled(series, st, tile_size):
    e = embed(series, st.embedding_dimension, st.time_delay)
    n = e.n_vectors
    grid = partition(n, tile_size)
    carry = CarryoverBuffers(n)
    hist = LineHistograms(n)
    for wave in grid.waves():
        for r, c in wave:
            t = create_recurrence_matrix(grid.tile(r, c), e, st)
            hist.recurrence_points += t.count_points()
            detect_diagonal_lines(t, carry, hist)
            detect_vertical_lines(t, carry, hist)
    flush_carryovers(carry, hist)
    return hist.diagonal, hist.vertical, hist.white_vertical, hist.recurrence_points


def test_operator_pipeline_matches_reference_goldens():
    cases = load_cases("small_cases")[::6]
    for series, st, res, meta in cases:
        s = settings_obj(st)
        for ts in (7, 64, 1000):
            assert_same(tiled(series, s, ts), result_arrays(res), f"case {meta['id']} T={ts}")


def test_tile_bits_match_recurrence_block():
    rng = np.random.default_rng(2)
    s = rng.uniform(0, 1, 300)
    from paper_2402_16853_b200 import AnalysisSettings

    st = AnalysisSettings(2, 1, "l2", 0.2, include_main_diagonal=False)
    e = embed(s, 2, 1)
    grid = partition(e.n_vectors, 77)
    t = create_recurrence_matrix(grid.tile(1, 2), e, st)
    want = recurrence_block(e, st, t.row_offset, t.row_offset + t.height, t.col_offset,
                            t.col_offset + t.width)
    assert t.bits.shape[0] == -(-(t.height * t.width) // 8)
    assert np.array_equal(t.matrix(), want)


def test_dependency_violations():
    from paper_2402_16853_b200 import AnalysisSettings

    s = np.random.default_rng(1).uniform(0, 1, 200)
    st = AnalysisSettings(1, 1, "l2", 0.1)
    e = embed(s, 1, 1)
    grid = partition(e.n_vectors, 50)
    carry = CarryoverBuffers(e.n_vectors)
    hist = LineHistograms(e.n_vectors)
    t = create_recurrence_matrix(grid.tile(1, 1), e, st)
    with pytest.raises(DependencyViolation):
        detect_diagonal_lines(t, carry, hist)      # tile (0, 0) not processed
    with pytest.raises(DependencyViolation):
        detect_vertical_lines(t, carry, hist)      # tile (0, 1) not processed
    with pytest.raises(DependencyViolation):
        detect_diagonal_lines(grid.tile(0, 0), carry, hist)  # no bits yet
