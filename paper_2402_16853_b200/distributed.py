"""Row-stripe decomposition across GPUs (one process per GPU).

Rows of the N x N matrix are split into contiguous stripes, one per rank,
on band boundaries.  Rows never cross stripes, so vertical and white-vertical
lines (row runs, by R = R^T) are complete on each rank; only diagonal lines
cross stripe edges.  Each rank reports, per diagonal k >= 0, the 1-run
starting at its top edge and ending at its bottom edge; rank 0 gathers those
(all_gather over NCCL / NVLink), folds them in row order with the carry
contract of engine.py:287-319 and adds the crossing runs; histograms are
summed with a reduce.  torch.distributed is plumbing; the compute is
librqa_b200.so.

The orchestration takes the per-stripe and stitch steps as callables so
that it can be exercised with the gloo backend on CPU (tests/test_distributed.py).
"""

import numpy as np

from .embedding import EmbeddedSeries
from .histograms import LineHistograms
from .settings import AnalysisSettings

__all__ = ["stripe_bounds", "run_analysis_distributed", "gpu_stripe_fn", "gpu_stitch_fn"]


def stripe_bounds(n: int, world: int, band: int) -> list:
    """Equal-work row stripes aligned to ``band`` rows: world+1 boundaries."""
    nb = -(-n // band)
    out = []
    for r in range(world + 1):
        out.append(min(n, (nb * r // world) * band))
    out[-1] = n
    return out


def gpu_stripe_fn(series_dev, settings, lo, hi, n, device):
    import torch

    from .device import MODE_STRIPE, run_rows_device

    hist = torch.zeros(3, n + 1, dtype=torch.int64, device=device)
    points = torch.zeros(1, dtype=torch.int64, device=device)
    pre = torch.zeros(n, dtype=torch.int32, device=device)
    suf = torch.zeros(n, dtype=torch.int32, device=device)
    run_rows_device(series_dev, settings, lo, hi, MODE_STRIPE, hist, points, pre, suf)
    return hist, points, pre, suf


def gpu_stitch_fn(pre_all, suf_all, bounds, n, hist):
    from .device import stitch_device

    stitch_device(pre_all, suf_all, bounds, n, hist)


def run_analysis_distributed(embedded: EmbeddedSeries, settings: AnalysisSettings, *,
                             group=None, device=None, band: int | None = None,
                             stripe_fn=None, stitch_fn=None):
    """Analysis over all ranks of ``group``; rank 0 returns LineHistograms.

    Other ranks return None.  ``device`` is this rank's torch device (default
    cuda:LOCAL current device).
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = embedded.n_vectors
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if stripe_fn is None:
        stripe_fn = gpu_stripe_fn
    if stitch_fn is None:
        stitch_fn = gpu_stitch_fn
    if band is None:
        from .device import band_rows

        band = band_rows(settings)
    bounds = stripe_bounds(n, world, band)
    series = torch.from_numpy(np.ascontiguousarray(embedded.values, np.float64)).to(device)
    hist, points, pre, suf = stripe_fn(series, settings, bounds[rank], bounds[rank + 1], n, device)
    pre_all = torch.empty(world, n, dtype=pre.dtype, device=device)
    suf_all = torch.empty(world, n, dtype=suf.dtype, device=device)
    dist.all_gather_into_tensor(pre_all, pre, group=group)
    dist.all_gather_into_tensor(suf_all, suf, group=group)
    dist.reduce(hist, dst=0, group=group)
    dist.reduce(points, dst=0, group=group)
    if rank != 0:
        return None
    stitch_fn(pre_all, suf_all, bounds, n, hist)
    h = hist.cpu().numpy()
    return LineHistograms(n, int(points.cpu().item()), h[0].copy(), h[1].copy(), h[2].copy())
