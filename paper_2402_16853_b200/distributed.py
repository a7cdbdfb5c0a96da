"""Row-stripe decomposition across GPUs (one process per GPU).

Rows of the N x N matrix are split into contiguous stripes, one per rank,
on band boundaries.  Rows never cross stripes, so vertical and white-vertical
lines (row runs, by R = R^T) are complete on each rank; only diagonal lines
cross stripe edges.  Each rank reports, per diagonal k >= 0, the 1-run
starting at its top edge and ending at its bottom edge; rank 0 gathers those
(gather over NCCL / NVLink), folds them in row order with the carry
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
    """Equal-work row stripes aligned to ``band`` rows: world+1 boundaries.

    Only the upper triangle is evaluated, so row i costs n - i cells; the
    boundaries split the triangle's area evenly (i_g = n (1 - sqrt(1 - g/G))),
    rounded to band multiples, monotone.
    """
    import math

    out = [0]
    for g in range(1, world):
        i = n * (1.0 - math.sqrt(1.0 - g / world))
        b = int(round(i / band)) * band
        out.append(max(out[-1], min(n, b)))
    out.append(n)
    return out


def gpu_stripe_fn(series_dev, settings, lo, hi, n, device, precision="fp64"):
    """This rank's stripe on its GPU: (hist [3,n+1], counts [2], StripeOutputs).

    counts = (recurrence points, fp32/fp64 mismatched cells)."""
    import torch

    from .device import MODE_STRIPE, StripeOutputs, run_rows_device

    hist = torch.zeros(3, n + 1, dtype=torch.int64, device=device)
    counts = torch.zeros(2, dtype=torch.int64, device=device)
    so = StripeOutputs.empty(n, device)
    run_rows_device(series_dev, settings, lo, hi, MODE_STRIPE, hist, counts[0:1], so,
                    precision=precision, mismatches=counts[1:2])
    return hist, counts, so


def gpu_stitch_fn(gathered, bounds, n, hist):
    from .device import stitch_device

    stitch_device(gathered, bounds, n, hist)


def _gloo_staged(fn, *tensors):
    """Run a gloo collective on CPU copies of CUDA tensors (test setups only)."""
    host = [t.cpu() for t in tensors]
    fn(*host)
    for t, h in zip(tensors, host):
        t.copy_(h)


def reduce_sum(t, dst=0, group=None):
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl" or not t.is_cuda:
        dist.reduce(t, dst=dst, group=group)
    else:
        _gloo_staged(lambda h: dist.reduce(h, dst=dst, group=group), t)


def all_reduce(t, op=None, group=None):
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if dist.get_backend(group) == "nccl" or not t.is_cuda:
        dist.all_reduce(t, op=op, group=group)
    else:
        _gloo_staged(lambda h: dist.all_reduce(h, op=op, group=group), t)


def exchange(so, world, group=None, dst=0):
    """Gather the stripe edge summaries on rank ``dst`` (the only rank that
    stitches) and sum the row parts there (disjoint rows).  Returns the
    gathered StripeOutputs on ``dst``, None elsewhere."""
    import torch
    import torch.distributed as dist

    from .device import StripeOutputs

    rank = dist.get_rank(group)
    n = so.prefix.numel()
    dev = so.prefix.device
    out = None
    if rank == dst:
        out = StripeOutputs(torch.empty(world, n, dtype=so.prefix.dtype, device=dev),
                            torch.empty(world, n, dtype=so.suffix.dtype, device=dev),
                            torch.empty(world, 2 * n, dtype=so.col.dtype, device=dev),
                            so.rowlead)
    nccl = dist.get_backend(group) == "nccl"
    for name in ("prefix", "suffix", "col"):
        src = getattr(so, name)
        if nccl:
            parts = list(getattr(out, name).unbind(0)) if rank == dst else None
            dist.gather(src, gather_list=parts, dst=dst, group=group)
        else:  # gloo (CPU tests / shared-GPU test runs): host copies
            parts = [torch.empty_like(src, device="cpu") for _ in range(world)] \
                if rank == dst else None
            dist.gather(src.cpu(), gather_list=parts, dst=dst, group=group)
            if rank == dst:
                getattr(out, name).copy_(torch.stack(parts))
    reduce_sum(so.rowlead, dst, group)
    return out


def run_analysis_distributed(embedded: EmbeddedSeries, settings: AnalysisSettings, *,
                             group=None, device=None, band: int | None = None,
                             stripe_fn=None, stitch_fn=None, precision: str = "fp64"):
    """Analysis over all ranks of ``group``; rank 0 returns LineHistograms.

    Other ranks return None.  ``device`` is this rank's torch device (default
    cuda:LOCAL current device).  With precision "fp32" the returned
    histograms carry ``mismatched_cells`` (summed over the ranks).
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = embedded.n_vectors
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if stripe_fn is None:
        def stripe_fn(*a):
            return gpu_stripe_fn(*a, precision=precision)
    if stitch_fn is None:
        stitch_fn = gpu_stitch_fn
    if band is None:
        from .device import band_rows

        band = band_rows(settings, n)
    bounds = stripe_bounds(n, world, band)
    series = torch.from_numpy(np.ascontiguousarray(embedded.values, np.float64)).to(device)
    hist, points, so = stripe_fn(series, settings, bounds[rank], bounds[rank + 1], n, device)
    gathered = exchange(so, world, group)
    reduce_sum(hist, 0, group)
    reduce_sum(points, 0, group)
    if rank != 0:
        return None
    stitch_fn(gathered, bounds, n, hist)
    h = hist.cpu().numpy()
    counts = points.cpu().numpy()
    out = LineHistograms(n, int(counts[0]), h[0].copy(), h[1].copy(), h[2].copy())
    if precision == "fp32":
        out.mismatched_cells = int(counts[1]) if counts.shape[0] > 1 else 0
    return out
