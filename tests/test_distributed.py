"""Multi-process orchestration of the row-stripe decomposition (gloo, CPU).

The per-stripe compute and the stitch are replaced by the Python model in
tests/stripe_model.py (no GPU here); the collectives, stripe bounds and the
stitching rules are the ones the GPU path uses (distributed.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from stripe_model import stitch, stripe_outputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_stripe_bounds_balance_upper_triangle():
    from paper_2402_16853_b200.distributed import stripe_bounds

    n, band = 1 << 20, 1024
    for g in (1, 2, 4, 8):
        b = stripe_bounds(n, g, band)
        assert b[0] == 0 and b[-1] == n and all(x % band == 0 for x in b[:-1])
        work = [(n - b[i] + n - b[i + 1]) * (b[i + 1] - b[i]) / 2 for i in range(g)]
        assert max(work) / min(work) < 1.01


@pytest.mark.parametrize("world", [1, 2, 3])
def test_model_stripes_match_oracle(oracle_lib, world):
    """The stripe/stitch rules reproduce the reference histograms."""
    from paper_2402_16853_b200.distributed import stripe_bounds

    rng = np.random.default_rng(world)
    for metric, m, tau, r in (("l2", 2, 1, 0.3), ("linf", 3, 2, 0.4), ("l1", 1, 1, 0.05)):
        s = np.sin(np.linspace(0, 12 * np.pi, 160)) + 0.3 * rng.uniform(-1, 1, 160)
        mat = oracle_lib.oracle_matrix(s, m, tau, metric, r)
        n = mat.shape[0]
        bounds = stripe_bounds(n, world, 16)
        hist = np.zeros((3, n + 1), np.int64)
        pts = 0
        outs = []
        for g in range(world):
            h, p, pre, suf, col, lead = stripe_outputs(mat, bounds[g], bounds[g + 1])
            hist += h
            pts += p
            outs.append((pre, suf, col, lead))
        lead = sum(o[3] for o in outs)
        stitch([o[0] for o in outs], [o[1] for o in outs], [o[2] for o in outs], lead, bounds, n,
               hist)
        d, v, w, p = oracle_lib.oracle_histograms(s, m, tau, metric, r, 0, tile_size=32)
        assert pts == p
        assert np.array_equal(hist[0], d) and np.array_equal(hist[1], v)
        assert np.array_equal(hist[2], w)


def _worker(rank, world, port, series, settings_args, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import oracle_matrix
    from paper_2402_16853_b200 import AnalysisSettings, embed
    from paper_2402_16853_b200.device import StripeOutputs
    from paper_2402_16853_b200.distributed import run_analysis_distributed

    st = AnalysisSettings(*settings_args)
    mat = oracle_matrix(series, st.embedding_dimension, st.time_delay, st.metric, st.radius,
                        st.theiler_window)

    def stripe_fn(series_dev, settings, lo, hi, n, device):
        h, p, pre, suf, col, lead = stripe_outputs(mat, lo, hi)
        to = lambda a, dt=torch.int32: torch.from_numpy(a.astype(np.int64)).to(dt)  # noqa: E731
        return (torch.from_numpy(h), torch.tensor([p], dtype=torch.int64),
                StripeOutputs(to(pre), to(suf), to(col, torch.int64), to(lead, torch.int64)))

    def stitch_fn(gathered, bounds, n, hist):
        h = hist.numpy()
        stitch(gathered.prefix.numpy(), gathered.suffix.numpy(), gathered.col.numpy(),
               gathered.rowlead.numpy(), bounds, n, h)

    res = run_analysis_distributed(embed(series, st.embedding_dimension, st.time_delay), st,
                                   device=torch.device("cpu"), band=16, stripe_fn=stripe_fn,
                                   stitch_fn=stitch_fn)
    if rank == 0:
        np.savez(result_path, d=res.diagonal, v=res.vertical, w=res.white_vertical,
                 p=res.recurrence_points)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_matches_oracle(oracle_lib, tmp_path, world):
    rng = np.random.default_rng(7)
    series = np.cumsum(rng.normal(size=150)) * 0.1
    args = (2, 2, "euclidean", 0.25)
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), series, args, out), nprocs=world, join=True)
    r = np.load(out)
    d, v, w, p = oracle_lib.oracle_histograms(series, 2, 2, "l2", 0.25, 0, tile_size=32)
    assert int(r["p"]) == p
    assert np.array_equal(r["d"], d) and np.array_equal(r["v"], v) and np.array_equal(r["w"], w)
