"""Python model of the row-stripe decomposition (test infrastructure).

Mirrors what librqa_b200.so reports for one stripe in stripe mode
(include/rqa_b200.h, rqa_run_device mode 1) and what rqa_stitch_device
folds, computed from a full recurrence matrix.  Used by the gloo tests of
the multi-process orchestration (tests/test_distributed.py) where no GPU is
available, and as an executable statement of the stitching rules.
"""

import numpy as np


def runs(seq):
    """[(start, stop, bit)] maximal runs of a 1-D bool array."""
    out = []
    n = len(seq)
    a = 0
    while a < n:
        b = a
        while b < n and seq[b] == seq[a]:
            b += 1
        out.append((a, b, int(seq[a])))
        a = b
    return out


def pack(length, bit):
    return (int(length) << 1) | int(bit)


def stripe_outputs(mat, lo, hi):
    """(hist [3, n+1], points, prefix[n], suffix[n], col[2n], rowpart[2n]) of rows [lo, hi)."""
    n = mat.shape[0]
    hist = np.zeros((3, n + 1), np.int64)
    pre = np.zeros(n, np.int64)
    suf = np.zeros(n, np.int64)
    col = np.zeros(2 * n, np.int64)
    lead = np.zeros(2 * n, np.int64)
    up = np.triu(mat)
    # upper-triangle cells stand for their mirror images; the diagonal once
    points = int(2 * up[lo:hi].sum() - sum(int(mat[i, i]) for i in range(lo, hi)))
    # diagonals k >= 0
    for k in range(n):
        e = min(hi, n - k)
        if lo >= e:
            continue
        seq = np.array([mat[i, i + k] for i in range(lo, e)], bool)
        w = 1 if k == 0 else 2
        p_set = False
        for a, b, bit in runs(seq):
            if not bit:
                continue
            top = a == 0
            bottom = b == len(seq) and e == hi
            if top:
                pre[k] = b - a
                p_set = True
                if bottom:
                    suf[k] = b - a
            elif bottom:
                suf[k] = b - a
            else:
                hist[0, b - a] += w
        if not p_set:
            pre[k] = 0
    # hooks: column part of column c inside the stripe (rows [lo, min(hi, c)))
    for c in range(n):
        e = min(hi, c)
        if lo >= e:
            continue
        rs = runs(mat[lo:e, c])
        if len(rs) == 1:
            col[2 * c] = col[2 * c + 1] = pack(rs[0][1] - rs[0][0], rs[0][2])
        else:
            col[2 * c] = pack(rs[0][1] - rs[0][0], rs[0][2])
            col[2 * c + 1] = pack(rs[-1][1] - rs[-1][0], rs[-1][2])
            for a, b, bit in rs[1:-1]:
                hist[1 if bit else 2, b - a] += 1
    # row parts of the stripe's rows (columns [i, n)): first and last run
    for i in range(lo, hi):
        rs = runs(mat[i, i:])
        lead[2 * i] = pack(rs[0][1] - rs[0][0], rs[0][2])
        lead[2 * i + 1] = pack(rs[-1][1] - rs[-1][0], rs[-1][2])
        for a, b, bit in rs[1:-1]:
            hist[1 if bit else 2, b - a] += 1
    return hist, points, pre, suf, col, lead


def _emit(hist, run):
    length, bit = run >> 1, run & 1
    if length:
        hist[1 if bit else 2, length] += 1


def _combine(a, b, hist):
    """Run-length segments (first, last, uniform); a then b (rqa_runs.cuh seg_combine)."""
    if a is None:
        return b
    if b is None:
        return a
    af, al, au = a
    bf, bl, bu = b
    if (al & 1) == (bf & 1):
        m = pack((al >> 1) + (bf >> 1), al & 1)
        if au and bu:
            return (m, m, True)
        if not au and not bu:
            _emit(hist, m)
        return (m if au else af, m if bu else bl, False)
    if not au:
        _emit(hist, al)
    if not bu:
        _emit(hist, bf)
    return (af, bl, False)


def stitch(pre, suf, col, lead, bounds, n, hist):
    """Final fold over stripes (rqa_fold.cuh unit_fold_stripes)."""
    for k in range(n):
        rows = n - k
        w = 1 if k == 0 else 2
        open_ = 0
        for g in range(len(bounds) - 1):
            lo, hi = bounds[g], bounds[g + 1]
            if lo >= rows:
                break
            if hi <= lo:
                continue
            L = min(hi, rows) - lo
            p = int(pre[g][k])
            if p == L:
                open_ += L
                continue
            if open_ + p > 0:
                hist[0, open_ + p] += w
            open_ = int(suf[g][k]) if hi <= rows else 0
        if open_ > 0:
            hist[0, open_] += w
    for c in range(n):
        acc = None
        for g in range(len(bounds) - 1):
            lo, hi = bounds[g], bounds[g + 1]
            if lo >= c:
                break
            if hi <= lo:
                continue
            L = min(hi, c) - lo
            first, last = int(col[g][2 * c]), int(col[g][2 * c + 1])
            acc = _combine(acc, (first, last, (first >> 1) == L), hist)
        first, last = int(lead[2 * c]), int(lead[2 * c + 1])
        acc = _combine(acc, (first, last, (first >> 1) == n - c), hist)
        _emit(hist, acc[0])
        if not acc[2]:
            _emit(hist, acc[1])
