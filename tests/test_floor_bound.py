"""CPU property test of the K5 step-floor bound (score_tc.cu floor_table_kernel /
step_floor_kernel / maxkey epilogue), restated in numpy: with nondecreasing
latency rows, a step whose largest expert count is h has maximum >= v(h) =
min_g lut[g][h], and a GPU whose load is <= s(h) = min_g (last n with
lut[g][n] <= v(h)) has latency <= v(h) -- so skipping such GPUs and starting
the maximum at v(h) leaves every step maximum unchanged (ties included)."""

from __future__ import annotations

import numpy as np
import pytest


def _levels(lut, h):
    v = lut[:, h].min(axis=0)                                   # [T]
    s = np.stack([np.searchsorted(lut[g], v, side="right") - 1 for g in range(lut.shape[0])])  # [G, T]
    return v, s.min(axis=0)


@pytest.mark.parametrize("G,E,tied", [(32, 256, False), (16, 128, False), (8, 64, True), (32, 64, True)])
def test_step_floor_keeps_every_maximum(G, E, tied):
    rng = np.random.default_rng(G * 100 + E + tied)
    T, C = 400, 40
    counts = rng.integers(0, 40, (T, E))
    for t in range(T):  # a few heavy experts per step (the DeepSeek-V3 regime)
        counts[t, rng.choice(E, 3, replace=False)] += rng.integers(200, 900, 3)
    nmax = int(counts.sum(axis=1).max())
    steps = np.cumsum(rng.uniform(0.0, 1.0, (1 if tied else G, nmax + 1)), axis=1)
    steps = np.round(steps, 1)  # plateaus: equal values inside and across rows
    lut = np.repeat(steps, G, axis=0) if tied else steps
    assert (np.diff(lut, axis=1) >= 0).all()
    h = counts.max(axis=1)
    v, lvl = _levels(lut, h)
    for _ in range(C):
        asg = rng.permutation(np.repeat(np.arange(G), E // G))
        loads = np.stack([counts[:, asg == g].sum(axis=1) for g in range(G)])  # [G, T]
        lat = lut[np.arange(G)[:, None], loads]
        exact = lat.max(axis=0)
        assert (v <= exact).all()
        skipped = loads <= lvl[None, :]
        assert (lat[skipped] <= np.broadcast_to(v, lat.shape)[skipped]).all()
        kept = np.where(skipped, -np.inf, lat)
        assert np.array_equal(np.maximum(v, kept.max(axis=0)), exact)
