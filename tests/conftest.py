"""Shared fixtures. GPU tests are marked `gpu`; everything else runs on CPU."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgemcore.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.build()
    return o


@pytest.fixture
def data_dir() -> Path:
    return GOLDEN


# ---------------------------------------------------------------------------
# instance builders (the same families the reference suite uses,
# /root/reference/pkg/tests/conftest.py:94-122, written for this package)


def unit_slope_profile(gem, num_gpus: int, max_tokens: int = 4096):
    """cost(n) == n on every GPU: two samples, interpolation everywhere."""
    curve = gem.CostCurve.from_pairs([(1, 1.0), (max_tokens, float(max_tokens))], tile_size=1, dense_limit=0)
    return gem.VariabilityProfile(tuple(curve for _ in range(num_gpus)), label="unit-slope")


def staircase_profile(gem, rng, num_gpus: int, tile: int = 16, tiles: int = 32):
    xs = np.arange(1, tiles + 1, dtype=np.int64) * tile
    curves = []
    for _ in range(num_gpus):
        ys = np.cumsum(rng.uniform(0.05, 0.5, tiles))
        curves.append(gem.CostCurve(xs, ys, tile, int(xs[-1])))
    return gem.VariabilityProfile(tuple(curves), label="random-staircase")


def mixed_profile(gem, rng, num_gpus: int):
    """Curves mixing staircase, interpolation and extrapolation regions."""
    curves = []
    for _ in range(num_gpus):
        n = int(rng.integers(2, 30))
        xs = np.sort(rng.choice(np.arange(1, 3000), n, replace=False)).astype(np.int64)
        ys = np.cumsum(rng.uniform(0.01, 2.0, n))
        dense = int(rng.choice(np.concatenate(([0], xs))))
        curves.append(gem.CostCurve(xs, ys, 16, dense))
    return gem.VariabilityProfile(tuple(curves))


def random_counts(rng, steps: int, experts: int, high: int = 50) -> np.ndarray:
    tok = rng.integers(0, high, (steps, experts))
    if not tok.any():
        tok[0, 0] = 1
    return tok


def balanced_assignment(rng, experts: int, gpus: int) -> np.ndarray:
    a = np.repeat(np.arange(gpus, dtype=np.int64), experts // gpus)
    rng.shuffle(a)
    return a
