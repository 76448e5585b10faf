"""Small shared helpers."""

from __future__ import annotations

import numpy as np


def readonly(arr: np.ndarray) -> np.ndarray:
    arr.setflags(write=False)
    return arr


def serial_sum(values) -> float:
    """Left-to-right fp64 sum of a few host values (the multi-layer aggregate,
    cli.py:427); every per-step score sum runs on the device."""
    total = 0.0
    for v in values:
        total = total + float(v)
    return total
