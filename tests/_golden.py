"""Loader for tests/golden/reference_vectors.json (made by make_golden.py from the reference)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

PATH = Path(__file__).resolve().parent / "golden" / "reference_vectors.json"


@lru_cache(maxsize=1)
def vectors() -> dict:
    return json.loads(PATH.read_text())


def f(h: str) -> float:
    return float.fromhex(h)


def fl(hs) -> np.ndarray:
    return np.array([float.fromhex(h) for h in hs], dtype=np.float64)


def curves_args(prof):
    """[(xs, ys, dense)] per GPU from a golden profile entry."""
    return [(np.asarray(c["xs"], dtype=np.int64), fl(c["ys"]), int(c["dense"])) for c in prof]


def profile(gem, prof):
    return gem.VariabilityProfile(tuple(gem.CostCurve(np.asarray(c["xs"], dtype=np.int64), fl(c["ys"]), c["tile"],
                                                      c["dense"]) for c in prof))
