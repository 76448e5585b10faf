"""Golden scale studies from the REAL reference (gemap.scale, oracle/_ref).

    python tests/golden/make_scale_golden.py   # in the build container

Writes tests/golden/scale_vectors.json: run_study outputs (expected gaps as
float.hex(), bit-exact) for every distribution kind; tests/test_gpu_api.py
checks the device implementation against them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1] / "oracle" / "_ref"))

import gemap  # noqa: E402

CASES = [
    ("uniform", (0.88, 1.11), (1, 2, 4, 8, 16, 32, 64), 10000, 0),
    ("normal", (1.0, 0.05), (1, 3, 7, 100), 3000, 5),
    ("normal", (0.02, 1.0), (2, 5), 500, 9),  # the positive floor is hit
    ("two_point", (1.0, 0.5, 0.9), (1, 2, 4), 20000, 2),
    ("empirical", (0.9, 1.0, 1.05, 0.97), (1, 2, 8, 9), 777, 31),
]

out = []
for kind, params, sizes, samples, seed in CASES:
    r = gemap.run_study(gemap.ThroughputDistribution(kind, params), sizes, samples, seed)
    out.append({"kind": kind, "params": list(params), "sizes": list(sizes), "samples": samples, "seed": seed,
                "expected_gap": [float(g).hex() for g in r.expected_gap]})
(HERE / "scale_vectors.json").write_text(json.dumps(out, indent=1) + "\n")
print("wrote", len(out), "studies")
