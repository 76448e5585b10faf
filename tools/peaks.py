"""Measure the tensor/FP64 peaks the rooflines of K2b (int8 tensor), K5 (fp16
tensor) and the fp64 score chains are quoted against, on this box's B200.

MEASURED_PEAKS.json (driver-written) holds HBM GB/s and dense bf16 TF/s only;
this adds cuBLAS(Lt) int8 (torch._int_mm, s32 accumulate), fp16 and fp64 GEMM
throughput at 8192^3 (best of 10, CUDA events) and writes
profiles/r02_peaks.json. Library GEMMs: a measured ceiling, not a spec sheet.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]


def best_of(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    n = 8192
    out = {"gpu": torch.cuda.get_device_name(0), "n": n, "how": "best of 10 CUDA-event timings of one n^3 GEMM"}
    a8 = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda")
    b8 = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda").t()
    try:
        ms = best_of(lambda: torch._int_mm(a8, b8))
        out["int8_tops"] = 2 * n ** 3 / ms / 1e9
    except Exception as exc:  # pragma: no cover
        out["int8_tops"] = None
        out["int8_error"] = repr(exc)
    for name, dt in (("fp16_tflops", torch.float16), ("bf16_tflops", torch.bfloat16), ("fp64_tflops", torch.float64)):
        m = n if dt != torch.float64 else 4096
        a = torch.randn(m, m, dtype=dt, device="cuda")
        b = torch.randn(m, m, dtype=dt, device="cuda")
        ms = best_of(lambda: a @ b)
        out[name] = 2 * m ** 3 / ms / 1e9
    print(json.dumps(out))
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
