"""Device timeline of the bench's statistics step (torch.profiler / CUPTI):
per-kernel durations and the idle gaps between them, to explain a phase of
bench.py's step_breakdown_ms. Not a bench number.

    python tools/stats_timeline.py [--layers 94] [--steps 4]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2605_19945_b200 import _lib, ingest  # noqa: E402
from paper_2605_19945_b200.trace import DeviceStats, finalize_stats  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=94)
    ap.add_argument("--tokens", type=int, default=1 << 24)
    ap.add_argument("--experts", type=int, default=128)
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    L, N, k, E, B = a.layers, a.tokens, 8, a.experts, 1024
    T = N // B
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
    ids = ingest.generate_topk_ids(spec, dtype=torch.int16)
    hist = torch.empty((L, T, E), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()

    def step():
        ds = DeviceStats.allocate(L, E, T)
        dropped = torch.zeros((L,), dtype=torch.int64, device="cuda")
        _lib.call("gem_topk_hist", ids.data_ptr(), 2, L, N, k, B, E, hist.data_ptr(), ds.colsum.data_ptr(),
                  ds.active.data_ptr(), ds.heavy.data_ptr(), dropped.data_ptr(), st.cuda_stream)
        _lib.call("gem_step_gram", hist.data_ptr(), L, T, E, B * k, ds.gram.data_ptr(), st.cuda_stream)
        out = finalize_stats(ds, with_corr=True)
        cls = ingest.classify_device(ds.colsum, ds.heavy, ds.gram, T)
        return out, cls

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    prev = None
    rows = []
    for e in evs:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = (s - prev) if prev is not None else 0
        rows.append({"name": e.name[:60], "us": round(d, 1), "gap_before_us": round(gap, 1)})
        prev = e.time_range.end
    for r in rows:
        print(json.dumps(r))
    cpu = [e for e in prof.events() if e.device_type.name == "CPU" and e.cpu_time_total > 200]
    cpu.sort(key=lambda e: -e.cpu_time_total)
    for e in cpu[:15]:
        print(json.dumps({"cpu_op": e.name[:60], "us": round(e.cpu_time_total, 1)}))


if __name__ == "__main__":
    main()
