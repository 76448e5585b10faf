"""K1 variant sweep: every GEM_HIST_CTA mode's histogram/colsum/active/dropped
against the default kernel's (bit-exact) and its CUDA-event time.

    python tools/k1_modes.py --layers 58 --experts 256 --modes 0,6,7
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_19945_b200 import _lib, ingest  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=94)
    ap.add_argument("--tokens", type=int, default=1 << 24)
    ap.add_argument("--experts", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--modes", default="0")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    L, N, k, E, B = a.layers, a.tokens, a.k, a.experts, 1024
    T = N // B
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
    ids = ingest.generate_topk_ids(spec, dtype=torch.int16)
    ids[0, 12345, 3] = E + 5  # one dropped id
    st = torch.cuda.current_stream()
    ref = None
    for m in a.modes.split(","):
        os.environ["GEM_HIST_CTA"] = m
        hist = torch.empty((L, T, E), dtype=torch.int32, device="cuda")
        outs = [torch.zeros((L, E), dtype=torch.int64, device="cuda"), torch.zeros((L, E), dtype=torch.int32, device="cuda"),
                torch.zeros((L, E), dtype=torch.int32, device="cuda"), torch.zeros((L,), dtype=torch.int64, device="cuda")]

        def run():
            for o in outs:
                o.zero_()
            _lib.call("gem_topk_hist", ids.data_ptr(), 2, L, N, k, B, E, hist.data_ptr(), *[o.data_ptr() for o in outs],
                      st.cuda_stream)

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            run()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        res = [hist] + outs
        same = None
        if ref is None:
            ref = [r.clone() for r in res]
        else:
            same = all(torch.equal(x, y) for x, y in zip(ref, res))
        byts = L * N * k * 2 + 2 * L * T * E * 4
        print(json.dumps({"mode": m, "ms": ms, "GBps": byts / ms / 1e6, "equal_to_first": same, "E": E, "L": L}),
              flush=True)


if __name__ == "__main__":
    main()
