"""Kernel microbenchmarks (CUDA events on the launching stream) and ncu drivers.

    python tools/kbench.py hist  [--layers 94] [--reps 10]
    python tools/kbench.py gram  [--layers 94]
    python tools/kbench.py score [--cands 1000]
    python tools/kbench.py swap  [--runs 64] [--steps 16384]

Each prints one JSON line per measurement. Use --reps 1 --warm 1 under ncu.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_19945_b200 import _lib, ingest  # noqa: E402


def timed(fn, reps, warm):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / max(reps, 1)


def bench_hist(args):
    L, N, k, E, B = args.layers, args.tokens, args.k, args.experts, 1024
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
    ids = ingest.generate_topk_ids(spec, dtype=torch.int16 if args.id_bytes == 2 else torch.int32)
    T = N // B
    hist = torch.empty((L, T, E), dtype=torch.int32, device="cuda")
    colsum = torch.zeros((L, E), dtype=torch.int64, device="cuda")
    active = torch.zeros((L, E), dtype=torch.int32, device="cuda")
    heavy = torch.zeros((L, E), dtype=torch.int32, device="cuda")
    dropped = torch.zeros((L,), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.call("gem_topk_hist", ids.data_ptr(), args.id_bytes, L, N, k, B, E, hist.data_ptr(), colsum.data_ptr(),
                  active.data_ptr(), heavy.data_ptr(), dropped.data_ptr(), st)

    ms = timed(run, args.reps, args.warm)
    byts = L * N * k * args.id_bytes + L * T * E * 4
    print(json.dumps({"kernel": "topk_hist", "ms": ms, "GBps": byts / ms / 1e6, "bytes": byts, "L": L, "N": N,
                      "E": E, "k": k}))


def bench_gram(args):
    L, T, E = args.layers, args.tokens // 1024, args.experts
    hist = torch.randint(0, 1024, (L, T, E), dtype=torch.int32, device="cuda")
    gram = torch.zeros((L, E, E), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    macs = L * T * E * E
    for fn in ("gem_step_gram_cc", "gem_step_gram_tc"):
        ms = timed(lambda: _lib.call(fn, hist.data_ptr(), L, T, E, gram.data_ptr(), st), args.reps, args.warm)
        print(json.dumps({"kernel": fn, "ms": ms, "GMACps": macs / ms / 1e6, "hbm_GBps": L * T * E * 4 / ms / 1e6}))


def bench_coselect(args):
    L, N, k, E, B = args.layers, args.tokens, args.k, args.experts, 1024
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
    ids = ingest.generate_topk_ids(spec, dtype=torch.int16 if args.id_bytes == 2 else torch.int32)
    out = torch.zeros((L, E, E), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ops = 2 * L * N * (128 * ((E + 127) // 128)) ** 2  # int8 tensor ops issued (padded one-hot OᵀO)
    for fn in args.paths.split(","):
        ms = timed(lambda: _lib.call(fn, ids.data_ptr(), args.id_bytes, L, N, k, E, out.data_ptr(), st), args.reps,
                   args.warm)
        print(json.dumps({"kernel": fn, "ms": ms, "tokens_per_s": L * N / ms * 1e3, "int8_TOPS": ops / ms / 1e9,
                          "id_GBps": L * N * k * args.id_bytes / ms / 1e6, "L": L, "N": N, "E": E, "k": k}))


def bench_score(args):
    import paper_2605_19945_b200 as gem
    from paper_2605_19945_b200 import mapping as gm

    L, N, k, E, B, G, C = args.layers, args.tokens, args.k, args.experts, 1024, args.gpus, args.cands
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
    h = ingest.ids_to_histograms(ingest.generate_topk_ids(spec), B, E)
    prof = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64,
                                                         max_tokens=B * k, rng_seed=0))
    rng = np.random.default_rng(0)
    base = np.repeat(np.arange(G, dtype=np.int8), E // G)
    cand = torch.from_numpy(np.stack([[rng.permutation(base) for _ in range(L)] for _ in range(C)])).cuda()
    ls = torch.empty((C, L), dtype=torch.float64, device="cuda")
    ms = timed(lambda: gm.score_candidates_device(h.hist, B * k, prof, cand, ls), args.reps, args.warm)
    print(json.dumps({"kernel": "score_batch", "ms": ms, "cands_per_s": C / ms * 1e3,
                      "cand_layer_steps_per_s": C * L * (N // B) / ms * 1e3}))


def bench_swap(args):
    import paper_2605_19945_b200 as gem
    from paper_2605_19945_b200 import _device

    L, N, k, E, B, G, R = 1, args.steps * 1024, args.k, args.experts, 1024, args.gpus, args.runs
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
    h = ingest.ids_to_histograms(ingest.generate_topk_ids(spec), B, E)
    prof = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64,
                                                         max_tokens=B * k, rng_seed=0))
    dc = _device.DeviceCurves.from_profile(prof)
    lut = dc.lut(B * k)
    rng = np.random.default_rng(0)
    base = np.repeat(np.arange(G, dtype=np.int8), E // G)
    assign = torch.from_numpy(np.stack([rng.permutation(base) for _ in range(R)])).cuda()
    T = N // B
    run_layer = torch.zeros(R, dtype=torch.int32, device="cuda")
    found = torch.empty(R, dtype=torch.int32, device="cuda")
    bi, bj = torch.empty_like(found), torch.empty_like(found)
    bc = torch.empty(R, dtype=torch.float64, device="cuda")
    wsb = int(_lib.lib().gem_search_workspace_bytes(R, T, E, G))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.call("gem_best_swap_runs", h.hist.data_ptr(), L, T, E, G, lut.data_ptr(), dc.lut_nmax, R,
                  run_layer.data_ptr(), assign.data_ptr(), found.data_ptr(), bi.data_ptr(), bj.data_ptr(),
                  bc.data_ptr(), ws.data_ptr(), wsb, st)

    ms = timed(run, args.reps, args.warm)
    pairs = E * E * (G - 1) // (2 * G)
    print(json.dumps({"kernel": "best_swap_runs", "ms": ms, "pair_steps_per_s": R * pairs * T / ms * 1e3,
                      "runs": R, "T": T}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=("hist", "gram", "coselect", "score", "swap"))
    ap.add_argument("--paths", default="gem_coselect_tc,gem_coselect_scatter")
    ap.add_argument("--layers", type=int, default=94)
    ap.add_argument("--tokens", type=int, default=1 << 24)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--experts", type=int, default=128)
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--cands", type=int, default=1000)
    ap.add_argument("--runs", type=int, default=64)
    ap.add_argument("--steps", type=int, default=16384)
    ap.add_argument("--id-bytes", type=int, default=2)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--warm", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    {"hist": bench_hist, "gram": bench_gram, "coselect": bench_coselect, "score": bench_score, "swap": bench_swap}[args.what](args)


if __name__ == "__main__":
    main()
