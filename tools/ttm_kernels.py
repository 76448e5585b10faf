"""Device-time breakdown of one full-trace time-to-mapping search (GPU box).

usage: python tools/ttm_kernels.py [window_steps] [--c5]   (default: the full trace, Qwen3-235B shape;
       --c5: DeepSeek-V3 shape, 58 layers x 256 experts on 32 GPUs)
Prints wall time, summed kernel time and the per-kernel totals (CUPTI via torch.profiler).
"""
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2605_19945_b200 as gem  # noqa: E402
import importlib  # noqa: E402
from paper_2605_19945_b200 import ingest  # noqa: E402
S = importlib.import_module("paper_2605_19945_b200.search")

L, N, k, E, B, G = (58, 1 << 24, 8, 256, 1024, 32) if "--c5" in sys.argv else (94, 1 << 24, 8, 128, 1024, 8)
spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
ids = ingest.generate_topk_ids(spec)
st = ingest.trace_statistics(ids, B, E)
prof = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64, max_tokens=B * k,
                                                     rng_seed=0))
cfg = gem.SearchConfig(rng_seed=0)
W = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else st.hist.hist.shape[1]
hist = st.hist.hist[:, :W].contiguous()
del ids
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.search_hist(hist, B * k, prof, cfg)
    torch.cuda.synchronize()
    print(f"search_hist W={W}: {1e3 * (time.perf_counter() - t0):.1f} ms wall")
with profile(activities=[ProfilerActivity.CUDA]) as p:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.search_hist(hist, B * k, prof, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
rows = [(e.key, e.device_time_total / 1e3, e.count) for e in p.key_averages() if e.device_time_total > 0]
rows.sort(key=lambda r: -r[1])
tot = sum(r[1] for r in rows)
print(f"profiled wall {1e3 * wall:.1f} ms, kernel total {tot:.1f} ms")
for name, ms, n in rows[:25]:
    print(f"{ms:10.2f} ms {n:6d}  {name[:90]}")
if True:  # per-launch device times of the refinement kernels, in launch order
    seq = {}
    for e in p.events():
        if e.device_time_total > 0 and any(s in e.name for s in ("approx_scan5", "exact_pairs", "apply_swap", "best_swap")):
            key = e.name.split("(")[0].split("::")[-1]
            seq.setdefault(key, []).append(round(e.device_time_total / 1e3, 3))
    for key, v in seq.items():
        print(key, v)
