"""Host-side profile of the time-to-mapping search (GPU box): phases + cProfile.

usage: python tools/ttm_profile.py [window_steps]   (default 16)
"""
import cProfile
import importlib
import pstats
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import paper_2605_19945_b200 as gem  # noqa: E402
from paper_2605_19945_b200 import ingest  # noqa: E402

S = importlib.import_module("paper_2605_19945_b200.search")
L, N, k, E, B, G = 94, 1 << 24, 8, 128, 1024, 8
W = int(sys.argv[1]) if len(sys.argv) > 1 else 16
spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
ids = ingest.generate_topk_ids(spec)
st = ingest.trace_statistics(ids, B, E)
prof = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64, max_tokens=B * k,
                                                     rng_seed=0))
cfg = gem.SearchConfig(rng_seed=0)
hist = st.hist.hist[:, :W].contiguous()
del ids


def tic():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    t0 = tic()
    out = S.search_hist(hist, B * k, prof, cfg)
    t1 = tic()
    print(f"search_hist W={W}: {1e3 * (t1 - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
S.search_hist(hist, B * k, prof, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
