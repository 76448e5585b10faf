import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2605_19945_b200 as gem
import importlib
from paper_2605_19945_b200 import ingest, _device, _lib
S = importlib.import_module("paper_2605_19945_b200.search")
L, N, k, E, B, G = 94, 1 << 24, 8, 128, 1024, 8
spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
ids = ingest.generate_topk_ids(spec)
st = ingest.trace_statistics(ids, B, E)
prof = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64, max_tokens=B*k, rng_seed=0))
cfg = gem.SearchConfig(rng_seed=0)
hist = st.hist.hist
mu = st.mean_utilization.cpu().numpy()
def tic(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(2):
    t0 = tic()
    batches = [S.layer_jobs(mu[l], G, cfg, l) for l in range(L)]
    batch = S.concat_batches(batches)
    t1 = tic()
    res = S.run_search_device(hist, B*k, prof, batch, cfg.convergence_threshold, cfg.swap_cap(E))
    t2 = tic()
    out = S.search_hist(hist, B*k, prof, cfg, mean_util=mu)
    t3 = tic()
    print(f"layer_jobs {1e3*(t1-t0):.1f} ms  run_search_device {1e3*(t2-t1):.1f} ms  search_hist total {1e3*(t3-t2):.1f} ms")
