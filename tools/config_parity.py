"""Whole-pipeline parity per BASELINE config against the reference build (GPU box).

For a config's synthetic router trace (the benchmark's generator) every
selected layer goes through the reference itself (oracle/_ref: compute_stats,
search with the default SearchConfig and seed 0, restarts on every host core)
and through the B200 path (one batched device search of those layers); the
multi-layer aggregate is the serial fp64 sum in layer order (cli.py:427).
usage: python tools/config_parity.py CONFIG [first_layer n_layers]
writes gpurun_out/config_parity_<CONFIG>.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (CONFIGS: the same shapes bench.py measures)
import paper_2605_19945_b200 as gem  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2605_19945_b200 import ingest  # noqa: E402
from paper_2605_19945_b200.search import aggregate_score, search_hist  # noqa: E402

ref = orc.import_reference()
assert ref is not None, "oracle/_ref (the reference build) is required"
name = sys.argv[1]
L, N, k, E, B, G, _ = bench.CONFIGS[name]
l0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nl = int(sys.argv[3]) if len(sys.argv) > 3 else L
cores = len(os.sched_getaffinity(0)) or 1
planted = {} if E >= 16 else {"consistent": 2, "num_groups": 1}
spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0, **planted)
st = ingest.trace_statistics(ingest.generate_topk_ids(spec), B, E)
hist = st.hist.hist[l0:l0 + nl].contiguous()
pspec = dict(num_gpus=G, setup="moderate", tile_size=64, max_tokens=B * k, rng_seed=0)
prof = gem.generate_profile(gem.VariabilitySetupSpec(**pspec))
rprof = ref.generate_profile(ref.VariabilitySetupSpec(**pspec))
cfg = gem.SearchConfig(rng_seed=0)

torch.cuda.synchronize()
t0 = time.perf_counter()
mine = search_hist(hist, B * k, prof, cfg)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0

out = {"config": name, "layers": [l0, l0 + nl], "steps": int(hist.shape[1]), "experts": E, "gpus": G, "per_layer": []}
ok = True
t_ref = 0.0
ref_results = []
for i in range(nl):
    h = hist[i].cpu().numpy().astype(np.int64)
    s0 = time.perf_counter()
    want = ref.search(ref.ExpertTrace(h), rprof, ref.SearchConfig(rng_seed=0), threads=cores)
    t_ref += time.perf_counter() - s0
    ref_results.append(want)
    got = mine[i]
    rs = ref.compute_stats(ref.ExpertTrace(h))
    ms = gem.compute_stats(gem.ExpertTrace(h))
    rec = {"layer": l0 + i,
           "score_bitexact": got.best_score == want.best_score,
           "mapping_equal": got.best_mapping.assignment.tolist() == want.best_mapping.assignment.tolist(),
           "trajectories_equal": [(r.provenance, tuple(r.trajectory)) for r in got.per_restart]
           == [(r.provenance, tuple(r.trajectory)) for r in want.per_restart],
           "stats_bitexact": bool(np.array_equal(rs.mean_utilization, ms.mean_utilization)
                                  and np.array_equal(rs.active_fraction, ms.active_fraction)),
           "corr_maxabs": float(np.max(np.abs(rs.correlation - ms.correlation)))}
    ok = ok and rec["score_bitexact"] and rec["mapping_equal"] and rec["trajectories_equal"] and rec["stats_bitexact"]
    ok = ok and rec["corr_maxabs"] <= 1e-12
    out["per_layer"].append(rec)
agg_ref = 0.0
for w in ref_results:
    agg_ref = agg_ref + w.best_score
out["aggregate_b200"] = aggregate_score(mine)
out["aggregate_reference"] = agg_ref
out["aggregate_bitexact"] = out["aggregate_b200"] == agg_ref
out["reference_search_s"] = round(t_ref, 2)
out["reference_threads"] = cores
out["b200_search_s"] = round(t_gpu, 4)
out["all_equal"] = bool(ok and out["aggregate_bitexact"])
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"config_parity_{name}.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "per_layer"}))
sys.exit(0 if out["all_equal"] else 1)
