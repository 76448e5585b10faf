"""Full-size parity at the headline shape (C4: Qwen3-235B, T = 16,384 steps per layer), GPU box.

The reference itself (oracle/_ref, the Cython build of gemap 0.1.0) is run on
the same counts as the B200 path:
  * search: gemap.search of whole layers (default SearchConfig, seed 0,
    restarts in parallel on every host core) vs the device search -- best
    mapping, best score, every restart's provenance and full trajectory;
  * statistics: gemap.compute_stats of a layer vs K1-K3 (utilisation and
    active fraction bit for bit, correlation within 1e-12);
  * scoring: gemap.score_mapping of random balanced candidates vs K5.
usage: python tools/fullsize_parity.py [layers...]   (default 0 47 93)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_19945_b200 as gem  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2605_19945_b200 import ingest  # noqa: E402
from paper_2605_19945_b200 import mapping as gm  # noqa: E402

ref = orc.import_reference()
assert ref is not None, "oracle/_ref (the reference build) is required"
layers = [int(a) for a in sys.argv[1:]] or [0, 47, 93]
L, N, k, E, B, G = 94, 1 << 24, 8, 128, 1024, 8
cores = len(os.sched_getaffinity(0)) or 1
spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0)
ids = ingest.generate_topk_ids(spec)
st = ingest.trace_statistics(ids, B, E)
hist = st.hist.hist
del ids
pspec = dict(num_gpus=G, setup="moderate", tile_size=64, max_tokens=B * k, rng_seed=0)
prof = gem.generate_profile(gem.VariabilitySetupSpec(**pspec))
rprof = ref.generate_profile(ref.VariabilitySetupSpec(**pspec))
out = {"shape": {"layers_checked": layers, "steps": int(hist.shape[1]), "experts": E, "gpus": G}, "layers": []}
ok = True
for l in layers:
    h = hist[l].cpu().numpy().astype(np.int64)
    rec = {"layer": l}
    # statistics
    rs = ref.compute_stats(ref.ExpertTrace(h))
    mine = gem.compute_stats(gem.ExpertTrace(h))
    rec["stats_mean_util_bitexact"] = bool(np.array_equal(rs.mean_utilization, mine.mean_utilization))
    rec["stats_active_bitexact"] = bool(np.array_equal(rs.active_fraction, mine.active_fraction))
    rec["stats_corr_maxabs"] = float(np.max(np.abs(rs.correlation - mine.correlation)))
    # search
    t0 = time.perf_counter()
    want = ref.search(ref.ExpertTrace(h), rprof, ref.SearchConfig(rng_seed=0), threads=cores)
    t_ref = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = gem.search(gem.ExpertTrace(h), prof, gem.SearchConfig(rng_seed=0))
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    rec["search_best_score"] = got.best_score
    rec["search_score_bitexact"] = got.best_score == want.best_score
    rec["search_mapping_equal"] = got.best_mapping.assignment.tolist() == want.best_mapping.assignment.tolist()
    rec["search_provenance_equal"] = got.provenance == want.provenance
    rec["search_trajectories_equal"] = all(
        a.provenance == b.provenance and tuple(a.trajectory) == tuple(b.trajectory)
        for a, b in zip(got.per_restart, want.per_restart)) and len(got.per_restart) == len(want.per_restart)
    rec["search_swaps"] = [r.swap_count for r in got.per_restart]
    rec["reference_search_s"] = round(t_ref, 2)
    rec["reference_threads"] = cores
    rec["b200_search_s"] = round(t_gpu, 4)
    # candidate scoring
    rng = np.random.default_rng(l)
    base = np.repeat(np.arange(G), E // G)
    cands = np.stack([rng.permutation(base) for _ in range(16)])
    cand_d = torch.from_numpy(cands.astype(np.int8)[:, None, :]).cuda()
    _, per_layer = gm.score_candidates_device(hist[l:l + 1].contiguous(), B * k, prof, cand_d)
    dev = per_layer[:, 0].cpu().numpy()
    refs = np.array([ref.score_mapping(ref.ExpertTrace(h), rprof, ref.ExpertMapping(c, G)) for c in cands])
    rec["scores_bitexact"] = bool(np.array_equal(dev, refs))
    rec["scores_checked"] = len(cands)
    for key in ("stats_mean_util_bitexact", "stats_active_bitexact", "search_score_bitexact", "search_mapping_equal",
                "search_provenance_equal", "search_trajectories_equal", "scores_bitexact"):
        ok = ok and bool(rec[key])
    ok = ok and rec["stats_corr_maxabs"] <= 1e-12
    out["layers"].append(rec)
    print(json.dumps(rec), flush=True)
out["all_equal"] = ok
print(json.dumps({"all_equal": ok}))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fullsize_parity.json", "w"), indent=1)
sys.exit(0 if ok else 1)
