"""Generate golden vectors from the REAL reference (`gemap`, /root/reference).

Run in the build container (where /root/reference exists and
oracle/build_ref.sh has installed the reference into oracle/_ref):

    python tests/golden/make_golden.py

Writes tests/golden/reference_vectors.json (floats as float.hex() so parity
checks are bit-exact) and re-renders the reference's Figure-11 lockstep
fixtures (pkg/tests/data/lockstep_*.json) through the reference's own
load/save functions. Nothing at test time imports the reference: the tests
compare the oracle and the CUDA package against these committed vectors.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = ROOT / "oracle" / "_ref"
sys.path.insert(0, str(REF))
os.environ["GEM_BACKEND"] = "cython"

import gemap  # noqa: E402
from gemap import kernels  # noqa: E402
from gemap.search import _Instance  # noqa: E402

assert kernels.active_name() == "cython", "build the reference with oracle/build_ref.sh first"


def hx(v) -> str:
    return float(v).hex()


def staircase(rng, G, tile=16, tiles=32):
    xs = np.arange(1, tiles + 1, dtype=np.int64) * tile
    return gemap.VariabilityProfile(tuple(
        gemap.CostCurve(xs, np.cumsum(rng.uniform(0.05, 0.5, tiles)), tile, int(xs[-1])) for _ in range(G)))


def mixed(rng, G):
    curves = []
    for _ in range(G):
        n = int(rng.integers(2, 30))
        xs = np.sort(rng.choice(np.arange(1, 3000), n, replace=False)).astype(np.int64)
        ys = np.cumsum(rng.uniform(0.01, 2.0, n))
        dense = int(rng.choice(np.concatenate(([0], xs))))
        curves.append(gemap.CostCurve(xs, ys, 16, dense))
    return gemap.VariabilityProfile(tuple(curves))


def counts(rng, T, E, high=50):
    tok = rng.integers(0, high, (T, E))
    if not tok.any():
        tok[0, 0] = 1
    return tok


def prof_json(p):
    return [{"xs": c.token_counts.tolist(), "ys": [hx(y) for y in c.latencies], "dense": c.dense_limit,
             "tile": c.tile_size} for c in p.curves]


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": "gemap " + gemap.__version__}

    # Figure-11 fixtures, re-rendered by the reference's own I/O
    src = Path("/root/reference/pkg/tests/data")
    gemap.save_mapping(gemap.load_mapping(src / "lockstep_mapping.json"), HERE / "lockstep_mapping.json")
    prof = gemap.load_profile(src / "lockstep_profile.json")
    gemap.save_profile(prof, HERE / "lockstep_profile.json")
    gemap.save_trace(gemap.load_trace(src / "lockstep_trace.json"), HERE / "lockstep_trace.json")

    # curve evaluation
    rng = np.random.default_rng(900)
    cases = []
    for _ in range(40):
        p = mixed(rng, 3)
        ns = rng.integers(-5, 6000, 200)
        cases.append({"profile": prof_json(p), "counts": ns.tolist(),
                      "cost": [[hx(v) for v in c.cost_many(ns)] for c in p.curves]})
    out["curves"] = cases

    # scoring + replay + stats
    rng = np.random.default_rng(901)
    cases = []
    for k in range(40):
        G = int(rng.integers(1, 5))
        E = G * int(rng.integers(1, 5))
        T = int(rng.integers(1, 20))
        tok = counts(rng, T, E, high=int(rng.integers(2, 400)))
        p = staircase(rng, G) if k % 2 else mixed(rng, G)
        a = np.repeat(np.arange(G), E // G)
        rng.shuffle(a)
        tr, m = gemap.ExpertTrace(tok), gemap.ExpertMapping(a, G)
        rep = gemap.replay(tr, p, m)
        st = gemap.compute_stats(tr)
        cases.append({
            "tokens": tok.tolist(), "profile": prof_json(p), "assignment": a.tolist(),
            "score": hx(gemap.score_mapping(tr, p, m)),
            "step_max": [hx(s.straggler_latency) for s in rep.step_costs],
            "straggler": [s.straggler_gpu for s in rep.step_costs],
            "busy": [hx(b) for b in rep.per_gpu_busy_time], "gpu_tokens": list(rep.per_gpu_total_tokens),
            "percentiles": {k2: hx(v) for k2, v in rep.percentiles.items()},
            "mean_utilization": [hx(v) for v in st.mean_utilization],
            "active_fraction": [hx(v) for v in st.active_fraction],
            "correlation": [[hx(v) for v in row] for row in st.correlation],
            "eplb": gemap.eplb_mapping(st, G).assignment.tolist(),
        })
    out["scoring"] = cases

    # backend protocol: best_swap / swap_candidate_score on explicit state
    rng = np.random.default_rng(902)
    be = kernels.get_backend("cython")
    cases = []
    for _ in range(60):
        G = int(rng.integers(1, 5))
        E = G * int(rng.integers(1, 5))
        T = int(rng.integers(1, 12))
        tok = counts(rng, T, E, high=400)
        p = mixed(rng, G)
        a = np.repeat(np.arange(G), E // G).astype(np.int64)
        rng.shuffle(a)
        inst = _Instance(gemap.ExpertTrace(tok), p)
        loads = inst.load_matrix(a)
        lat = inst.latency_matrix(be, loads)
        found, i, j, cand = be.best_swap(inst.tokens, a, loads, lat, *inst.curve_args())
        cross = [(x, y) for x in range(E) for y in range(x + 1, E) if a[x] != a[y]]
        pair = cross[int(rng.integers(0, len(cross)))] if cross else None
        sc = be.swap_candidate_score(inst.tokens, a, loads, lat, *inst.curve_args(), *pair) if pair else None
        cases.append({"tokens": tok.tolist(), "profile": prof_json(p), "assignment": a.tolist(),
                      "best_swap": [bool(found), int(i), int(j), hx(cand)],
                      "pair": list(pair) if pair else None, "pair_score": hx(sc) if pair else None})
    out["protocol"] = cases

    # search: greedy seeds, refine, full search with trajectories
    rng = np.random.default_rng(903)
    cases = []
    for k in range(16):
        G = int(rng.integers(2, 5))
        E = G * int(rng.integers(2, 5))
        T = int(rng.integers(4, 16))
        tok = counts(rng, T, E, high=int(rng.integers(20, 300)))
        p = staircase(rng, G) if k % 2 else mixed(rng, G)
        tr = gemap.ExpertTrace(tok)
        cfg = gemap.SearchConfig(restarts=int(rng.integers(2, 7)), rng_seed=int(rng.integers(0, 1000)))
        res = gemap.search(tr, p, cfg)
        st = gemap.compute_stats(tr)
        init = gemap.initial_mapping(st, 1, tr, p, np.random.default_rng(cfg.rng_seed ^ 1))
        cases.append({
            "tokens": tok.tolist(), "profile": prof_json(p), "restarts": cfg.restarts, "seed": cfg.rng_seed,
            "best_score": hx(res.best_score), "best_assignment": res.best_mapping.assignment.tolist(),
            "provenance": res.provenance,
            "records": [{"provenance": r.provenance, "swaps": r.swap_count,
                         "trajectory": [hx(v) for v in r.trajectory]} for r in res.per_restart],
            "initial_1": init.assignment.tolist(),
        })
    out["search"] = cases

    # synthetic generators (host-side, reference numpy streams)
    spec = gemap.SyntheticTraceSpec(num_experts=16, num_steps=40, tokens_per_step=1000, consistent_experts=(2, 5, 15),
                                    temporal_groups=(gemap.TemporalGroup((0, 3)), gemap.TemporalGroup((10,), 0.3, 2.0)),
                                    rng_seed=4)
    out["generate_trace"] = gemap.generate_trace(spec).tokens.tolist()
    out["generate_profile"] = prof_json(gemap.generate_profile(gemap.VariabilitySetupSpec(
        num_gpus=5, setup="moderate", tile_size=64, max_tokens=8192, rng_seed=11)))

    (HERE / "reference_vectors.json").write_text(json.dumps(out) + "\n")
    print("wrote", HERE / "reference_vectors.json")


if __name__ == "__main__":
    main()
