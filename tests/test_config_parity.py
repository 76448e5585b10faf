"""Every BASELINE config shape, whole pipeline, against the REFERENCE BUILD.

For each of the five BASELINE.json configs (bench.CONFIGS: Mixtral, OLMoE,
Qwen3-30B, Qwen3-235B, DeepSeek-V3) a bounded slice of the benchmark's own
synthetic router trace (one layer, a few hundred steps; Mixtral's full 64
steps) goes through

  * the B200 path: K1 ingestion, statistics, the batched device search with
    the default SearchConfig (30 restarts + baseline seeds, seed 0) and the
    batched candidate scorer (gem_score_batch: the tcgen05 path, at
    E = 256 / G = 32 with split key rows and u32 keys; the CUDA-core v1 path
    at E = 8);
  * the reference itself, built from /root/reference into oracle/_ref by
    oracle/build_ref.sh (shipped to the GPU box with the repo snapshot):
    gemap.compute_stats, gemap.search, gemap.score_mapping
    (/root/reference/pkg/src/gemap/trace.py:87-114, search.py:256-312,
    mapping.py:162-166);
  * the C oracle for the candidate scores of every candidate.

Mappings, best scores, every restart's trajectory, utilisation and active
fraction must be identical bit for bit; Pearson within the reference's 1e-12.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import bench  # noqa: E402
import paper_2605_19945_b200 as gem  # noqa: E402
from paper_2605_19945_b200 import ingest  # noqa: E402
from paper_2605_19945_b200.mapping import score_candidates_device  # noqa: E402
from paper_2605_19945_b200.search import search_hist  # noqa: E402

# (config, steps in the slice, layer, candidates scored)
SLICES = [("mixtral", 64, 5, 64), ("olmoe", 384, 3, 48), ("qwen3-30b", 256, 7, 48), ("qwen3-235b", 256, 40, 48),
          ("deepseek-v3", 192, 11, 32)]


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle as orc

    r = orc.import_reference()
    if r is None:
        pytest.skip("oracle/_ref (the reference build) is not present")
    return r


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name,steps,layer,C", SLICES, ids=[s[0] for s in SLICES])
def test_config_slice_matches_reference(oracle, ref, name, steps, layer, C):
    L, N, k, E, B, G, _ = bench.CONFIGS[name]
    planted = {} if E >= 16 else {"consistent": 2, "num_groups": 1}
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0,
                                **planted)
    steps = min(steps, spec.num_steps)
    # the benchmark trace's tokens [0, steps*B), all layers (the generator is token-offset exact)
    ids = ingest.generate_topk_ids(spec, token_offset=0, num_tokens=steps * B)
    st = ingest.trace_statistics(ids[layer:layer + 1].contiguous(), B, E).check()
    hist = st.hist.hist
    h = hist[0].cpu().numpy().astype(np.int64)
    # ingestion against the oracle restatement
    want_h, _ = oracle.topk_hist(ids[layer:layer + 1].cpu().numpy(), B, E)
    assert np.array_equal(h, want_h[0])

    pspec = dict(num_gpus=G, setup="moderate", tile_size=64, max_tokens=B * k, rng_seed=0)
    prof = gem.generate_profile(gem.VariabilitySetupSpec(**pspec))
    rprof = ref.generate_profile(ref.VariabilitySetupSpec(**pspec))
    rtrace = ref.ExpertTrace(h)

    # statistics
    rs = ref.compute_stats(rtrace)
    assert np.array_equal(st.mean_utilization[0].cpu().numpy(), rs.mean_utilization)
    assert np.array_equal(st.active_fraction[0].cpu().numpy(), rs.active_fraction)
    assert np.allclose(st.correlation[0].cpu().numpy(), rs.correlation, rtol=0, atol=1e-12)

    # search: default config, seed 0 (the CLI's per-layer call)
    mine = search_hist(hist, B * k, prof, gem.SearchConfig(rng_seed=0))[0]
    cores = len(os.sched_getaffinity(0)) or 1
    want = ref.search(rtrace, rprof, ref.SearchConfig(rng_seed=0), threads=cores)
    assert mine.best_score == want.best_score
    assert mine.best_mapping.assignment.tolist() == want.best_mapping.assignment.tolist()
    assert mine.provenance == want.provenance
    assert [(r.provenance, tuple(r.trajectory), r.swap_count, r.final_score) for r in mine.per_restart] == \
        [(r.provenance, tuple(r.trajectory), r.swap_count, r.final_score) for r in want.per_restart]

    # candidate scores: balanced random mappings (the bench's candidate family)
    rng = np.random.default_rng(C + E)
    cand = np.stack([rng.permutation(np.repeat(np.arange(G), E // G)) for _ in range(C)])
    total, per_layer = score_candidates_device(hist, B * k, prof, torch.from_numpy(cand[:, None, :].astype(np.int8))
                                               .cuda())
    got = per_layer[:, 0].cpu().numpy()
    assert np.array_equal(total.cpu().numpy(), got)
    cv = oracle.Curves.from_profile(prof)
    for c in range(C):
        assert got[c] == oracle.score(h, cand[c], cv), c
    for c in range(0, C, max(1, C // 8)):  # the reference's own score_mapping on a sample
        assert got[c] == ref.score_mapping(rtrace, rprof, ref.ExpertMapping(cand[c], G)), c
