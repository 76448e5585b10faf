"""Host-side logic (no GPU): validation, file formats, synthetic generators,
baselines and configuration — the same behaviour the reference tests pin
(/root/reference/pkg/tests/test_{trace,profiles,mapping,baselines,search}.py)."""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_2605_19945_b200 as gem
from _golden import fl, vectors
from paper_2605_19945_b200.trace import TraceStats


# ------------------------------------------------------------------ traces

def test_trace_rejects_invalid():
    with pytest.raises(gem.ValidationError):
        gem.ExpertTrace(np.zeros((2, 2), dtype=np.int64))
    with pytest.raises(gem.ValidationError):
        gem.ExpertTrace(np.array([[1, -1]]))
    with pytest.raises(gem.ValidationError):
        gem.ExpertTrace(np.zeros((0, 3), dtype=np.int64))
    with pytest.raises(gem.ValidationError):
        gem.ExpertTrace(np.array([1, 2, 3]))
    with pytest.raises(gem.ValidationError):
        gem.ExpertTrace(np.array([[1.5, 2.0]]))


def test_trace_is_immutable_and_compares_by_value():
    t = gem.ExpertTrace(np.array([[1, 2]]))
    with pytest.raises(ValueError):
        t.tokens[0, 0] = 5
    assert t == gem.ExpertTrace(np.array([[1, 2]]))
    assert t.num_steps == 1 and t.num_experts == 2 and t.step_total(0) == 3


def test_csv_loading(tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("step,expert,tokens\n0,0,1\n0,1,2\n0,2,3\n0,3,3\n")
    assert gem.load_trace(p).tokens[0].tolist() == [1, 2, 3, 3]
    p.write_text("step,expert,tokens\n1,2,7\n")
    t = gem.load_trace(p)
    assert t.tokens.shape == (2, 3) and t.tokens.sum() == 7
    p.write_text("a,b,c\n0,0,1\n")
    with pytest.raises(gem.ParseError, match="line 1"):
        gem.load_trace(p)
    p.write_text("step,expert,tokens\n0,0,1\n0,1,oops\n")
    with pytest.raises(gem.ParseError, match="line 3"):
        gem.load_trace(p)
    p.write_text("step,expert,tokens\n0,0,-4\n")
    with pytest.raises(gem.ValidationError):
        gem.load_trace(p)
    p.write_text("step,expert,tokens\n0,0,1\n0,0,2\n")
    with pytest.raises(gem.ParseError, match="duplicate"):
        gem.load_trace(p)


def test_json_loading(tmp_path):
    p = tmp_path / "t.json"
    p.write_text('{"num_experts": 2,,}')
    with pytest.raises(gem.ParseError, match="line"):
        gem.load_trace(p)
    p.write_text(json.dumps({"num_experts": 2, "num_steps": 2, "tokens": [[1, 2], [3]]}))
    with pytest.raises(gem.ValidationError):
        gem.load_trace(p)
    p.write_text(json.dumps({"num_experts": 0, "num_steps": 0, "tokens": []}))
    with pytest.raises(gem.ValidationError):
        gem.load_trace(p)


def test_round_trips(tmp_path):
    spec = gem.SyntheticTraceSpec(num_experts=12, num_steps=40, tokens_per_step=777, consistent_experts=(1, 5),
                                  temporal_groups=(gem.TemporalGroup((2, 3)),), rng_seed=99)
    tr = gem.generate_trace(spec)
    gem.save_trace(tr, tmp_path / "r.json")
    assert gem.load_trace(tmp_path / "r.json") == tr
    t2 = gem.ExpertTrace(np.array([[0, 5, 0], [1, 0, 2]]))
    gem.save_trace(t2, tmp_path / "r.csv")
    assert gem.load_trace(tmp_path / "r.csv") == t2


def test_generate_trace_matches_reference_stream():
    spec = gem.SyntheticTraceSpec(num_experts=16, num_steps=40, tokens_per_step=1000, consistent_experts=(2, 5, 15),
                                  temporal_groups=(gem.TemporalGroup((0, 3)), gem.TemporalGroup((10,), 0.3, 2.0)),
                                  rng_seed=4)
    assert gem.generate_trace(spec).tokens.tolist() == vectors()["generate_trace"]


def test_generator_properties():
    single = gem.generate_trace(gem.SyntheticTraceSpec(num_experts=1, num_steps=10, tokens_per_step=64))
    assert np.all(single.tokens == 64)
    spec = gem.SyntheticTraceSpec(num_experts=16, num_steps=50, tokens_per_step=1000, consistent_experts=(2, 5, 15),
                                  temporal_groups=(gem.TemporalGroup((0, 3)), gem.TemporalGroup((10,), 0.3, 2.0)),
                                  rng_seed=4)
    assert np.all(gem.generate_trace(spec).tokens.sum(axis=1) == 1000)
    with pytest.raises(gem.GenerationError):
        gem.generate_trace(gem.SyntheticTraceSpec(num_experts=2, num_steps=200, tokens_per_step=10,
                                                  consistent_experts=(0, 1), consistent_probability=0.5))
    with pytest.raises(gem.ValidationError):
        gem.SyntheticTraceSpec(num_experts=4, num_steps=1, tokens_per_step=8, consistent_experts=(1,),
                               temporal_groups=(gem.TemporalGroup((1, 2)),))
    with pytest.raises(gem.ValidationError):
        gem.SyntheticTraceSpec(num_experts=4, num_steps=1, tokens_per_step=8, consistent_experts=(4,))


# ---------------------------------------------------------------- profiles

def test_curve_validation():
    with pytest.raises(gem.ValidationError):
        gem.CostCurve(np.array([5, 3]), np.array([1.0, 2.0]), 1, 0)
    with pytest.raises(gem.ValidationError):
        gem.CostCurve(np.array([1, 2]), np.array([0.0, 1.0]), 1, 0)
    with pytest.raises(gem.ValidationError):
        gem.CostCurve(np.array([0, 2]), np.array([1.0, 2.0]), 1, 0)
    with pytest.raises(gem.ValidationError, match="dips"):
        gem.CostCurve(np.array([1, 2]), np.array([1.0, 0.8]), 1, 0)
    assert gem.CostCurve(np.array([1, 2]), np.array([1.0, 0.99]), 1, 0).latencies.tolist() == [1.0, 1.0]
    with pytest.raises(gem.ValidationError, match="dense_limit"):
        gem.CostCurve(np.array([64, 128]), np.array([1.0, 2.0]), 64, 100)
    a = gem.CostCurve(np.array([16]), np.array([1.0]), 16, 0)
    b = gem.CostCurve(np.array([32]), np.array([1.0]), 32, 0)
    with pytest.raises(gem.ValidationError, match="tile"):
        gem.VariabilityProfile((a, b))


def test_generate_profile_matches_reference():
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=5, setup="moderate", tile_size=64, max_tokens=8192,
                                                      rng_seed=11))
    want = vectors()["generate_profile"]
    for c, w in zip(p.curves, want):
        assert c.token_counts.tolist() == w["xs"] and c.dense_limit == w["dense"]
        assert np.array_equal(c.latencies, fl(w["ys"]))


def test_setups():
    assert all(c == gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=4)).curves[0]
               for c in gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=4)).curves)
    f = gem.VariabilitySetupSpec(num_gpus=8, setup="moderate", rng_seed=5).resolve_speed_factors()
    assert np.all(f >= 0.88) and np.all(f <= 1.11)
    assert gem.VariabilitySetupSpec(num_gpus=3, setup="high").resolve_speed_factors().tolist() == [0.88, 1.0, 1.0]
    with pytest.raises(gem.ValidationError):
        gem.VariabilitySetupSpec(num_gpus=2, setup="explicit")
    with pytest.raises(gem.ValidationError):
        gem.VariabilitySetupSpec(num_gpus=2, setup="low", speed_factors=(1.0, 1.0))
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=1, setup="low", tile_size=64, max_tokens=10_000))
    assert p.curves[0].num_samples <= 100 and p.curves[0].dense_limit == 32 * 64


def test_profile_io(tmp_path):
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=3, setup="moderate", rng_seed=9, tile_size=32,
                                                      max_tokens=8192))
    gem.save_profile(p, tmp_path / "p.json")
    assert gem.load_profile(tmp_path / "p.json") == p
    payload = json.loads((tmp_path / "p.json").read_text())
    payload["num_gpus"] = 4
    (tmp_path / "p.json").write_text(json.dumps(payload))
    with pytest.raises(gem.ValidationError, match="curves"):
        gem.load_profile(tmp_path / "p.json")


# ---------------------------------------------------- mappings / baselines

def test_mapping_validation_and_io(tmp_path):
    with pytest.raises(gem.ValidationError):
        gem.ExpertMapping(np.array([0, 0, 0, 1]), 2)
    with pytest.raises(gem.ValidationError):
        gem.ExpertMapping(np.array([0, 1, 0]), 2)
    with pytest.raises(gem.ValidationError):
        gem.ExpertMapping(np.array([0, 2]), 2)
    m = gem.ExpertMapping(np.array([1, 0, 0, 1]), 2)
    gem.save_mapping(m, tmp_path / "m.json", policy="linear")
    assert gem.load_mapping(tmp_path / "m.json") == m
    assert m.experts_on(1).tolist() == [0, 3] and m.experts_per_gpu == 2


def test_linear_mapping():
    assert gem.linear_mapping(8, 2).assignment.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    assert gem.linear_mapping(4, 4).assignment.tolist() == [0, 1, 2, 3]
    with pytest.raises(gem.ValidationError):
        gem.linear_mapping(6, 4)


def test_eplb_hand_instance():
    stats = TraceStats(np.array([0.4, 0.3, 0.2, 0.1]), np.ones(4), np.eye(4))
    assert gem.eplb_mapping(stats, 2).assignment.tolist() == [0, 1, 1, 0]
    with pytest.raises(gem.ValidationError):
        gem.eplb_mapping(TraceStats(np.array([0.5, 0.3, 0.2]), np.ones(3), np.eye(3)), 2)


def test_search_config():
    c = gem.SearchConfig()
    assert (c.restarts, c.noise_fraction, c.convergence_threshold, c.seed_with_baselines) == (30, 0.20, 0.001, True)
    assert c.swap_cap(128) == 1280 and gem.SearchConfig(max_swaps_per_restart=5).swap_cap(128) == 5
    for bad in ({"restarts": 0}, {"convergence_threshold": 1.5}, {"rng_seed": -1}, {"noise_fraction": -0.1}):
        with pytest.raises(gem.ValidationError):
            gem.SearchConfig(**bad)


def test_nearest_rank_percentile():
    from paper_2605_19945_b200.mapping import nearest_rank_percentile

    assert nearest_rank_percentile(np.arange(1.0, 11.0), 90) == 9.0
    assert nearest_rank_percentile(np.array([5.0, 4.0, 4.0]), 50) == 4.0
    assert nearest_rank_percentile(np.array([1.0, 2.0, 3.0]), 99) == 3.0


def test_thread_count_validation(monkeypatch):
    from paper_2605_19945_b200.search import _thread_count

    monkeypatch.setenv("GEM_THREADS", "x")
    with pytest.raises(gem.ValidationError):
        _thread_count(None)
    with pytest.raises(gem.ValidationError):
        _thread_count(-1)
    assert _thread_count(3) == 3


def test_backend_selection():
    from paper_2605_19945_b200 import kernels

    assert kernels.get_backend(None).BACKEND == "cuda" and kernels.active_name() == "cuda"
    assert kernels.available_backends() == ("cuda",)
    with pytest.raises(ValueError):
        kernels.get_backend("python")


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without a CUDA device every compute entry point raises instead of degrading."""
    import torch

    from paper_2605_19945_b200 import _device

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    trace = gem.ExpertTrace(np.array([[1, 2], [3, 4]]))
    with pytest.raises(_device.NoDeviceError):
        gem.compute_stats(trace)


def test_product_never_imports_the_oracle():
    import pathlib

    pkg = pathlib.Path(gem.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f


def test_all_layer_jobs_equals_per_layer_jobs():
    """The batched job builder reproduces layer_jobs (the reference's restart
    orders, search.py:134-193) for every layer, including key ties."""
    import importlib

    S = importlib.import_module("paper_2605_19945_b200.search")
    rng = np.random.default_rng(3)
    mu = rng.random((5, 16))
    mu[2, 3] = mu[2, 7]  # exact tie
    mu[4] = 1.0 / 16     # all tied
    for cfg in (gem.SearchConfig(rng_seed=7, restarts=6), gem.SearchConfig(rng_seed=1, restarts=3,
                                                                            seed_with_baselines=False)):
        want = S.concat_batches([S.layer_jobs(mu[l], 4, cfg, l) for l in range(5)])
        got = S.all_layer_jobs(mu, 4, cfg)
        assert np.array_equal(got.order, want.order)
        assert np.array_equal(got.assign, want.assign)
        assert np.array_equal(got.needs_greedy, want.needs_greedy)
        assert np.array_equal(got.run_layer, want.run_layer)
        assert got.provenance == want.provenance
        # the keys shipped for the device sort give the same orders
        dev = S.all_layer_jobs(mu, 4, cfg, device_order=True)
        assert dev.order is None and np.array_equal(dev.assign, want.assign)
        greedy_rows = want.needs_greedy.astype(bool)
        assert np.array_equal(np.argsort(-dev.keys[greedy_rows], axis=1, kind="stable"), want.order[greedy_rows])


def test_eplb_assignments_equals_per_row():
    """The batched LPT (all layers at once) makes the per-layer decisions of
    eplb_assignment (reference baselines.py:24-53), ties included."""
    from paper_2605_19945_b200.baselines import eplb_assignment, eplb_assignments

    rng = np.random.default_rng(5)
    mu = rng.random((12, 32))
    mu[3] = 1.0 / 32                  # all tied
    mu[5, rng.integers(0, 32, 10)] = 0.0  # ties at zero
    mu[7] = np.round(mu[7] * 4) / 4   # few distinct values, equal GPU totals
    for G in (1, 2, 4, 8, 32):
        got = eplb_assignments(mu, G)
        want = np.stack([eplb_assignment(mu[l], G) for l in range(mu.shape[0])])
        assert np.array_equal(got, want)


def test_bench_reference_arm_trace_is_the_benchmark_trace():
    """bench.k9_params (the reference arm's numpy restatement of the planted
    layout, so that arm never imports this package) == ingest.planted_layout
    for every BASELINE config, and the C oracle's layer/token-offset generation
    reproduces the matching slice of the whole trace."""
    import numpy as np

    import bench
    from oracle import oracle
    from paper_2605_19945_b200 import ingest

    for name, (L, N, k, E, B, G, C) in bench.CONFIGS.items():
        planted = {} if E >= 16 else {"consistent": 2, "num_groups": 1}
        spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0,
                                    **planted)
        w, r = ingest.planted_layout(spec)
        bw, br, pc, pb, bm, seed = bench.k9_params(name)
        assert np.array_equal(w, bw) and np.array_equal(r, br), name
        assert (pc, pb, bm, seed) == (ingest._prob_u32(spec.consistent_probability),
                                       ingest._prob_u32(spec.burst_probability), spec.burst_multiplier, spec.seed)
    w, r, pc, pb, bm, seed = bench.k9_params("mixtral")
    whole = oracle.gen_topk(3, 3 * 1024, 2, 1024, 8, w[:3], r[:3], pc, pb, bm, seed)
    part = bench._k9_ids(("mixtral", 2, 1024, 2048))
    assert np.array_equal(whole[2, 1024:3072], part)
