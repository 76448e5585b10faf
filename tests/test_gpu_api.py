"""The reference's public-API behaviour, on the B200 kernels: known-answer
cases and acceptance criteria from /root/reference/pkg/tests (Figure 11,
curve KATs, greedy/refine hand instances, search accounting, c2/c3/c5/c7),
re-stated for this package."""

from __future__ import annotations

import bisect
import itertools
import statistics

import numpy as np
import pytest

from conftest import balanced_assignment, random_counts, staircase_profile, unit_slope_profile

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_19945_b200 as gem  # noqa: E402
from paper_2605_19945_b200 import kernels  # noqa: E402


def bisect_cost(samples, dense_limit, n):
    """Independent scalar curve lookup (the reference suite's evaluator rules)."""
    if n <= 0:
        return 0.0
    xs = [s[0] for s in samples]
    ys = [s[1] for s in samples]
    i = bisect.bisect_left(xs, n)
    if i < len(xs) and xs[i] == n:
        return ys[i]
    if n <= dense_limit:
        return ys[i]
    if i == len(xs):
        (x0, y0) = (0, 0.0) if len(xs) == 1 else (xs[-2], ys[-2])
        x1, y1 = xs[-1], ys[-1]
    elif i == 0:
        x0, y0, x1, y1 = 0, 0.0, xs[0], ys[0]
    else:
        x0, y0, x1, y1 = xs[i - 1], ys[i - 1], xs[i], ys[i]
    return y0 + (y1 - y0) * (n - x0) / (x1 - x0)


def loop_score(tokens, profile, assignment):
    total = 0.0
    for t in range(tokens.shape[0]):
        worst = 0.0
        for g, c in enumerate(profile.curves):
            load = int(tokens[t][np.asarray(assignment) == g].sum())
            v = bisect_cost(list(zip(c.token_counts.tolist(), c.latencies.tolist())), c.dense_limit, load)
            worst = max(worst, v)
        total = total + worst
    return total


def enumerate_optimum(trace, profile):
    E = trace.num_experts
    best = None
    for chosen in itertools.combinations(range(E), E // 2):
        a = [1] * E
        for e in chosen:
            a[e] = 0
        s = loop_score(trace.tokens, profile, a)
        best = s if best is None or s < best else best
    return best


@pytest.fixture
def lockstep(data_dir):
    return (gem.load_trace(data_dir / "lockstep_trace.json"), gem.load_profile(data_dir / "lockstep_profile.json"),
            gem.load_mapping(data_dir / "lockstep_mapping.json"))


def test_figure11_golden(lockstep):
    trace, profile, mapping = lockstep
    assert gem.gpu_loads(trace, mapping, 0).tolist() == [3, 6]
    rep = gem.replay(trace, profile, mapping)
    assert [s.straggler_latency for s in rep.step_costs] == [5.0, 4.0, 4.0]
    assert rep.total_score == 13.0 and gem.score_mapping(trace, profile, mapping) == 13.0
    assert rep.percentiles["p50"] == 4.0 and rep.step_costs[0].straggler_gpu == 1


def test_curve_known_answers():
    c = gem.CostCurve(np.array([64, 128]), np.array([1.0, 1.8]), 64, 128)
    assert (c.cost(0), c.cost(1), c.cost(64), c.cost(65), c.cost(128)) == (0.0, 1.0, 1.0, 1.8, 1.8)
    assert gem.CostCurve(np.array([1024, 2048]), np.array([5.0, 9.0]), 64, 0).cost(1536) == pytest.approx(7.0)
    assert gem.CostCurve(np.array([100, 200]), np.array([1.0, 2.0]), 1, 0).cost(300) == pytest.approx(3.0)
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=4, setup="high", tile_size=64))
    assert p.curves[0].cost(64) == pytest.approx(1 / 0.88, abs=1e-9) and p.curves[1].cost(64) == pytest.approx(1.0)
    e = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=2, setup="explicit", speed_factors=(1.0, 1.25),
                                                      base_latency=0.7, fixed_overhead=0.1, tile_size=32))
    for g, f in enumerate((1.0, 1.25)):
        for n in (1, 31, 32, 33, 200, 1024):
            assert e.curves[g].cost(n) == pytest.approx(0.1 + 0.7 * ((n + 31) // 32) / f, rel=1e-12)


def test_curves_match_scalar_lookup_randomized():
    rng = np.random.default_rng(6)
    for _ in range(40):
        n = int(rng.integers(1, 25))
        xs = np.sort(rng.choice(np.arange(1, 5000), n, replace=False))
        ys = np.cumsum(rng.uniform(0.01, 2.0, n))
        dense = int(rng.choice(np.concatenate(([0], xs))))
        c = gem.CostCurve(xs, ys, 16, dense)
        grid = np.sort(rng.integers(0, 8000, 300))
        got = c.cost_many(grid)
        samples = list(zip(c.token_counts.tolist(), c.latencies.tolist()))
        assert got.tolist() == [bisect_cost(samples, c.dense_limit, int(v)) for v in grid]
        assert np.all(np.diff(got) >= 0.0)
        assert all(c.cost(x) == y for x, y in samples[:3])


def test_staircase_flat_and_equal_latency_load():
    curve = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=1, setup="low", tile_size=64,
                                                          max_tokens=2048)).curves[0]
    v = curve.cost_many(np.arange(1, 2049))
    for k in range(32):
        assert len(set(v[k * 64:(k + 1) * 64].tolist())) == 1
    low = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=2, setup="low", tile_size=64))
    assert gem.equal_latency_load(low.curves[0], low.curves[1], 100) == 128
    pair = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=2, setup="explicit", speed_factors=(1.0, 1.14),
                                                         tile_size=64, max_tokens=8192))
    for n_a in (64, 512, 1024, 4096):
        assert abs(gem.equal_latency_load(pair.curves[0], pair.curves[1], n_a) - 1.14 * n_a) <= 64
    fast = gem.CostCurve(np.array([1, 10]), np.array([0.1, 0.2]), 1, 0)
    slow = gem.CostCurve(np.array([1, 10]), np.array([5.0, 6.0]), 1, 0)
    assert gem.equal_latency_load(fast, slow, 5) == 0


def test_scoring_properties():
    rng = np.random.default_rng(21)
    for _ in range(10):
        tok = random_counts(rng, 10, 6)
        p = staircase_profile(gem, rng, 2)
        a = balanced_assignment(rng, 6, 2)
        assert gem.score_mapping(gem.ExpertTrace(tok), p, gem.ExpertMapping(a, 2)) == loop_score(tok, p, a)
    tr = gem.ExpertTrace(np.array([[4, 4], [1, 1]]))
    assert gem.score_mapping(tr, unit_slope_profile(gem, 1), gem.ExpertMapping(np.array([0, 0]), 1)) == 10.0
    slow = gem.CostCurve(np.array([1, 4096]), np.array([2.0, 8192.0]), 1, 0)
    fast = gem.CostCurve(np.array([1, 4096]), np.array([1.0, 4096.0]), 1, 0)
    prof = gem.VariabilityProfile((slow, fast))
    t2 = gem.ExpertTrace(np.array([[10, 1], [9, 2]]))
    assert gem.score_mapping(t2, prof, gem.ExpertMapping(np.array([0, 1]), 2)) != \
        gem.score_mapping(t2, prof, gem.ExpertMapping(np.array([1, 0]), 2))
    with pytest.raises(gem.DimensionError):
        gem.score_mapping(t2, prof, gem.ExpertMapping(np.array([0, 1, 0, 1]), 2))
    assert gem.gpu_loads(gem.ExpertTrace(np.array([[0, 0], [1, 1]])), gem.ExpertMapping(np.array([0, 1]), 2),
                         0).tolist() == [0, 0]


def test_replay_busy_time_and_totals():
    tr = gem.ExpertTrace(np.array([[2, 3], [4, 5]]))
    rep = gem.replay(tr, unit_slope_profile(gem, 2), gem.ExpertMapping(np.array([0, 1]), 2))
    assert rep.per_gpu_total_tokens == (6, 8) and rep.per_gpu_busy_time == (6.0, 8.0)
    assert rep.mean_step_latency == rep.total_score / 2


def test_compute_stats_known_answers():
    st = gem.compute_stats(gem.ExpertTrace(np.array([[1, 1], [2, 2], [5, 5]])))
    assert st.correlation[0, 0] == 1.0 and st.correlation[0, 1] == pytest.approx(1.0)
    assert gem.compute_stats(gem.ExpertTrace(np.array([[1, 3], [2, 2], [3, 1]]))).correlation[0, 1] == \
        pytest.approx(-1.0)
    z = gem.compute_stats(gem.ExpertTrace(np.array([[2, 1], [2, 5], [2, 3]])))
    assert z.correlation[0, 1] == 0.0 and z.correlation[0, 0] == 1.0
    assert gem.compute_stats(gem.ExpertTrace(np.array([[1, 0], [1, 0], [0, 0], [1, 2]]))).active_fraction.tolist() \
        == [0.75, 0.25]
    rng = np.random.default_rng(11)
    tr = gem.ExpertTrace(rng.integers(0, 20, (25, 4)))
    st = gem.compute_stats(tr)
    for a in range(4):
        for b in range(a + 1, 4):
            want = statistics.correlation(tr.tokens[:, a].tolist(), tr.tokens[:, b].tolist())
            assert st.correlation[a, b] == pytest.approx(want, abs=1e-12)


def test_greedy_and_refine_hand_instances():
    tr = gem.ExpertTrace(np.array([[4, 3, 2, 1]]))
    p = unit_slope_profile(gem, 2)
    m = gem.initial_mapping(gem.compute_stats(tr), 0, tr, p, np.random.default_rng(0))
    assert gem.gpu_loads(tr, m, 0).tolist() == [5, 5]
    tr3 = gem.ExpertTrace(np.array([[4, 3, 2, 1]] * 3))
    start = gem.ExpertMapping(np.array([0, 0, 1, 1]), 2)
    assert gem.score_mapping(tr3, p, start) == 21.0
    refined, swaps = gem.refine(start, tr3, p, gem.SearchConfig())
    assert swaps == 1 and gem.score_mapping(tr3, p, refined) == 15.0
    with pytest.raises(gem.ValidationError):
        gem.initial_mapping(gem.compute_stats(gem.ExpertTrace(np.array([[1, 2, 3]]))), 0,
                            gem.ExpertTrace(np.array([[1, 2, 3]])), p, np.random.default_rng(0))


def test_search_accounting():
    res = gem.search(gem.ExpertTrace(np.full((1, 4), 5)), unit_slope_profile(gem, 2),
                     gem.SearchConfig(restarts=1, rng_seed=0))
    assert res.best_score == 10.0
    rng = np.random.default_rng(24)
    tr = gem.ExpertTrace(random_counts(rng, 10, 8))
    p = staircase_profile(gem, rng, 2)
    res = gem.search(tr, p, gem.SearchConfig(restarts=4, rng_seed=3))
    assert len(res.per_restart) == 6 and res.best_score == min(r.final_score for r in res.per_restart)
    for r in res.per_restart:
        assert r.final_score <= r.initial_score and len(r.trajectory) == r.swap_count + 1
        assert r.trajectory[0] == r.initial_score and r.trajectory[-1] == r.final_score
        assert all(b <= a for a, b in zip(r.trajectory, r.trajectory[1:]))
    nb = gem.search(tr, p, gem.SearchConfig(restarts=3, rng_seed=2, seed_with_baselines=False))
    assert len(nb.per_restart) == 3 and all(r.provenance.startswith("greedy:") for r in nb.per_restart)
    a = gem.search(tr, p, gem.SearchConfig(restarts=6, rng_seed=5), threads=1)
    b = gem.search(tr, p, gem.SearchConfig(restarts=6, rng_seed=5), threads=4)
    assert a.best_score == b.best_score and a.best_mapping == b.best_mapping and a.provenance == b.provenance


def test_c2_enumeration_optimality():
    matched = 0
    for k in range(40):
        rng = np.random.default_rng(1000 + k)
        tr = gem.ExpertTrace(random_counts(rng, 16, 8))
        p = staircase_profile(gem, rng, 2)
        best = enumerate_optimum(tr, p)
        res = gem.search(tr, p, gem.SearchConfig(rng_seed=1000 + k))
        rel = (res.best_score - best) / best
        matched += res.best_score <= best or rel < 1e-12
        assert rel < 0.02
    assert matched >= 38


def test_c3_dominance_and_c5_differential():
    for k in range(10):
        rng = np.random.default_rng(20 + k)
        tr = gem.ExpertTrace(random_counts(rng, 12, 8))
        p = staircase_profile(gem, rng, 4)
        res = gem.search(tr, p, gem.SearchConfig(restarts=3, rng_seed=1))
        assert res.best_score <= gem.score_mapping(tr, p, gem.linear_mapping(8, 4))
        assert res.best_score <= gem.score_mapping(tr, p, gem.eplb_mapping(gem.compute_stats(tr), 4))
    spec = gem.SyntheticTraceSpec(num_experts=16, num_steps=16, tokens_per_step=2048, consistent_experts=(2, 5, 15),
                                  temporal_groups=(gem.TemporalGroup((0, 3)), gem.TemporalGroup((10, 11))))
    tr = gem.generate_trace(spec)
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=4, setup="high", tile_size=64, max_tokens=4096))
    eplb = gem.score_mapping(tr, p, gem.eplb_mapping(gem.compute_stats(tr), 4))
    res = gem.search(tr, p, gem.SearchConfig(rng_seed=0))
    assert (eplb - res.best_score) / eplb >= 0.02


def test_c7_incremental_equals_full_score():
    be = kernels.active()
    rng = np.random.default_rng(7)
    for _ in range(300):
        G = int(rng.integers(2, 5))
        per = int(rng.integers(1, 5))
        E = G * per
        T = int(rng.integers(1, 17))
        tok = random_counts(rng, T, E, high=300)
        p = staircase_profile(gem, rng, G, tile=16, tiles=48)
        a = balanced_assignment(rng, E, G)
        xs = np.concatenate([c.token_counts for c in p.curves])
        ys = np.concatenate([c.latencies for c in p.curves])
        off = np.concatenate(([0], np.cumsum([c.num_samples for c in p.curves]))).astype(np.int64)
        dl = np.asarray([c.dense_limit for c in p.curves], dtype=np.int64)
        loads = np.stack([tok[:, a == g].sum(axis=1) for g in range(G)], axis=1)
        lat = np.stack([be.eval_curve_packed(xs, ys, off, dl, g, loads[:, g]) for g in range(G)], axis=1)
        cross = [(i, j) for i in range(E) for j in range(i + 1, E) if a[i] != a[j]]
        i, j = cross[int(rng.integers(0, len(cross)))]
        inc = be.swap_candidate_score(tok, a, loads, lat, xs, ys, off, dl, i, j)
        sw = a.copy()
        sw[i], sw[j] = sw[j], sw[i]
        assert inc == gem.score_mapping(gem.ExpertTrace(tok), p, gem.ExpertMapping(sw, G))


def test_single_gpu_has_no_swaps():
    be = kernels.active()
    tok = np.array([[1, 2, 3, 4]] * 4, dtype=np.int64)
    p = unit_slope_profile(gem, 1)
    c = p.curves[0]
    a = np.zeros(4, dtype=np.int64)
    loads = tok.sum(axis=1, keepdims=True)
    lat = c.cost_many(loads)
    found, i, j, cand = be.best_swap(tok, a, loads, lat, c.token_counts, c.latencies, np.array([0, 2]),
                                     np.array([0]))
    assert (found, i, j) == (False, -1, -1) and cand == float("inf")
