"""CUDA kernels vs the CPU oracle and the reference golden vectors (bit-exact
for every integer and every score; Pearson within 1e-12 absolute)."""

from __future__ import annotations

import numpy as np
import pytest

from _golden import curves_args, f, fl, profile as golden_profile, vectors
from conftest import balanced_assignment, mixed_profile, random_counts, staircase_profile

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_19945_b200 as gem  # noqa: E402
from paper_2605_19945_b200 import ingest, kernels  # noqa: E402


# --------------------------------------------------------------------- curves

def test_curve_eval_golden():
    be = kernels.active()
    for case in vectors()["curves"]:
        p = golden_profile(gem, case["profile"])
        ns = np.asarray(case["counts"], dtype=np.int64)
        for g, want in enumerate(case["cost"]):
            assert np.array_equal(p.curves[g].cost_many(ns), fl(want))
            xs = np.concatenate([c.token_counts for c in p.curves])
            ys = np.concatenate([c.latencies for c in p.curves])
            off = np.concatenate(([0], np.cumsum([c.num_samples for c in p.curves]))).astype(np.int64)
            dl = np.asarray([c.dense_limit for c in p.curves], dtype=np.int64)
            assert np.array_equal(be.eval_curve_packed(xs, ys, off, dl, g, ns), fl(want))


# -------------------------------------------------------------- ingestion (K1)

@pytest.mark.parametrize("dtype", [torch.int16, torch.int32])
@pytest.mark.parametrize("shape", [(3, 5000, 8, 256, 64), (2, 1000, 2, 100, 7), (1, 777, 3, 50, 300),
                                   (2, 40000, 8, 9000, 16)])
def test_topk_hist_random_ids(oracle, dtype, shape):
    L, N, k, B, E = shape
    rng = np.random.default_rng(sum(shape))
    ids = rng.integers(-2, E + 2, (L, N, k)).astype(np.int16 if dtype == torch.int16 else np.int32)
    h = ingest.ids_to_histograms(torch.from_numpy(ids).cuda(), B, E, check_dropped=False)
    want, dropped = oracle.topk_hist(ids, B, E)
    assert np.array_equal(h.hist.cpu().numpy(), want)
    assert np.array_equal(h.dropped.cpu().numpy(), dropped)
    assert np.array_equal(h.colsum.cpu().numpy(), want.sum(axis=1))
    assert np.array_equal(h.active.cpu().numpy(), (want > 0).sum(axis=1))
    assert np.array_equal(h.heavy.cpu().numpy(), np.stack([oracle.heavy_counts(w) for w in want]))


@pytest.mark.parametrize("shape", [(2, 64 * 1024, 8, 1024, 128), (1, 37 * 512, 8, 512, 100), (3, 33 * 256, 4, 256, 64),
                                   (1, 40 * 1024, 8, 1024, 8), (1, 40 * 512, 8, 512, 160), (2, 33 * 1024, 8, 1024, 256),
                                   (1, 20 * 1024, 8, 1024, 300), (1, 20 * 1024, 8, 1024, 301)])
def test_topk_hist_ring_path(oracle, shape):
    """The cp.async-ring K1 (int16, whole 2 KB batches per step, N a multiple of
    B; wide counters to E = 160, packed for even E): full and partial 32-step
    units, odd E, out-of-range ids (E = 301 takes the register-buffered kernel)."""
    L, N, k, B, E = shape
    rng = np.random.default_rng(sum(shape))
    ids = rng.integers(-3, E + 3, (L, N, k)).astype(np.int16)
    h = ingest.ids_to_histograms(torch.from_numpy(ids).cuda(), B, E, check_dropped=False)
    want, dropped = oracle.topk_hist(ids, B, E)
    assert np.array_equal(h.hist.cpu().numpy(), want)
    assert np.array_equal(h.dropped.cpu().numpy(), dropped)
    assert np.array_equal(h.colsum.cpu().numpy(), want.sum(axis=1))
    assert np.array_equal(h.active.cpu().numpy(), (want > 0).sum(axis=1))
    assert np.array_equal(h.heavy.cpu().numpy(), np.stack([oracle.heavy_counts(w) for w in want]))


@pytest.mark.parametrize("mode", ["1", "0"])
@pytest.mark.parametrize("shape", [(2, 64 * 1024, 8, 1024, 128), (1, 37 * 512, 8, 512, 100), (3, 33 * 1024, 8, 1024, 256),
                                   (1, 45 * 512, 8, 512, 200), (2, 40 * 256, 8, 256, 64), (1, 35 * 1024, 8, 1024, 250),
                                   (3, 9 * 1024, 8, 1024, 256)])
def test_topk_hist_cta_path(oracle, monkeypatch, shape, mode):
    """The CTA-shared-counter K1 (W warps share lane-private u32 counters, ids
    loaded straight into registers 3 steps ahead, two named barriers per
    step): forced on (mode 1, also E <= 128) and off (mode 0: the ring
    kernels) give the oracle's counts -- W = 8 (8 batches per step), W = 4 and
    W = 2 with 2 rows per lane (4 / 2 batches per step), partial 32-step
    units, units spanning layers, out-of-range ids."""
    monkeypatch.setenv("GEM_HIST_CTA", mode)
    L, N, k, B, E = shape
    rng = np.random.default_rng(sum(shape) + 1)
    ids = rng.integers(-3, E + 3, (L, N, k)).astype(np.int16)
    h = ingest.ids_to_histograms(torch.from_numpy(ids).cuda(), B, E, check_dropped=False)
    want, dropped = oracle.topk_hist(ids, B, E)
    assert np.array_equal(h.hist.cpu().numpy(), want)
    assert np.array_equal(h.dropped.cpu().numpy(), dropped)
    assert np.array_equal(h.colsum.cpu().numpy(), want.sum(axis=1))
    assert np.array_equal(h.active.cpu().numpy(), (want > 0).sum(axis=1))
    assert np.array_equal(h.heavy.cpu().numpy(), np.stack([oracle.heavy_counts(w) for w in want]))


@pytest.mark.parametrize("E", [128, 256])
def test_topk_hist_ring_heavy_with_sparse_drops(oracle, E):
    """Heavy-step counts on the ring path: steps are full, so the row total is
    B*k except in units that dropped ids, which recount from their rows."""
    L, N, k, B = 2, 96 * 1024, 8, 1024
    rng = np.random.default_rng(E)
    ids = rng.integers(0, E, (L, N, k)).astype(np.int16)
    ids[0, 5 * 1024 + 7, 3] = E + 4        # one dropped id in unit 0 of layer 0
    ids[1, 70 * 1024:70 * 1024 + 900, :] = np.int16(-1)  # a step that lost most of its ids (unit 2 of layer 1)
    h = ingest.ids_to_histograms(torch.from_numpy(ids).cuda(), B, E, check_dropped=False)
    want, dropped = oracle.topk_hist(ids, B, E)
    assert np.array_equal(h.hist.cpu().numpy(), want)
    assert np.array_equal(h.dropped.cpu().numpy(), dropped)
    assert np.array_equal(h.heavy.cpu().numpy(), np.stack([oracle.heavy_counts(w) for w in want]))


def test_topk_hist_unaligned_view(oracle):
    rng = np.random.default_rng(9)
    base = rng.integers(0, 32, (1, 4097, 3)).astype(np.int16)
    ids = torch.from_numpy(base).cuda()[:, 1:, :].contiguous()
    h = ingest.ids_to_histograms(ids, 64, 32)
    want, _ = oracle.topk_hist(base[:, 1:, :].copy(), 64, 32)
    assert np.array_equal(h.hist.cpu().numpy(), want)


def test_dropped_ids_raise():
    ids = torch.tensor([[[0, 1], [5, 2]]], dtype=torch.int16).cuda()
    with pytest.raises(gem.ValidationError):
        ingest.ids_to_histograms(ids, 2, 4)


@pytest.mark.parametrize("dtype", [torch.int16, torch.int32])
def test_generator_matches_oracle(oracle, dtype):
    spec = ingest.TopkTraceSpec(num_layers=3, num_tokens=5000, top_k=4, num_experts=24, tokens_per_step=300, seed=11)
    ids = ingest.generate_topk_ids(spec, dtype=dtype)
    w, r = ingest.planted_layout(spec)
    want = oracle.gen_topk(3, 5000, 4, 300, 24, w, r, ingest._prob_u32(0.85), ingest._prob_u32(0.17), 3, 11,
                           id_bytes=2 if dtype == torch.int16 else 4)
    assert np.array_equal(ids.cpu().numpy(), want)
    part = ingest.generate_topk_ids(spec, dtype=dtype, token_offset=1234, num_tokens=2000)
    assert np.array_equal(part.cpu().numpy(), want[:, 1234:3234])


# ------------------------------------------------------- statistics (K2, K3)

def test_stats_and_classes_match_oracle(oracle):
    spec = ingest.TopkTraceSpec(num_layers=3, num_tokens=200 * 512, top_k=8, num_experts=64, tokens_per_step=512,
                                seed=5)
    ids = ingest.generate_topk_ids(spec)
    st = ingest.trace_statistics(ids, 512, 64)
    hist = st.hist.hist.cpu().numpy().astype(np.int64)
    for l in range(3):
        mu, af, corr = oracle.stats(hist[l])
        assert np.array_equal(st.mean_utilization[l].cpu().numpy(), mu)
        assert np.array_equal(st.active_fraction[l].cpu().numpy(), af)
        c = st.correlation[l].cpu().numpy()
        assert np.allclose(c, corr, rtol=0, atol=1e-12)
        assert np.array_equal(c, c.T)
        g = st.gram[l].cpu().numpy()
        want_g = oracle.gram(hist[l])
        iu = np.triu_indices(64)
        assert np.array_equal(g[iu], want_g[iu])
        cls, grp = oracle.classify(hist[l])
        assert np.array_equal(st.classes.cls[l].cpu().numpy(), cls)
        assert np.array_equal(st.classes.group[l].cpu().numpy(), grp)


def _gram_np(h: np.ndarray) -> np.ndarray:
    """exact int64 X^T X (object arithmetic is not needed: |entries| < 2^62 here)."""
    h = h.astype(np.int64)
    return h.T @ h


@pytest.mark.parametrize("shape", [(2, 300, 128, 1024), (1, 16384 + 77, 128, 65535), (3, 1000, 256, 4096),
                                   (1, 129, 256, 65535), (2, 40000, 128, 2048)])
def test_step_gram_tensor_cores_vs_cuda_cores(shape):
    """K2: tcgen05 kind::i8 limb kernel == CUDA-core kernel == exact numpy, bit for bit
    (ragged T, T > one 16384-step s32 segment, counts up to the 65535 limb limit, E=256 off-diagonal blocks)."""
    from paper_2605_19945_b200 import _lib

    L, T, E, hi = shape
    rng = np.random.default_rng(T + E)
    h = rng.integers(0, hi + 1, (L, T, E)).astype(np.int32)
    h[:, ::7, :] = 0
    h[0, 0, :] = hi
    hd = torch.from_numpy(h).cuda()
    st = torch.cuda.current_stream().cuda_stream
    g_tc = torch.zeros((L, E, E), dtype=torch.int64, device="cuda")
    g_cc = torch.zeros((L, E, E), dtype=torch.int64, device="cuda")
    _lib.call("gem_step_gram_tc", hd.data_ptr(), L, T, E, g_tc.data_ptr(), st)
    _lib.call("gem_step_gram_cc", hd.data_ptr(), L, T, E, g_cc.data_ptr(), st)
    assert _lib.lib().gem_step_gram_path(E, hi) == 1
    iu = np.triu_indices(E)
    a, b = g_tc.cpu().numpy(), g_cc.cpu().numpy()
    for l in range(L):
        want = _gram_np(h[l])
        assert np.array_equal(a[l][iu], want[iu])
        assert np.array_equal(b[l][iu], want[iu])


def test_step_gram_accumulates_and_dispatches():
    from paper_2605_19945_b200 import _lib

    rng = np.random.default_rng(1)
    h = torch.from_numpy(rng.integers(0, 100, (1, 500, 128)).astype(np.int32)).cuda()
    g = ingest.step_coactivation(h, max_count=100)
    g = ingest.step_coactivation(h, gram=g, max_count=100)  # accumulates
    want = 2 * _gram_np(h[0].cpu().numpy())
    iu = np.triu_indices(128)
    assert np.array_equal(g[0].cpu().numpy()[iu], want[iu])
    assert _lib.lib().gem_step_gram_path(128, -1) == 0
    assert _lib.lib().gem_step_gram_path(128, 65536) == 0
    assert _lib.lib().gem_step_gram_path(64, 100) == 0
    assert _lib.lib().gem_step_gram_path(256, 8192) == 1


@pytest.mark.parametrize("E,steps", [(128, 400), (256, 300), (64, 400)])
def test_planted_groups_recovered(oracle, E, steps):
    """Recall AND precision of the classifier on the benchmark generator:
    temporal == exactly the planted groups (one group each, lowest-index
    label); every planted consistent expert is consistent; every expert called
    consistent is genuinely heavy (>= its fair share 1/E of the routed ids) and
    heavy in >= 80% of steps; light background experts are CLASS_OTHER."""
    spec = ingest.TopkTraceSpec(num_layers=2, num_tokens=steps * 1024, top_k=8, num_experts=E, seed=3)
    st = ingest.trace_statistics(ingest.generate_topk_ids(spec), 1024, E)
    _, role = ingest.planted_layout(spec)
    hist = st.hist.hist.cpu().numpy().astype(np.int64)
    for l in range(2):
        cls = st.classes.cls[l].cpu().numpy()
        grp = st.classes.group[l].cpu().numpy()
        want_cls, want_grp = oracle.classify(hist[l])
        assert np.array_equal(cls, want_cls) and np.array_equal(grp, want_grp)
        planted_t = set(np.flatnonzero(role[l] >= 2).tolist())
        assert set(np.flatnonzero(cls == ingest.CLASS_TEMPORAL).tolist()) == planted_t
        for g in range(spec.num_groups):
            members = np.flatnonzero(role[l] == 2 + g)
            assert len({int(grp[m]) for m in members}) == 1 and grp[members[0]] == members.min()
        for e in np.flatnonzero(role[l] == 1):
            assert cls[e] == ingest.CLASS_CONSISTENT
        mu = st.mean_utilization[l].cpu().numpy()
        heavy = st.hist.heavy[l].cpu().numpy()
        cons = np.flatnonzero(cls == ingest.CLASS_CONSISTENT)
        assert (mu[cons] * E >= 0.9).all() and (heavy[cons] * 5 >= 4 * steps).all()
        light = np.flatnonzero((role[l] == 0) & (mu * E < 0.5))
        assert len(light) > E // 4 and (cls[light] == ingest.CLASS_OTHER).all()
        assert len(cons) < E // 4  # not the round-1 degenerate "almost everyone is consistent"


def test_device_stats_heavy_from_counts(oracle):
    """gem_hist_colstats (the ExpertTrace path) produces the same active/heavy counts as K1 / the oracle."""
    from paper_2605_19945_b200.trace import device_stats

    rng = np.random.default_rng(4)
    h = rng.integers(0, 40, (3, 700, 37)).astype(np.int32)
    h[:, ::5, :] = 0       # empty steps are heavy for nobody
    h[1, 3, :] = 0
    h[1, 3, 7] = 9
    ds = device_stats(torch.from_numpy(h).cuda(), with_gram=False)
    for l in range(3):
        cs, ac, hv = oracle.colstats3(h[l].astype(np.int64))
        assert np.array_equal(ds.colsum[l].cpu().numpy(), cs)
        assert np.array_equal(ds.active[l].cpu().numpy(), ac)
        assert np.array_equal(ds.heavy[l].cpu().numpy(), hv)


def test_compute_stats_golden():
    for case in vectors()["scoring"]:
        tr = gem.ExpertTrace(np.asarray(case["tokens"], dtype=np.int64))
        st = gem.compute_stats(tr)
        assert np.array_equal(st.mean_utilization, fl(case["mean_utilization"]))
        assert np.array_equal(st.active_fraction, fl(case["active_fraction"]))
        want = np.array([fl(r) for r in case["correlation"]])
        assert np.allclose(st.correlation, want, rtol=0, atol=1e-12)
        assert np.array_equal(st.correlation, st.correlation.T)
        assert gem.eplb_mapping(st, len(case["profile"])).assignment.tolist() == case["eplb"]


# ------------------------------------------------------------ scoring (K4, K5)

def test_score_and_replay_golden():
    for case in vectors()["scoring"]:
        tr = gem.ExpertTrace(np.asarray(case["tokens"], dtype=np.int64))
        p = golden_profile(gem, case["profile"])
        m = gem.ExpertMapping(np.asarray(case["assignment"]), p.num_gpus)
        assert gem.score_mapping(tr, p, m) == f(case["score"])
        rep = gem.replay(tr, p, m)
        assert [s.straggler_latency for s in rep.step_costs] == list(fl(case["step_max"]))
        assert [s.straggler_gpu for s in rep.step_costs] == case["straggler"]
        assert list(rep.per_gpu_busy_time) == list(fl(case["busy"]))
        assert list(rep.per_gpu_total_tokens) == case["gpu_tokens"]
        assert rep.total_score == f(case["score"])
        assert {k: f(v) for k, v in case["percentiles"].items()} == rep.percentiles


def test_score_candidates_batch_matches_oracle(oracle):
    from paper_2605_19945_b200 import mapping as gm
    from paper_2605_19945_b200 import _device

    rng = np.random.default_rng(77)
    L, T, E, G, C = 3, 50, 32, 4, 300
    tok = np.stack([random_counts(rng, T, E, high=200) for _ in range(L)])
    p = staircase_profile(gem, rng, G, tile=64, tiles=128)
    cand = np.stack([[balanced_assignment(rng, E, G) for _ in range(L)] for _ in range(C)])
    hist, nmax = _device.counts_to_device_int32(tok)
    total, per_layer = gm.score_candidates_device(hist, nmax, p, torch.from_numpy(cand.astype(np.int8)).cuda())
    total, per_layer = total.cpu().numpy(), per_layer.cpu().numpy()
    cv = oracle.Curves.from_profile(p)
    for c in range(0, C, 7):
        want_l = [oracle.score(tok[l], cand[c, l], cv) for l in range(L)]
        assert per_layer[c].tolist() == want_l
        s = 0.0
        for v in want_l:
            s = s + v
        assert total[c] == s


@pytest.mark.parametrize("L,T,E,G,C,high,balanced", [(2, 300, 128, 8, 100, 120, True), (3, 129, 64, 8, 70, 400, True),
                                                      (1, 1000, 128, 4, 33, 60, True), (2, 77, 64, 16, 40, 300, True),
                                                      (2, 200, 128, 8, 45, 90, False), (1, 64, 128, 1, 5, 50, True),
                                                      (2, 90, 128, 32, 20, 500, True), (1, 130, 64, 32, 9, 700, True),
                                                      (2, 150, 256, 32, 21, 60, True), (1, 260, 256, 8, 40, 40, True),
                                                      (2, 131, 256, 32, 13, 400, False)])
@pytest.mark.parametrize("split,key32", [(False, False), (True, False), (False, True), (True, True)])
def test_score_batch_tensor_cores_vs_cuda_cores(oracle, monkeypatch, L, T, E, G, C, high, balanced, split, key32):
    """K5 (tcgen05 kind::i8 one-hot loads + exact order keys) == K5 v1 == oracle, bit for bit:
    ragged T and candidate tiles, G = 4/8/16/32, E = 64/128/256 (E = 256: two K
    parts through one A buffer), unbalanced candidate tables; split=True keeps
    only a quarter of every key row in shared memory (the rest is gathered
    from the global table, the DeepSeek-V3 path); G = 1 is declined by the
    tensor-core path (the caller runs v1); key32=True forces the u32 order
    keys (used when the window holds more than 65,536 distinct latencies;
    declined for G = 4 and E = 64/G = 8, where u32 staging does not fit)."""
    from paper_2605_19945_b200 import _device, _lib

    if split:
        monkeypatch.setenv("GEM_SCORE_SPLIT", "1")
    if key32:
        monkeypatch.setenv("GEM_SCORE_KEY32", "1")
    rng = np.random.default_rng(L * 1000 + T + E + G)
    tok = np.stack([random_counts(rng, T, E, high=high) for _ in range(L)])
    p = mixed_profile(gem, rng, G) if G > 1 else staircase_profile(gem, rng, 1, tile=64, tiles=256)
    if balanced:
        cand = np.stack([[balanced_assignment(rng, E, G) for _ in range(L)] for _ in range(C)])
    else:
        cand = rng.integers(0, G, (C, L, E))
    hist, nmax = _device.counts_to_device_int32(tok)
    dc = _device.DeviceCurves.from_profile(p)
    lut = dc.lut(nmax)
    cd = torch.from_numpy(cand.astype(np.int8)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    out = {}
    for fn in ("gem_score_batch_tc", "gem_score_batch_v1"):
        ls = torch.zeros((C, L), dtype=torch.float64, device="cuda")
        err = torch.zeros((1,), dtype=torch.int32, device="cuda")
        rc = getattr(_lib.lib(), fn)(hist.data_ptr(), L, T, E, G, cd.data_ptr(), C, lut.data_ptr(), dc.lut_nmax,
                                     ls.data_ptr(), err.data_ptr(), st)
        if fn == "gem_score_batch_tc" and (G not in (4, 8, 16, 32) or (key32 and (G == 4 or (G == 8 and E == 64)))):
            assert rc == 1
            continue
        assert rc == 0, (fn, rc, _lib.lib().gem_last_error())
        assert int(err.item()) == 0
        out[fn] = ls.cpu().numpy()
    cv = oracle.Curves.from_profile(p)
    if "gem_score_batch_tc" not in out:
        for c in range(0, C, 11):
            assert out["gem_score_batch_v1"][c].tolist() == [oracle.score(tok[l], cand[c, l], cv) for l in range(L)]
        return
    assert np.array_equal(out["gem_score_batch_tc"], out["gem_score_batch_v1"])
    for c in range(0, C, 11):
        assert out["gem_score_batch_tc"][c].tolist() == [oracle.score(tok[l], cand[c, l], cv) for l in range(L)]


def test_score_batch_tc_declines_unsupported_shapes():
    from paper_2605_19945_b200 import _device, _lib

    tok = np.ones((1, 10, 32), dtype=np.int64)
    hist, nmax = _device.counts_to_device_int32(tok)
    cd = torch.zeros((3, 1, 32), dtype=torch.int8, device="cuda")
    lut = torch.zeros((4, nmax + 1), dtype=torch.float64, device="cuda")
    ls = torch.zeros((3, 1), dtype=torch.float64, device="cuda")
    err = torch.zeros((1,), dtype=torch.int32, device="cuda")
    assert _lib.lib().gem_score_batch_tc(hist.data_ptr(), 1, 10, 32, 4, cd.data_ptr(), 3, lut.data_ptr(), nmax,
                                         ls.data_ptr(), err.data_ptr(), None) == 1  # E = 32: not on this path


# ------------------------------------------------------ protocol (tier 1 ABI)

def test_protocol_golden():
    be = kernels.active()
    assert be.BACKEND == "cuda"
    for case in vectors()["protocol"]:
        tok = np.asarray(case["tokens"], dtype=np.int64)
        p = golden_profile(gem, case["profile"])
        a = np.asarray(case["assignment"], dtype=np.int64)
        xs = np.concatenate([c.token_counts for c in p.curves])
        ys = np.concatenate([c.latencies for c in p.curves])
        off = np.concatenate(([0], np.cumsum([c.num_samples for c in p.curves]))).astype(np.int64)
        dl = np.asarray([c.dense_limit for c in p.curves], dtype=np.int64)
        G = p.num_gpus
        loads = np.zeros((tok.shape[0], G), dtype=np.int64)
        for g in range(G):
            loads[:, g] = tok[:, a == g].sum(axis=1)
        lat = np.stack([be.eval_curve_packed(xs, ys, off, dl, g, loads[:, g]) for g in range(G)], axis=1)
        found, i, j, cand = be.best_swap(tok, a, loads, lat, xs, ys, off, dl)
        want = case["best_swap"]
        assert (found, i, j) == (want[0], want[1], want[2]) and cand == f(want[3])
        if case["pair"]:
            got = be.swap_candidate_score(tok, a, loads, lat, xs, ys, off, dl, *case["pair"])
            assert got == f(case["pair_score"])


# ------------------------------------------------------------ search (K6-K8)

def test_search_golden():
    for case in vectors()["search"]:
        tr = gem.ExpertTrace(np.asarray(case["tokens"], dtype=np.int64))
        p = golden_profile(gem, case["profile"])
        res = gem.search(tr, p, gem.SearchConfig(restarts=case["restarts"], rng_seed=case["seed"]))
        assert res.best_score == f(case["best_score"])
        assert res.best_mapping.assignment.tolist() == case["best_assignment"]
        assert res.provenance == case["provenance"]
        for got, want in zip(res.per_restart, case["records"]):
            assert got.provenance == want["provenance"]
            assert got.swap_count == want["swaps"]
            assert list(got.trajectory) == list(fl(want["trajectory"]))
        st = gem.compute_stats(tr)
        init = gem.initial_mapping(st, 1, tr, p, np.random.default_rng(case["seed"] ^ 1))
        assert init.assignment.tolist() == case["initial_1"]


@pytest.mark.parametrize("G,E,T,high", [(2, 8, 16, 300), (4, 16, 40, 300), (8, 64, 128, 300), (3, 12, 1, 300),
                                        (8, 8, 30, 300), (2, 128, 12, 300), (32, 256, 6, 40), (4, 16, 20, 4000),
                                        (64, 128, 10, 60), (48, 96, 7, 80)])
def test_search_matches_oracle(oracle, G, E, T, high):
    """Covers the shared-memory swap scan (one pass, multi-pass with 64x64 expert pairs per GPU pair,
    16 runs per CTA at G=32), the L1 fallback (step totals > 11k: the two table rows exceed smem)
    and G > 32 (the exact v1 greedy and scan: the reference takes any number of GPUs)."""
    rng = np.random.default_rng(G * 1000 + E + T)
    tok = random_counts(rng, T, E, high=high)
    p = mixed_profile(gem, rng, G) if E < 64 else staircase_profile(gem, rng, G, tile=64, tiles=256)
    res = gem.search(gem.ExpertTrace(tok), p, gem.SearchConfig(restarts=5, rng_seed=E))
    want = oracle.search(tok, oracle.Curves.from_profile(p), restarts=5, rng_seed=E)
    assert res.best_score == want["best_score"]
    assert res.best_mapping.assignment.tolist() == want["best_assignment"].tolist()
    assert [r.trajectory for r in res.per_restart] == [tuple(r["trajectory"]) for r in want["records"]]


def test_search_layers_matches_per_layer(oracle):
    rng = np.random.default_rng(4)
    traces = [gem.ExpertTrace(random_counts(rng, 24, 16, high=100)) for _ in range(5)]
    p = staircase_profile(gem, rng, 4)
    cfg = gem.SearchConfig(restarts=3, rng_seed=9)
    batched = gem.search_layers(traces, p, cfg)
    cv = oracle.Curves.from_profile(p)
    for tr, res in zip(traces, batched):
        want = oracle.search(tr.tokens, cv, restarts=3, rng_seed=9)
        assert res.best_score == want["best_score"]
        assert res.best_mapping.assignment.tolist() == want["best_assignment"].tolist()


def test_refine_matches_oracle(oracle):
    rng = np.random.default_rng(12)
    for _ in range(10):
        tok = random_counts(rng, 20, 12, high=200)
        p = mixed_profile(gem, rng, 3)
        a = balanced_assignment(rng, 12, 3)
        got, swaps = gem.refine(gem.ExpertMapping(a, 3), gem.ExpertTrace(tok), p, gem.SearchConfig())
        wa, _, wswaps, _ = oracle.refine(tok, a, oracle.Curves.from_profile(p), 1e-3, 120)
        assert swaps == wswaps and got.assignment.tolist() == wa.tolist()


def _generated_counts(L, steps, E, k, B, seed):
    """Router-like counts from the K9 generator (Zipf popularity, planted groups) via the oracle twin."""
    from oracle import oracle as orc

    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=steps * B, top_k=k, num_experts=E, tokens_per_step=B,
                                seed=seed)
    w, role = ingest.planted_layout(spec)
    ids = orc.gen_topk(L, spec.num_tokens, k, B, E, w, role, ingest._prob_u32(spec.consistent_probability),
                       ingest._prob_u32(spec.burst_probability), spec.burst_multiplier, seed)
    hist, _ = orc.topk_hist(ids, B, E)
    return hist.astype(np.int64)


def test_search_router_like_trace_matches_oracle(oracle):
    """K6 v5 (clamped fp32 screen, 2^-16 window), K7 v3 and K8 at a router-like shape:
    E = 64, G = 8, 512 steps of 1024 tokens x top-8 from the synthetic generator,
    the moderate variability profile; every restart's trajectory bit for bit."""
    tok = _generated_counts(1, 512, 64, 8, 1024, seed=3)[0]
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=8, setup="moderate", tile_size=64, max_tokens=8192,
                                                      rng_seed=2))
    res = gem.search(gem.ExpertTrace(tok), p, gem.SearchConfig(restarts=3, rng_seed=11))
    want = oracle.search(tok, oracle.Curves.from_profile(p), restarts=3, rng_seed=11)
    assert res.best_score == want["best_score"]
    assert res.best_mapping.assignment.tolist() == want["best_assignment"].tolist()
    assert [r.trajectory for r in res.per_restart] == [tuple(r["trajectory"]) for r in want["records"]]


def test_search_deepseek_like_trace_matches_oracle(oracle):
    """The C5 shape (E = 256, G = 32, router-like counts): the load window is wide
    enough that the greedy's 32 fp32 table rows stay in global memory (L1/L2
    gathers) and the scan runs v5 with only its GPU pair's two rows in shared memory."""
    tok = _generated_counts(1, 48, 256, 8, 1024, seed=5)[0]
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=32, setup="moderate", tile_size=64,
                                                      max_tokens=8192, rng_seed=4))
    res = gem.search(gem.ExpertTrace(tok), p, gem.SearchConfig(restarts=2, rng_seed=3))
    want = oracle.search(tok, oracle.Curves.from_profile(p), restarts=2, rng_seed=3)
    assert res.best_score == want["best_score"]
    assert res.best_mapping.assignment.tolist() == want["best_assignment"].tolist()
    assert [r.trajectory for r in res.per_restart] == [tuple(r["trajectory"]) for r in want["records"]]


def test_search_exact_ties_follow_reference_rules(oracle):
    """Duplicated expert columns and GPUs with identical curves make many greedy placements
    and swap candidates tie exactly: lowest GPU in greedy, first (i, j) in the scan."""
    rng = np.random.default_rng(21)
    base = random_counts(rng, 96, 16, high=120)
    tok = np.concatenate([base, base], axis=1)  # experts e and e+16 identical
    xs = np.arange(1, 65, dtype=np.int64) * 32
    ys = np.cumsum(rng.uniform(0.05, 0.5, 64))
    curve = gem.CostCurve(xs, ys, 32, int(xs[-1]))
    p = gem.VariabilityProfile(tuple([curve] * 4), label="identical")  # four identical GPUs
    res = gem.search(gem.ExpertTrace(tok), p, gem.SearchConfig(restarts=4, rng_seed=5))
    want = oracle.search(tok, oracle.Curves.from_profile(p), restarts=4, rng_seed=5)
    assert res.best_score == want["best_score"]
    assert res.best_mapping.assignment.tolist() == want["best_assignment"].tolist()
    assert [r.trajectory for r in res.per_restart] == [tuple(r["trajectory"]) for r in want["records"]]
    assert [r.provenance for r in res.per_restart] == [r["provenance"] for r in want["records"]]


def test_best_swap_screen_versions_agree(monkeypatch):
    """One best-swap scan over many random runs: K6 v5 (default), v5 without the gather
    clamp and v4 (GEM_SCAN_V4) return the same pair and the same exact candidate score."""
    from paper_2605_19945_b200 import _device, _lib

    L, T, E, G, R = 2, 700, 64, 8, 40
    tok = _generated_counts(L, T, E, 8, 1024, seed=9)
    hist, nmax = _device.counts_to_device_int32(tok)
    p = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64, max_tokens=8192,
                                                      rng_seed=4))
    dc = _device.DeviceCurves.from_profile(p)
    lut = dc.lut(nmax)
    rng = np.random.default_rng(0)
    assign = torch.from_numpy(np.stack([balanced_assignment(rng, E, G) for _ in range(R)]).astype(np.int8)).cuda()
    run_layer = torch.from_numpy(np.arange(R, dtype=np.int32) % L).cuda()
    wsb = int(_lib.lib().gem_search_workspace_bytes(R, T, E, G))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")

    def scan():
        found = torch.empty(R, dtype=torch.int32, device="cuda")
        bi, bj = torch.empty_like(found), torch.empty_like(found)
        bc = torch.empty(R, dtype=torch.float64, device="cuda")
        _lib.call("gem_best_swap_runs", hist.data_ptr(), L, T, E, G, lut.data_ptr(), dc.lut_nmax, R,
                  run_layer.data_ptr(), assign.data_ptr(), found.data_ptr(), bi.data_ptr(), bj.data_ptr(),
                  bc.data_ptr(), ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
        return found.cpu().numpy(), bi.cpu().numpy(), bj.cpu().numpy(), bc.cpu().numpy()

    v5 = scan()
    monkeypatch.setenv("GEM_SCAN_NOCLAMP", "1")
    v5n = scan()
    monkeypatch.delenv("GEM_SCAN_NOCLAMP")
    monkeypatch.setenv("GEM_SCAN_V4", "1")
    v4 = scan()
    for a, b in ((v5, v5n), (v5, v4)):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    # and one run against the reference kernel protocol (oracle best_swap)
    from oracle import oracle as orc

    r = 3
    a0 = assign[r].cpu().numpy().astype(np.int64)
    t0 = tok[r % L]
    loads = orc.load_matrix(t0, a0, G)
    cv = orc.Curves.from_profile(p)
    lat = orc.latency_matrix(cv, loads)
    found, i, j, cand = orc.best_swap(t0, a0, loads, lat, cv)
    assert (bool(v5[0][r]), int(v5[1][r]), int(v5[2][r]), float(v5[3][r])) == (bool(found), i, j, cand)


def test_restart_order_kernel_matches_lexsort():
    """gem_restart_order == np.lexsort((arange(E), -keys)) per row (search.py:188-193),
    with exact ties, zeros, -0.0 and all-equal rows."""
    from paper_2605_19945_b200 import _device, _lib

    rng = np.random.default_rng(17)
    for R, E in ((7, 128), (3, 256), (5, 13), (2, 1)):
        keys = rng.random((R, E))
        keys[0, : E // 2] = keys[0, E // 2: 2 * (E // 2)]  # pairs of equal keys
        keys[1 % R] = 0.0
        if E > 3:
            keys[2 % R, :3] = [0.0, -0.0, 0.0]
        d = _device.upload(keys, torch.float64)
        out = _device.empty((R, E), torch.int16)
        _lib.call("gem_restart_order", d.data_ptr(), R, E, out.data_ptr(), _device.stream())
        got = out.cpu().numpy()
        want = np.stack([np.lexsort((np.arange(E), -keys[r])) for r in range(R)])
        assert np.array_equal(got, want)


# ------------------------------------------------- full size, against the reference build

def test_fullsize_layer_matches_reference_build(oracle):
    """One whole C4-shaped layer (2^24 tokens x top-8 -> 16,384 steps, E = 128, G = 8)
    through the reference itself (oracle/_ref, travels with the repo) and the
    B200 path: statistics, candidate scores and a 2-restart search with every
    trajectory, bit for bit (tools/fullsize_parity.py runs three layers with
    the default 30 restarts)."""
    import os

    ref = oracle.import_reference()
    if ref is None:
        pytest.skip("oracle/_ref (the reference build) is not present")
    spec = ingest.TopkTraceSpec(num_layers=1, num_tokens=1 << 24, top_k=8, num_experts=128, tokens_per_step=1024,
                                seed=1)
    st = ingest.trace_statistics(ingest.generate_topk_ids(spec), 1024, 128)
    h = st.hist.hist[0].cpu().numpy().astype(np.int64)
    assert h.shape == (16384, 128)
    rs = ref.compute_stats(ref.ExpertTrace(h))
    mine = gem.compute_stats(gem.ExpertTrace(h))
    assert np.array_equal(rs.mean_utilization, mine.mean_utilization)
    assert np.array_equal(rs.active_fraction, mine.active_fraction)
    assert np.max(np.abs(rs.correlation - mine.correlation)) <= 1e-12
    pspec = dict(num_gpus=8, setup="moderate", tile_size=64, max_tokens=8192, rng_seed=1)
    prof = gem.generate_profile(gem.VariabilitySetupSpec(**pspec))
    rprof = ref.generate_profile(ref.VariabilitySetupSpec(**pspec))
    rng = np.random.default_rng(7)
    for _ in range(4):
        a = rng.permutation(np.repeat(np.arange(8), 16))
        assert gem.score_mapping(gem.ExpertTrace(h), prof, gem.ExpertMapping(a, 8)) == ref.score_mapping(
            ref.ExpertTrace(h), rprof, ref.ExpertMapping(a, 8))
    cfg = dict(restarts=2, rng_seed=3)
    want = ref.search(ref.ExpertTrace(h), rprof, ref.SearchConfig(**cfg), threads=len(os.sched_getaffinity(0)))
    got = gem.search(gem.ExpertTrace(h), prof, gem.SearchConfig(**cfg))
    assert got.best_score == want.best_score
    assert got.best_mapping.assignment.tolist() == want.best_mapping.assignment.tolist()
    assert [(r.provenance, tuple(r.trajectory)) for r in got.per_restart] == [
        (r.provenance, tuple(r.trajectory)) for r in want.per_restart]


def _skewed_counts(rng, T, E, high):
    """Zipf-like rows: a few heavy experts (identity changing over t) over a
    light background -- the DeepSeek-V3 regime where the step floor skips most
    GPU columns."""
    tok = rng.integers(0, max(2, high // 8), (T, E))
    for t in range(T):
        heavy = rng.choice(E, 3, replace=False)
        tok[t, heavy] += rng.integers(high // 2, high, 3)
    return tok


@pytest.mark.parametrize("E,G,split,key32,tied", [(256, 32, True, True, False), (256, 32, False, False, False),
                                                  (128, 16, False, False, False), (64, 32, True, False, False),
                                                  (256, 32, True, True, True), (128, 16, True, True, True)])
def test_score_batch_step_floors(oracle, monkeypatch, E, G, split, key32, tied):
    """K5 step floors (G >= 16): columns whose loads stay at or below the step's
    skip level are not gathered and the maximum starts at the floor key. Must
    equal the no-skip kernel, the CUDA-core scorer and the oracle bit for bit,
    on skewed counts (most columns skipped) and on identical GPU curves (every
    maximum tied with the floor value)."""
    from paper_2605_19945_b200 import _device, _lib

    if split:
        monkeypatch.setenv("GEM_SCORE_SPLIT", "1")
    if key32:
        monkeypatch.setenv("GEM_SCORE_KEY32", "1")
    rng = np.random.default_rng(E * 7 + G + 3 * split + 5 * tied)
    L, T, C = 2, 300, 24
    tok = np.stack([_skewed_counts(rng, T, E, high=900) for _ in range(L)])
    if tied:
        one = staircase_profile(gem, rng, 1, tile=16, tiles=200).curves[0]
        p = gem.VariabilityProfile(tuple(one for _ in range(G)))
    else:
        p = mixed_profile(gem, rng, G)
    cand = np.stack([[balanced_assignment(rng, E, G) for _ in range(L)] for _ in range(C)])
    hist, nmax = _device.counts_to_device_int32(tok)
    dc = _device.DeviceCurves.from_profile(p)
    lut = dc.lut(nmax)
    cd = torch.from_numpy(cand.astype(np.int8)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    out = {}
    for name, fn, noskip in (("skip", "gem_score_batch_tc", False), ("noskip", "gem_score_batch_tc", True),
                             ("v1", "gem_score_batch_v1", False)):
        if noskip:
            monkeypatch.setenv("GEM_SCORE_NOSKIP", "1")
        else:
            monkeypatch.delenv("GEM_SCORE_NOSKIP", raising=False)
        ls = torch.zeros((C, L), dtype=torch.float64, device="cuda")
        err = torch.zeros((1,), dtype=torch.int32, device="cuda")
        rc = getattr(_lib.lib(), fn)(hist.data_ptr(), L, T, E, G, cd.data_ptr(), C, lut.data_ptr(), dc.lut_nmax,
                                     ls.data_ptr(), err.data_ptr(), st)
        assert rc == 0, (name, rc, _lib.lib().gem_last_error())
        out[name] = ls.cpu().numpy()
    assert np.array_equal(out["skip"], out["noskip"])
    assert np.array_equal(out["skip"], out["v1"])
    cv = oracle.Curves.from_profile(p)
    for c in range(0, C, 5):
        assert out["skip"][c].tolist() == [oracle.score(tok[l], cand[c, l], cv) for l in range(L)]
