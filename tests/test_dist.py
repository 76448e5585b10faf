"""The N>1 path on CPU: world-size-2 gloo runs of the sharded pipeline
(paper_2605_19945_b200.dist) with the oracle as the compute backend, checked
against a single-process oracle run on the unsharded trace."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19945_b200.dist import (
    ShardPlan,
    allgather_hist,
    exchange_hist,
    sharded_candidate_scores,
    sharded_candidate_scores_by_layer,
    sharded_search,
    sharded_statistics,
)
from paper_2605_19945_b200.trace import DeviceStats

L, T, B, K, E, G, C = 5, 24, 32, 4, 16, 4, 12
WEIGHT_SEED, GEN_SEED = 3, 17


def _inputs():
    from oracle import oracle

    rng = np.random.default_rng(WEIGHT_SEED)
    weight = rng.integers(1, 5000, (L, E)).astype(np.uint32)
    role = np.zeros((L, E), dtype=np.int8)
    role[:, 1], role[:, [2, 3]] = 1, 2
    ids = oracle.gen_topk(L, T * B, K, B, E, weight, role, int(0.85 * 2**32), int(0.17 * 2**32), 3, GEN_SEED)
    cand = np.stack([[rng.permutation(np.repeat(np.arange(G), E // G)) for _ in range(L)] for _ in range(C)])
    return ids, cand


def _curves():
    from oracle import oracle

    xs = np.arange(1, 65, dtype=np.int64) * 4
    return oracle.Curves([(xs, np.cumsum(np.full(64, 0.25 + 0.05 * g)), int(xs[-1])) for g in range(G)])


class OracleOps:
    """CPU twin of DeviceOps: same contract, oracle arithmetic."""

    def __init__(self, curves):
        from oracle import oracle

        self.o = oracle
        self.curves = curves

    def topk_hist(self, ids_local, B, E, T_global):
        hist, _ = self.o.topk_hist(ids_local.numpy(), B, E)
        st = DeviceStats.allocate(hist.shape[0], E, T_global, device=torch.device("cpu"))
        for l in range(hist.shape[0]):
            cs, ac, hv = self.o.colstats3(hist[l])
            st.colsum[l], st.active[l], st.heavy[l] = torch.from_numpy(cs), torch.from_numpy(ac), torch.from_numpy(hv)
        return torch.from_numpy(hist.astype(np.int32)), st

    def gram(self, hist, max_count, stats):
        stats.gram.copy_(torch.from_numpy(np.stack([self.o.gram(h.numpy()) for h in hist])))

    def finalize(self, st):
        cs, ac, hv, gr, T = st.colsum.numpy(), st.active.numpy().astype(np.int64), st.heavy.numpy(), \
            st.gram.numpy(), st.num_steps
        mu = np.stack([c / int(c.sum()) for c in cs])
        classes = [self.o.classify_from_stats(cs[l], hv[l], gr[l], T) for l in range(cs.shape[0])]
        return mu, ac / T, np.stack([c for c, _ in classes]), np.stack([g for _, g in classes])

    def search(self, hist_owned, nmax, profile, config):
        res = [self.o.search(h.numpy(), self.curves, restarts=config["restarts"], rng_seed=config["seed"])
               for h in hist_owned]
        return (torch.from_numpy(np.stack([r["best_assignment"] for r in res])),
                torch.tensor([r["best_score"] for r in res], dtype=torch.float64))

    def score(self, hist_owned, nmax, profile, cand):
        c = cand.numpy()
        return torch.tensor([[self.o.score(hist_owned[l].numpy(), c[i, l], self.curves)
                              for l in range(hist_owned.shape[0])] for i in range(c.shape[0])], dtype=torch.float64)

    def layer_sum(self, per_layer):
        return torch.from_numpy(np.cumsum(per_layer.numpy(), axis=1)[:, -1].copy())  # serial per row


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids, cand = _inputs()
        plan = ShardPlan(world, rank, L, T)
        t0, t1 = plan.step_range()
        ops = OracleOps(_curves())
        st = sharded_statistics(torch.from_numpy(ids[:, t0 * B:t1 * B].copy()), plan, ops, B, E)
        owned = exchange_hist(st.hist_local, plan)
        full = allgather_hist(st.hist_local, plan)
        cfg = {"restarts": 3, "seed": 5}
        mp_res = sharded_search(owned, plan, ops, None, cfg, B * K)
        total, per_layer = sharded_candidate_scores(full, plan, ops, None, torch.from_numpy(cand), B * K)
        total2, per_layer2 = sharded_candidate_scores_by_layer(owned, plan, ops, None, torch.from_numpy(cand), B * K)
        assert torch.equal(total, total2) and torch.equal(per_layer, per_layer2)
        if rank == 0:
            mu, af, cls, grp = st.finalized
            np.savez(out_path, colsum=st.colsum.numpy(), active=st.active.numpy(), heavy=st.heavy.numpy(),
                     gram=st.gram.numpy(), mu=mu, af=af, cls=cls, grp=grp, owned=owned.numpy(), full=full.numpy(),
                     asg=mp_res.assignments.numpy(), scores=mp_res.scores.numpy(), agg=np.array([mp_res.aggregate]),
                     total=total.numpy(), per_layer=per_layer.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_plan_covers_everything():
    for world in (1, 2, 3, 8):
        for Lx, Tx in ((94, 16384), (5, 7), (3, 24)):
            plans = [ShardPlan(world, r, Lx, Tx) for r in range(world)]
            steps = [p.step_range() for p in plans]
            layers = [p.layer_range() for p in plans]
            assert steps[0][0] == 0 and steps[-1][1] == Tx
            assert layers[0][0] == 0 and layers[-1][1] == Lx
            assert all(a[1] == b[0] for a, b in zip(steps, steps[1:]))
            assert all(a[1] == b[0] for a, b in zip(layers, layers[1:]))
            assert max(b - a for a, b in layers) - min(b - a for a, b in layers) <= 1


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3, 4, 6])
def test_gloo_pipeline_matches_single_process(tmp_path, oracle, world):
    """world 3 and 4 split the 5 layers and 24 steps unevenly (2/2/1, 2/1/1/1);
    world 6 leaves one rank without a layer and splits 12 candidates 2 each."""
    out = tmp_path / "rank0.npz"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    got = np.load(out)
    ids, cand = _inputs()
    curves = _curves()
    hist, _ = oracle.topk_hist(ids, B, E)
    # statistics: exact integers, bit-exact floats
    l0, l1 = ShardPlan(world, 0, L, T).layer_range()
    assert np.array_equal(got["owned"], hist[l0:l1])  # the layers rank 0 owns
    assert np.array_equal(got["full"], hist)
    assert np.array_equal(got["colsum"], hist.sum(axis=1))
    assert np.array_equal(got["active"], (hist > 0).sum(axis=1))
    assert np.array_equal(got["heavy"], np.stack([oracle.heavy_counts(h) for h in hist]))
    for l in range(L):
        assert np.array_equal(got["gram"][l], oracle.gram(hist[l]))
        mu, af, _ = oracle.stats(hist[l])
        assert np.array_equal(got["mu"][l], mu) and np.array_equal(got["af"][l], af)
        cls, grp = oracle.classify(hist[l])
        assert np.array_equal(got["cls"][l], cls) and np.array_equal(got["grp"][l], grp)
    # search: every layer's mapping and score, aggregate in layer order
    agg = 0.0
    for l in range(L):
        want = oracle.search(hist[l], curves, restarts=3, rng_seed=5)
        assert got["asg"][l].tolist() == want["best_assignment"].tolist()
        assert got["scores"][l] == want["best_score"]
        agg = agg + want["best_score"]
    assert got["agg"][0] == agg
    # candidates: per-layer scores and serial layer sums
    for c in range(C):
        per = [oracle.score(hist[l], cand[c, l], curves) for l in range(L)]
        assert got["per_layer"][c].tolist() == per
        s = 0.0
        for v in per:
            s = s + v
        assert got["total"][c] == s
