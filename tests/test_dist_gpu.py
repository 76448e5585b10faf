"""The sharded pipeline (paper_2605_19945_b200.dist) with the B200 kernels
(DeviceOps) at world size 2 on ONE GPU: two processes share cuda:0 over a gloo
group (collectives stage through host memory). Every result must be
bit-identical to the single-process device run of the unsharded trace."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

L, B, K, E, G, C = 5, 256, 8, 64, 8, 24
T = 40


def _spec():
    from paper_2605_19945_b200 import ingest

    return ingest.TopkTraceSpec(num_layers=L, num_tokens=T * B, top_k=K, num_experts=E, tokens_per_step=B, seed=21)


def _profile():
    import paper_2605_19945_b200 as gem

    return gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64,
                                                         max_tokens=B * K, rng_seed=2))


def _cand():
    rng = np.random.default_rng(8)
    return np.stack([[rng.permutation(np.repeat(np.arange(G), E // G)) for _ in range(L)] for _ in range(C)])


def _config():
    import paper_2605_19945_b200 as gem

    return gem.SearchConfig(restarts=4, rng_seed=9)


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_19945_b200 import dist as gd, ingest

        plan = gd.ShardPlan(world, rank, L, T)
        t0, t1 = plan.step_range()
        ids = ingest.generate_topk_ids(_spec(), token_offset=t0 * B, num_tokens=(t1 - t0) * B)
        ops = gd.DeviceOps()
        st = gd.sharded_statistics(ids, plan, ops, B, E)
        owned = gd.exchange_hist(st.hist_local, plan)
        full = gd.allgather_hist(st.hist_local, plan)
        res = gd.sharded_search(owned, plan, ops, _profile(), _config(), B * K)
        cand = torch.from_numpy(_cand()).cuda()
        total, per_layer = gd.sharded_candidate_scores(full, plan, ops, _profile(), cand, B * K)
        torch.cuda.synchronize()
        if rank == 0:
            mu, af, corr, cls, grp = st.finalized
            np.savez(out_path, pack=st.stats.pack.cpu().numpy(), mu=mu.cpu().numpy(), af=af.cpu().numpy(),
                     corr=corr.cpu().numpy(), cls=cls.cpu().numpy(), grp=grp.cpu().numpy(), full=full.cpu().numpy(),
                     asg=res.assignments.cpu().numpy(), scores=res.scores.cpu().numpy(),
                     agg=np.array([res.aggregate]), total=total.cpu().numpy(), per_layer=per_layer.cpu().numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2])
def test_device_ops_world2_on_one_gpu_bit_identical(tmp_path, world):
    from paper_2605_19945_b200 import ingest
    from paper_2605_19945_b200.mapping import score_candidates_device
    from paper_2605_19945_b200.search import search_hist

    out = tmp_path / "rank0.npz"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    got = np.load(out)
    # the single-process device run of the whole trace
    ids = ingest.generate_topk_ids(_spec())
    st = ingest.trace_statistics(ids, B, E)
    st.check()
    assert np.array_equal(got["pack"], st.hist.stats.pack.cpu().numpy())  # colsum/active/heavy/Gram, one buffer
    assert np.array_equal(got["full"], st.hist.hist.cpu().numpy())
    assert np.array_equal(got["mu"], st.mean_utilization.cpu().numpy())
    assert np.array_equal(got["af"], st.active_fraction.cpu().numpy())
    assert np.array_equal(got["corr"], st.correlation.cpu().numpy())
    assert np.array_equal(got["cls"], st.classes.cls.cpu().numpy())
    assert np.array_equal(got["grp"], st.classes.group.cpu().numpy())
    res = search_hist(st.hist.hist, B * K, _profile(), _config())
    assert got["scores"].tolist() == [r.best_score for r in res]
    assert got["asg"].tolist() == [r.best_mapping.assignment.tolist() for r in res]
    agg = 0.0
    for r in res:
        agg = agg + r.best_score
    assert got["agg"][0] == agg
    total, per_layer = score_candidates_device(st.hist.hist, B * K, _profile(),
                                               torch.from_numpy(_cand()).cuda().to(torch.int8))
    assert np.array_equal(got["total"], total.cpu().numpy())
    assert np.array_equal(got["per_layer"], per_layer.cpu().numpy())
