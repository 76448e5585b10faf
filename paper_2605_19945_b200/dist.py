"""Sharding GEM's data-parallel core over the GPUs of one node (one process per GPU).

North-star subsystem (4). Each rank holds the router ids of a contiguous,
step-aligned TOKEN range (what an EP serving rank observes: its own tokens,
every layer). The only data-path exchanges are:

  1. one all-reduce (SUM, int64/int32 — exact, order-free) of the per-expert
     totals, active-step counts and the step co-activation Gram;
  2. one all-to-all that routes histogram rows to the rank owning each layer
     (layers are split into contiguous blocks), because a candidate score or a
     search run is ONE serial fp64 chain over all steps of a layer and must
     never be split;
  3. all-gathers of per-layer results (search outcome; per-layer candidate
     scores), after which the multi-layer fp64 sums are taken serially in
     ascending layer order on every rank.

No floating-point arithmetic crosses ranks, so every result is bit-identical
to the single-GPU one. The math is delegated to an `ops` object (DeviceOps for
the B200 kernels); the CPU tests drive the same orchestration with the oracle
over gloo.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    num_layers: int
    num_steps: int

    def step_range(self, r: int | None = None) -> tuple[int, int]:
        r = self.rank if r is None else r
        per = -(-self.num_steps // self.world)
        return min(self.num_steps, r * per), min(self.num_steps, (r + 1) * per)

    def layer_range(self, r: int | None = None) -> tuple[int, int]:
        r = self.rank if r is None else r
        base, extra = divmod(self.num_layers, self.world)
        lo = r * base + min(r, extra)
        return lo, lo + base + (1 if r < extra else 0)

    @property
    def max_layers(self) -> int:
        return -(-self.num_layers // self.world)


def _group_world(group):
    return dist.get_world_size(group), dist.get_rank(group)


def allreduce_stats(colsum: torch.Tensor, active: torch.Tensor, gram: torch.Tensor | None, group=None) -> None:
    """In-place exact SUM of the additive integer statistics."""
    for t in (colsum, active, gram):
        if t is not None:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def exchange_hist(hist_local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """[L, T_local, E] token-range rows -> [L_owned, T, E] full-length rows of this rank's layers."""
    L, T_loc, E = hist_local.shape
    world = plan.world
    send_sizes = [(plan.layer_range(p)[1] - plan.layer_range(p)[0]) * T_loc * E for p in range(world)]
    l0, l1 = plan.layer_range()
    Lm = l1 - l0
    recv_steps = [plan.step_range(q)[1] - plan.step_range(q)[0] for q in range(world)]
    recv_sizes = [Lm * s * E for s in recv_steps]
    out = torch.empty(sum(recv_sizes), dtype=hist_local.dtype, device=hist_local.device)
    dist.all_to_all_single(out, hist_local.contiguous().view(-1), output_split_sizes=recv_sizes,
                           input_split_sizes=send_sizes, group=group)
    parts, off = [], 0
    for q in range(world):
        parts.append(out[off:off + recv_sizes[q]].view(Lm, recv_steps[q], E))
        off += recv_sizes[q]
    return torch.cat(parts, dim=1).contiguous()


def gather_layers(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """Stack per-layer rows [L_owned, ...] of every rank into [L, ...] (layer order)."""
    Lm = local.shape[0]
    pad = torch.zeros((plan.max_layers,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:Lm] = local
    bufs = [torch.empty_like(pad) for _ in range(plan.world)]
    dist.all_gather(bufs, pad, group=group)
    rows = []
    for q in range(plan.world):
        a, b = plan.layer_range(q)
        rows.append(bufs[q][: b - a])
    return torch.cat(rows, dim=0)


def gather_layer_columns(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """[C, L_owned] per-rank columns -> [C, L] in layer order."""
    return gather_layers(local.t().contiguous(), plan, group).t().contiguous()


# ---------------------------------------------------------------------------
# the sharded pipeline


@dataclass
class ShardedStats:
    hist_local: torch.Tensor   # [L, T_local, E] this rank's steps
    colsum: torch.Tensor       # [L, E] global (after all-reduce)
    active: torch.Tensor       # [L, E]
    gram: torch.Tensor         # [L, E, E]
    finalized: tuple           # ops.finalize(...) output (replicated)


def sharded_statistics(ids_local, plan: ShardPlan, ops, tokens_per_step: int, num_experts: int,
                       group=None) -> ShardedStats:
    hist, colsum, active = ops.topk_hist(ids_local, tokens_per_step, num_experts)
    gram = ops.gram(hist, tokens_per_step * ids_local.shape[-1])  # every count <= B*k
    allreduce_stats(colsum, active, gram, group)
    fin = ops.finalize(colsum, active, gram, plan.num_steps)
    return ShardedStats(hist, colsum, active, gram, fin)


@dataclass
class ShardedMapping:
    assignments: torch.Tensor  # [L, E] int64, every layer's best mapping
    scores: torch.Tensor       # [L] fp64, every layer's best score
    aggregate: float           # serial fp64 sum in layer order (cli.py:427)


def sharded_search(hist_owned: torch.Tensor, plan: ShardPlan, ops, profile, config, nmax: int,
                   group=None) -> ShardedMapping:
    asg, scores = ops.search(hist_owned, nmax, profile, config)  # [Lm, E] int64, [Lm] fp64
    all_asg = gather_layers(asg, plan, group)
    all_scores = gather_layers(scores, plan, group)
    agg = 0.0
    for v in all_scores.cpu().tolist():
        agg = agg + v
    return ShardedMapping(all_asg, all_scores, agg)


def sharded_candidate_scores(hist_owned: torch.Tensor, plan: ShardPlan, ops, profile, cand: torch.Tensor,
                             nmax: int, group=None):
    """cand [C, L, E] (replicated) -> (total [C] serial over layers, per-layer [C, L])."""
    l0, l1 = plan.layer_range()
    local = ops.score(hist_owned, nmax, profile, cand[:, l0:l1].contiguous())  # [C, Lm] fp64
    per_layer = gather_layer_columns(local, plan, group)
    return ops.layer_sum(per_layer), per_layer


class DeviceOps:
    """The B200 kernels behind the sharded pipeline."""

    def topk_hist(self, ids_local, B, E):
        from .ingest import ids_to_histograms

        h = ids_to_histograms(ids_local, B, E, check_dropped=False)
        return h.hist, h.colsum, h.active

    def gram(self, hist, max_count=-1):
        from .ingest import step_coactivation

        return step_coactivation(hist, max_count=max_count)

    def finalize(self, colsum, active, gram, T):
        from .ingest import classify_device
        from .trace import DeviceStats, finalize_stats

        mu, af, corr = finalize_stats(DeviceStats(colsum, active, gram, T))
        cls = classify_device(colsum, active, gram, T).check()
        return mu, af, corr, cls.cls, cls.group

    def search(self, hist_owned, nmax, profile, config):
        from .search import search_hist

        res = search_hist(hist_owned, nmax, profile, config)
        asg = torch.from_numpy(np.stack([r.best_mapping.assignment for r in res])).to(hist_owned.device)
        scores = torch.tensor([r.best_score for r in res], dtype=torch.float64, device=hist_owned.device)
        return asg, scores

    def score(self, hist_owned, nmax, profile, cand):
        from .mapping import score_candidates_device

        _, per_layer = score_candidates_device(hist_owned, nmax, profile, cand.to(torch.int8))
        return per_layer

    def layer_sum(self, per_layer):
        from . import _lib
        from ._device import ptr, stream

        C, L = per_layer.shape
        out = torch.empty((C,), dtype=torch.float64, device=per_layer.device)
        _lib.call("gem_layer_sum", ptr(per_layer.contiguous()), C, L, ptr(out), stream())
        return out
