"""Sharding GEM's data-parallel core over the GPUs of one node (one process per GPU).

North-star subsystem (4). Each rank holds the router ids of a contiguous,
step-aligned TOKEN range (what an EP serving rank observes: its own tokens,
every layer). The data-path exchanges are:

  1. ONE all-reduce (SUM over int64 words — exact, order-free) of the packed
     statistics buffer (trace.DeviceStats.pack): per-expert totals, active and
     heavy step counts, the step co-activation Gram and, when requested, the
     token-level co-selection counts;
  2. for the search: one all-to-all that routes histogram rows to the rank
     owning each layer (layers split into contiguous blocks), because a search
     run is ONE serial fp64 chain over all steps of a layer and must never be
     split; then an all-gather of the per-layer results;
  3. for candidate scoring: candidates are split by INDEX;
     every rank needs all layers' full-length rows, so the histogram shards
     are all-gathered once, each rank scores its candidate range on every
     layer, and the fp64 scores (per layer and the serial layer sum, computed
     on the rank that owns the candidate) are all-gathered.

No floating-point arithmetic crosses ranks, so every result is bit-identical
to the single-GPU one. The math is delegated to an `ops` object (DeviceOps for
the B200 kernels); the CPU tests drive the same orchestration with the oracle
over gloo, and a two-process gloo test drives DeviceOps on one GPU (gloo
collectives on CUDA tensors stage through host memory, see _collective).
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

    def candidate_range(self, C: int, r: int | None = None) -> tuple[int, int]:
        r = self.rank if r is None else r
        base, extra = divmod(C, self.world)
        lo = r * base + min(r, extra)
        return lo, lo + base + (1 if r < extra else 0)

    @property
    def max_layers(self) -> int:
        return -(-self.num_layers // self.world)


def _staged(group) -> bool:
    """gloo has no device path for every collective: stage CUDA tensors through host."""
    return dist.get_backend(group) == "gloo"


def _collective(fn, group, *tensors):
    """Run fn(*tensors) on host copies when the backend needs them, copying results back."""
    if not _staged(group) or not any(t.is_cuda for t in tensors):
        fn(*tensors)
        return
    host = [t.cpu() for t in tensors]
    fn(*host)
    for t, h in zip(tensors, host):
        t.copy_(h)


def allreduce_stats(stats, group=None) -> None:
    """In-place exact SUM of the packed additive integer statistics (ONE collective)."""
    _collective(lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group), group, stats.pack)


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
    src = hist_local.contiguous().view(-1)
    _collective(lambda o, i: dist.all_to_all_single(o, i, output_split_sizes=recv_sizes, input_split_sizes=send_sizes,
                                                    group=group), group, out, src)
    parts, off = [], 0
    for q in range(world):
        parts.append(out[off:off + recv_sizes[q]].view(Lm, recv_steps[q], E))
        off += recv_sizes[q]
    return torch.cat(parts, dim=1).contiguous()


def allgather_hist(hist_local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """[L, T_local, E] token-range rows of every rank -> [L, T, E] on every rank."""
    L, _, E = hist_local.shape
    per = -(-plan.num_steps // plan.world)
    pad = torch.zeros((L, per, E), dtype=hist_local.dtype, device=hist_local.device)
    pad[:, :hist_local.shape[1]] = hist_local
    bufs = [torch.empty_like(pad) for _ in range(plan.world)]
    _collective(lambda *b: dist.all_gather(list(b[1:]), b[0], group=group), group, pad, *bufs)
    parts = []
    for q in range(plan.world):
        a, b = plan.step_range(q)
        parts.append(bufs[q][:, : b - a])
    return torch.cat(parts, dim=1).contiguous()


def _gather_rows(local: torch.Tensor, rows: int, counts: list[int], group=None) -> torch.Tensor:
    """All-gather variable-length leading-dimension blocks (padded to `rows`) and concatenate in rank order."""
    pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in counts]
    _collective(lambda *b: dist.all_gather(list(b[1:]), b[0], group=group), group, pad, *bufs)
    return torch.cat([bufs[q][:n] for q, n in enumerate(counts)], dim=0)


def gather_layers(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """Stack per-layer rows [L_owned, ...] of every rank into [L, ...] (layer order)."""
    counts = [plan.layer_range(q)[1] - plan.layer_range(q)[0] for q in range(plan.world)]
    return _gather_rows(local, plan.max_layers, counts, group)


def gather_layer_columns(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """[C, L_owned] per-rank columns -> [C, L] in layer order."""
    return gather_layers(local.t().contiguous(), plan, group).t().contiguous()


# ---------------------------------------------------------------------------
# the sharded pipeline


@dataclass
class ShardedStats:
    hist_local: torch.Tensor   # [L, T_local, E] this rank's steps
    stats: object              # DeviceStats-like: global sums after the all-reduce (views of .pack)
    finalized: tuple           # ops.finalize(...) output (replicated)

    @property
    def colsum(self):
        return self.stats.colsum

    @property
    def active(self):
        return self.stats.active

    @property
    def heavy(self):
        return self.stats.heavy

    @property
    def gram(self):
        return self.stats.gram


def sharded_statistics(ids_local, plan: ShardPlan, ops, tokens_per_step: int, num_experts: int,
                       group=None) -> ShardedStats:
    hist, stats = ops.topk_hist(ids_local, tokens_per_step, num_experts, plan.num_steps)
    ops.gram(hist, tokens_per_step * ids_local.shape[-1], stats)  # every count <= B*k
    allreduce_stats(stats, group)
    fin = ops.finalize(stats)
    return ShardedStats(hist, stats, fin)


@dataclass
class ShardedMapping:
    assignments: torch.Tensor  # [L, E] int64, every layer's best mapping
    scores: torch.Tensor       # [L] fp64, every layer's best score
    aggregate: float           # serial fp64 sum in layer order (cli.py:427)


def sharded_search(hist_owned: torch.Tensor, plan: ShardPlan, ops, profile, config, nmax: int,
                   group=None) -> ShardedMapping:
    E = hist_owned.shape[2]
    if hist_owned.shape[0]:
        asg, scores = ops.search(hist_owned, nmax, profile, config)  # [Lm, E] int64, [Lm] fp64
    else:  # more ranks than layers: this rank owns none
        asg = torch.zeros((0, E), dtype=torch.int64, device=hist_owned.device)
        scores = torch.zeros((0,), dtype=torch.float64, device=hist_owned.device)
    all_asg = gather_layers(asg, plan, group)
    all_scores = gather_layers(scores, plan, group)
    agg = 0.0
    for v in all_scores.cpu().tolist():
        agg = agg + v
    return ShardedMapping(all_asg, all_scores, agg)


def sharded_candidate_scores(hist_full: torch.Tensor, plan: ShardPlan, ops, profile, cand: torch.Tensor,
                             nmax: int, group=None):
    """Candidates split by index. hist_full [L, T, E] (allgather_hist), cand [C, L, E] (replicated)
    -> (total [C] serial over layers, per-layer [C, L]), identical on every rank."""
    C = cand.shape[0]
    c0, c1 = plan.candidate_range(C)
    L = hist_full.shape[0]
    if c1 > c0:
        per_layer = ops.score(hist_full, nmax, profile, cand[c0:c1].contiguous())  # [Cr, L] fp64
        total = ops.layer_sum(per_layer)
    else:
        per_layer = torch.zeros((0, L), dtype=torch.float64, device=hist_full.device)
        total = torch.zeros((0,), dtype=torch.float64, device=hist_full.device)
    counts = [plan.candidate_range(C, q)[1] - plan.candidate_range(C, q)[0] for q in range(plan.world)]
    rows = max(counts)
    both = torch.cat([total.view(-1, 1), per_layer], dim=1)  # one all-gather for both
    g = _gather_rows(both, rows, counts, group)
    return g[:, 0].contiguous(), g[:, 1:].contiguous()


def sharded_candidate_scores_by_layer(hist_owned: torch.Tensor, plan: ShardPlan, ops, profile, cand: torch.Tensor,
                                      nmax: int, group=None):
    """Alternative split by LAYER (no histogram all-gather; the max rank carries ceil(L/P) layers)."""
    l0, l1 = plan.layer_range()
    if l1 > l0:
        local = ops.score(hist_owned, nmax, profile, cand[:, l0:l1].contiguous())  # [C, Lm] fp64
    else:
        local = torch.zeros((cand.shape[0], 0), dtype=torch.float64, device=cand.device)
    per_layer = gather_layer_columns(local, plan, group)
    return ops.layer_sum(per_layer), per_layer


class DeviceOps:
    """The B200 kernels behind the sharded pipeline."""

    def topk_hist(self, ids_local, B, E, T_global):
        from .ingest import ids_to_histograms

        h = ids_to_histograms(ids_local, B, E, check_dropped=False)
        h.stats.num_steps = T_global  # the statistics are completed by the all-reduce
        return h.hist, h.stats

    def gram(self, hist, max_count, stats):
        from .ingest import step_coactivation

        step_coactivation(hist, stats.gram, max_count=max_count)

    def finalize(self, stats):
        from .ingest import classify_device
        from .trace import finalize_stats

        mu, af, corr = finalize_stats(stats)
        cls = classify_device(stats.colsum, stats.heavy, stats.gram, stats.num_steps).check()
        return mu, af, corr, cls.cls, cls.group

    def search(self, hist_owned, nmax, profile, config):
        from .search import search_hist

        res = search_hist(hist_owned, nmax, profile, config)
        asg = torch.from_numpy(np.stack([r.best_mapping.assignment for r in res])).to(hist_owned.device)
        scores = torch.tensor([r.best_score for r in res], dtype=torch.float64, device=hist_owned.device)
        return asg, scores

    def score(self, hist, nmax, profile, cand):
        from .mapping import score_candidates_device

        _, per_layer = score_candidates_device(hist, nmax, profile, cand.to(torch.int8))
        return per_layer

    def layer_sum(self, per_layer):
        from . import _lib
        from ._device import ptr, stream

        C, L = per_layer.shape
        out = torch.empty((C,), dtype=torch.float64, device=per_layer.device)
        _lib.call("gem_layer_sum", ptr(per_layer.contiguous()), C, L, ptr(out), stream())
        return out
