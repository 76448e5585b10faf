"""Router top-k trace ingestion, co-activation and expert classification.

North-star subsystems (1) and (2). The reference starts from an already
counted trace (`ExpertTrace`, /root/reference/pkg/src/gemap/trace.py:24-45);
here the input is what an MoE router actually emits — top-k expert ids per
token, int16 or int32, [layers, tokens, k] — and everything downstream of it
stays on the device:

  ids --K1--> hist [L,T,E] int32 (+ colsum, active-step counts, dropped ids)
      --K2--> step co-activation Gram  G[a,b] = sum_t h_a(t) h_b(t)  (int64, exact)
      --K3--> mean_utilization / active_fraction / Pearson  (trace.py:87-114)
      --K3b-> consistent / temporal classes and correlated-temporal groups

The histogram of layer l is exactly `ExpertTrace.tokens` for that layer, so
every reference entry point (score_mapping, search, ...) consumes it directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from ._device import ptr, stream
from .errors import ValidationError
from .trace import DeviceStats, ExpertTrace, TraceStats, finalize_stats

CLASS_OTHER = _lib.GEM_CLASS_OTHER
CLASS_CONSISTENT = _lib.GEM_CLASS_CONSISTENT
CLASS_TEMPORAL = _lib.GEM_CLASS_TEMPORAL
ROLE_BACKGROUND, ROLE_CONSISTENT = 0, 1  # role >= 2: member of temporal group role-2


# ---------------------------------------------------------------------------
# synthetic router ids (K9)


@dataclass(frozen=True)
class TopkTraceSpec:
    """Synthetic routing trace of a model shape (BASELINE.json configs).

    Per layer: Zipf(zipf_s) popularity over a seeded expert permutation; the
    `consistent` most popular experts are gated on per step with
    `consistent_probability`; `num_groups` temporal groups of `group_size`
    experts (next in popularity) burst jointly with `burst_probability` at
    `burst_multiplier` x weight; all other experts are always on. Every token
    picks `top_k` distinct experts proportionally to the gated weights."""

    num_layers: int
    num_tokens: int
    top_k: int
    num_experts: int
    tokens_per_step: int = 1024
    zipf_s: float = 1.1
    consistent: int = 3
    num_groups: int = 2
    group_size: int = 2
    consistent_probability: float = 0.85
    burst_probability: float = 0.17
    burst_multiplier: int = 3
    seed: int = 0

    def __post_init__(self):
        if min(self.num_layers, self.num_tokens, self.top_k, self.num_experts, self.tokens_per_step) < 1:
            raise ValidationError("TopkTraceSpec: sizes must be >= 1")
        designated = self.consistent + self.num_groups * self.group_size
        if designated + self.top_k > self.num_experts:
            raise ValidationError("TopkTraceSpec: need at least top_k background experts")
        if self.top_k > 32 or self.num_experts > 512:
            raise ValidationError("TopkTraceSpec: top_k <= 32 and num_experts <= 512")

    @property
    def num_steps(self) -> int:
        return -(-self.num_tokens // self.tokens_per_step)


def planted_layout(spec: TopkTraceSpec) -> tuple[np.ndarray, np.ndarray]:
    """(integer weights [L,E] uint32, roles [L,E] int8) — the planted ground truth."""
    L, E = spec.num_layers, spec.num_experts
    weight = np.zeros((L, E), dtype=np.uint32)
    role = np.zeros((L, E), dtype=np.int8)
    ranks = np.arange(E)
    base = np.maximum(1, np.rint((1 << 20) / np.power(ranks + 1.0, spec.zipf_s))).astype(np.uint32)
    for l in range(L):
        perm = np.random.default_rng([spec.seed, l]).permutation(E)  # perm[r] = expert of rank r
        weight[l, perm] = base
        r = 0
        for _ in range(spec.consistent):
            role[l, perm[r]] = ROLE_CONSISTENT
            r += 1
        for g in range(spec.num_groups):
            for _ in range(spec.group_size):
                role[l, perm[r]] = 2 + g
                r += 1
    return weight, role


def _prob_u32(p: float) -> int:
    return min(int(round(p * 4294967296.0)), 0xFFFFFFFF)


def generate_topk_ids(spec: TopkTraceSpec, dtype: torch.dtype = torch.int16, token_offset: int = 0,
                      num_tokens: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device ids [L, n, k] for global tokens [token_offset, token_offset+n) (Philox; exact CPU twin in oracle/)."""
    n = spec.num_tokens - token_offset if num_tokens is None else num_tokens
    weight, role = planted_layout(spec)
    w = _device.upload(weight.view(np.int32), torch.int32)  # uint32 bits in int32 storage
    r = _device.upload(role, torch.int8)
    id_bytes = {torch.int16: 2, torch.int32: 4}[dtype]
    if out is None:
        out = _device.empty((spec.num_layers, n, spec.top_k), dtype)
    _lib.call("gem_gen_topk", spec.num_layers, n, spec.top_k, spec.tokens_per_step, spec.num_experts, ptr(w),
              ptr(r), _prob_u32(spec.consistent_probability), _prob_u32(spec.burst_probability),
              spec.burst_multiplier, spec.seed, token_offset, id_bytes, ptr(out), stream())
    return out


# ---------------------------------------------------------------------------
# K1: ids -> histograms


@dataclass
class Histograms:
    """Per-step expert histograms of a (shard of a) top-k trace, on the device.

    The additive per-expert statistics live in `stats` (one int64 buffer for
    colsum / active / heavy / Gram / co-selection: one all-reduce combines
    token-range shards)."""

    hist: torch.Tensor      # [L, T, E] int32
    stats: DeviceStats      # colsum [L,E] int64, active/heavy [L,E] int32, gram, coselect (accumulated)
    dropped: torch.Tensor   # [L] int64 ids outside [0, E)
    tokens_per_step: int
    top_k: int = -1         # ids per token (bounds every count by tokens_per_step * top_k)

    @property
    def colsum(self) -> torch.Tensor:
        return self.stats.colsum

    @property
    def active(self) -> torch.Tensor:
        return self.stats.active

    @property
    def heavy(self) -> torch.Tensor:
        return self.stats.heavy

    @property
    def max_count(self) -> int:
        """Upper bound on every histogram cell (-1 = unknown)."""
        return self.tokens_per_step * self.top_k if self.top_k > 0 else -1

    @property
    def num_layers(self) -> int:
        return self.hist.shape[0]

    @property
    def num_steps(self) -> int:
        return self.hist.shape[1]

    @property
    def num_experts(self) -> int:
        return self.hist.shape[2]

    def to_traces(self) -> list[ExpertTrace]:
        """One reference `ExpertTrace` per layer (int64 counts on the host)."""
        h = _device.host(self.hist).astype(np.int64)
        return [ExpertTrace(h[l]) for l in range(h.shape[0])]


@_device.nvtx("gem.K1 ids_to_histograms")
def ids_to_histograms(ids: torch.Tensor, tokens_per_step: int, num_experts: int,
                      hist: torch.Tensor | None = None, check_dropped: bool = True,
                      with_gram: bool = True, with_coselect: bool = False) -> Histograms:
    """K1: top-k ids [L, N, k] (int16/int32, device) -> per-step histograms.

    Steps are consecutive blocks of `tokens_per_step` tokens (the last may be
    short). Ids outside [0, num_experts) are counted in `dropped`; with
    check_dropped (default) any dropped id raises ValidationError (this
    synchronises). with_gram / with_coselect reserve the Gram and the
    co-selection counts in the same statistics buffer (filled by K2 / K2b)."""
    if ids.dim() != 3:
        raise ValidationError(f"ids must be [layers, tokens, k], got shape {tuple(ids.shape)}")
    if ids.dtype not in (torch.int16, torch.int32):
        raise ValidationError("ids must be int16 or int32")
    if not ids.is_cuda:
        ids = ids.to(_device.device())
    ids = ids.contiguous()
    L, N, k = ids.shape
    T = -(-N // tokens_per_step)
    if hist is None:
        hist = _device.empty((L, T, num_experts), torch.int32)
    ds = DeviceStats.allocate(L, num_experts, T, with_gram=with_gram, with_coselect=with_coselect)
    dropped = _device.zeros((L,), torch.int64)
    _lib.call("gem_topk_hist", ptr(ids), ids.element_size(), L, N, k, tokens_per_step, num_experts, ptr(hist),
              ptr(ds.colsum), ptr(ds.active), ptr(ds.heavy), ptr(dropped), stream())
    if with_coselect:
        token_coselection(ids, num_experts, out=ds.coselect)
    h = Histograms(hist, ds, dropped, tokens_per_step, k)
    if check_dropped and int(dropped.sum().item()):
        raise ValidationError(f"{int(dropped.sum().item())} expert ids outside [0, {num_experts})")
    return h


# ---------------------------------------------------------------------------
# K2b: token-level co-selection


def token_coselection(ids: torch.Tensor, num_experts: int, out: torch.Tensor | None = None,
                      path: str = "auto") -> torch.Tensor:
    """K2b: C[l,a,b] = #tokens of layer l whose top-k ids hold both a and b (int32 [L,E,E]).

    OᵀO of the 0/1 selection indicator: ids outside [0, E) are ignored and a
    repeated id within one token counts once, so diag(C[l]) equals K1's
    colsum[l] for distinct router ids. ACCUMULATES into `out` (zeros if None).
    path: "auto" (tcgen05 kind::i8 where gem_coselect_path allows, CUDA-core
    scatter otherwise), "tc" or "scatter"."""
    if ids.dim() != 3 or ids.dtype not in (torch.int16, torch.int32):
        raise ValidationError("ids must be int16/int32 [layers, tokens, k]")
    if not ids.is_cuda:
        ids = ids.to(_device.device())
    ids = ids.contiguous()
    L, N, k = ids.shape
    if out is None:
        out = _device.zeros((L, num_experts, num_experts), torch.int32)
    if tuple(out.shape) != (L, num_experts, num_experts) or out.dtype != torch.int32:
        raise ValidationError("out must be int32 [layers, E, E]")
    fn = {"auto": "gem_coselect", "tc": "gem_coselect_tc", "scatter": "gem_coselect_scatter"}[path]
    _lib.call(fn, ptr(ids), ids.element_size(), L, N, k, num_experts, ptr(out), stream())
    return out


def coselection_path(ids: torch.Tensor, num_experts: int) -> str:
    """Which kernel gem_coselect runs for these ids: "tc" or "scatter"."""
    L, N, k = ids.shape
    return "tc" if _lib.lib().gem_coselect_path(ptr(ids), ids.element_size(), N, k, num_experts) == 1 else "scatter"


# ---------------------------------------------------------------------------
# K2 + K3: statistics, co-activation, classification


def step_coactivation(hist: torch.Tensor, gram: torch.Tensor | None = None, max_count: int = -1) -> torch.Tensor:
    """K2: G[l,a,b] = sum_t hist[l,t,a] * hist[l,t,b] (int64; upper triangle a<=b authoritative).

    max_count bounds every count (-1 = unknown); with E % 128 == 0 and
    max_count <= 65535 the Gram runs on the tensor cores (tcgen05 kind::i8)."""
    L, T, E = hist.shape
    if gram is None:
        gram = _device.zeros((L, E, E), torch.int64)
    _lib.call("gem_step_gram", ptr(hist), L, T, E, max_count, ptr(gram), stream())
    return gram


@dataclass
class ExpertClasses:
    cls: torch.Tensor    # [L, E] int8: CLASS_OTHER / CLASS_CONSISTENT / CLASS_TEMPORAL
    group: torch.Tensor  # [L, E] int16: lowest expert index of the correlated-temporal group, -1 otherwise
    err: torch.Tensor | None = None  # [1] int32 device flag set by K3b on int128 range overflow

    def check(self) -> "ExpertClasses":
        """Raise if the (asynchronous) classification overflowed its exact predicate range."""
        if self.err is not None and int(self.err.item()):
            raise _lib.KernelError("gem_classify: correlation statistics exceed the exact int128 predicate range")
        return self


@dataclass(frozen=True)
class ClassifyConfig:
    """The paper's split of the heavily used experts:

    * a step is *heavy* for expert e when e receives at least its fair share of
      the step's routed ids, h_t[e] * E >= sum_e' h_t[e'] (and h_t[e] > 0);
    * consistent: heavy in >= consistent_fraction of the steps ("used in almost
      every time step"; planted consistent experts are on in ~85% of steps);
    * temporal: not consistent, heavy in at least one step, and Pearson
      r >= correlation_threshold with another such expert (correlated temporal
      experts, r = 0.88 in PAPER.md Fig. 8); groups are the connected
      components of that graph, labelled by their lowest expert index;
    * everything else (light experts) is CLASS_OTHER.

    Thresholds are exact rationals (num, den) so every predicate is integer-exact."""

    consistent_fraction: tuple[int, int] = (4, 5)
    correlation_threshold: tuple[int, int] = (4, 5)


def classify_device(colsum, heavy, gram, num_steps: int, config: ClassifyConfig = ClassifyConfig(),
                    out: ExpertClasses | None = None) -> ExpertClasses:
    """K3b on the device, asynchronously (out: optional preallocated classes; its err flag is re-zeroed)."""
    L, E = colsum.shape
    if out is not None:
        cls, grp, err = out.cls, out.group, out.err
        err.zero_()
    else:
        cls = _device.empty((L, E), torch.int8)
        grp = _device.empty((L, E), torch.int16)
        err = _device.zeros((1,), torch.int32)
    cn, cd = config.consistent_fraction
    rn, rd = config.correlation_threshold
    _lib.call("gem_classify", ptr(colsum), ptr(heavy), ptr(gram), L, num_steps, E, cn, cd, rn, rd, ptr(cls),
              ptr(grp), ptr(err), stream())
    return ExpertClasses(cls, grp, err)


@dataclass
class TraceStatistics:
    """Everything the statistics phase produces, per layer, on the device."""

    hist: Histograms
    gram: torch.Tensor
    mean_utilization: torch.Tensor  # [L, E] fp64
    active_fraction: torch.Tensor   # [L, E] fp64
    correlation: torch.Tensor | None  # [L, E, E] fp64
    classes: ExpertClasses | None
    extra: dict = field(default_factory=dict)

    def check(self) -> "TraceStatistics":
        """Raise on any asynchronous kernel-side error flag (synchronises the stream)."""
        if self.classes is not None:
            self.classes.check()
        return self

    def layer_stats(self, l: int) -> TraceStats:
        """The reference's TraceStats for layer l."""
        return TraceStats(_device.host(self.mean_utilization[l]), _device.host(self.active_fraction[l]),
                          _device.host(self.correlation[l]))


@_device.nvtx("gem.trace_statistics")
def trace_statistics(ids: torch.Tensor, tokens_per_step: int, num_experts: int, correlation: bool = True,
                     classify: bool = True, config: ClassifyConfig = ClassifyConfig(),
                     coselect: bool = False) -> TraceStatistics:
    """The whole statistics phase for one top-k trace (all layers): K1 (+ K2b) -> K2 -> K3 -> K3b.

    coselect=True also fills hist.stats.coselect with the token-level
    co-selection counts (K2b)."""
    h = ids_to_histograms(ids, tokens_per_step, num_experts, check_dropped=False, with_coselect=coselect)
    return statistics_from_histograms(h, correlation=correlation, classify=classify, config=config)


def finalize_statistics(h: Histograms, correlation: bool = True, classify: bool = True,
                        config: ClassifyConfig = ClassifyConfig()) -> TraceStatistics:
    """K3 + K3b over statistics whose sums are complete (e.g. after the all-reduce)."""
    ds = h.stats
    mu, af, corr = finalize_stats(ds, with_corr=correlation)
    classes = classify_device(ds.colsum, ds.heavy, ds.gram, ds.num_steps, config) if classify else None
    return TraceStatistics(h, ds.gram, mu, af, corr, classes)


@_device.nvtx("gem.K2-K3b statistics")
def statistics_from_histograms(h: Histograms, correlation: bool = True, classify: bool = True,
                               config: ClassifyConfig = ClassifyConfig()) -> TraceStatistics:
    compute_gram(h)
    return finalize_statistics(h, correlation=correlation, classify=classify, config=config)


def compute_gram(h: Histograms) -> torch.Tensor:
    """K2 into the statistics buffer (allocating the Gram there if it has none)."""
    ds = h.stats
    if ds.gram is None:
        ds.gram = _device.zeros((h.num_layers, h.num_experts, h.num_experts), torch.int64)
    return step_coactivation(h.hist, ds.gram, max_count=h.max_count)
