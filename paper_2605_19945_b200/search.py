"""GEM-Place: greedy init, best-swap refinement, K restarts
(reference: /root/reference/pkg/src/gemap/search.py).

All restarts of all layers run together on the device (gem_search_runs): one
greedy CTA per run, then refinement rounds in which every still-active run is
scanned (one CTA per run x GPU pair) and updated. The host only draws the
restart noise with numpy's PCG64 (the same generator and call order as the
reference, search.py:187-193,286), seeds the linear/EPLB runs, and picks the
winner by strictly-lower score in job order (search.py:302-305). Results are
bit-identical to the reference, trajectories included.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from ._device import ptr, stream
from ._util import serial_sum
from .baselines import eplb_assignment, eplb_assignments, linear_assignment
from .errors import ValidationError
from .mapping import ExpertMapping, _check_dimensions
from .profiles import VariabilityProfile
from .trace import ExpertTrace, TraceStats, device_stats, finalize_stats

DEFAULT_RESTARTS = 30
DEFAULT_NOISE_FRACTION = 0.20
DEFAULT_CONVERGENCE_THRESHOLD = 0.001
MAX_SWAPS_PER_EXPERT = 10


@dataclass(frozen=True)
class SearchConfig:
    restarts: int = DEFAULT_RESTARTS
    noise_fraction: float = DEFAULT_NOISE_FRACTION
    convergence_threshold: float = DEFAULT_CONVERGENCE_THRESHOLD
    rng_seed: int = 0
    seed_with_baselines: bool = True
    max_swaps_per_restart: int | None = None

    def __post_init__(self):
        if self.restarts < 1:
            raise ValidationError("restarts must be >= 1")
        if self.noise_fraction < 0.0:
            raise ValidationError("noise_fraction must be >= 0")
        if not 0.0 < self.convergence_threshold < 1.0:
            raise ValidationError("convergence_threshold must be in (0, 1)")
        if self.rng_seed < 0:
            raise ValidationError("rng_seed must be non-negative")
        if self.max_swaps_per_restart is not None and self.max_swaps_per_restart < 1:
            raise ValidationError("max_swaps_per_restart must be >= 1")

    def swap_cap(self, num_experts: int) -> int:
        if self.max_swaps_per_restart is not None:
            return self.max_swaps_per_restart
        return MAX_SWAPS_PER_EXPERT * num_experts


@dataclass(frozen=True)
class RestartRecord:
    provenance: str
    initial_score: float
    final_score: float
    swap_count: int
    trajectory: tuple[float, ...]

    def to_dict(self) -> dict:
        return {
            "provenance": self.provenance,
            "initial_score": self.initial_score,
            "final_score": self.final_score,
            "swap_count": self.swap_count,
        }


@dataclass(frozen=True)
class SearchResult:
    best_mapping: ExpertMapping
    best_score: float
    per_restart: tuple[RestartRecord, ...]
    provenance: str

    def to_dict(self) -> dict:
        return {
            "best_score": self.best_score,
            "provenance": self.provenance,
            "best_mapping": self.best_mapping.to_dict(),
            "per_restart": [r.to_dict() for r in self.per_restart],
        }


# ---------------------------------------------------------------------------
# host-side job preparation


class _Instance:
    """Packed profile arrays and per-step loads of one (trace, profile) pair, in
    the layout of the kernel-backend protocol (/root/reference/pkg/src/gemap/search.py:98-131).

    The protocol's callers (the reference's own tests, third-party drivers of
    `kernels.get_backend(...)`) build their arguments with this; the device
    search does not use it. Loads come from the device replay (gem_replay),
    latencies from the backend the caller passes."""

    def __init__(self, trace: ExpertTrace, profile: VariabilityProfile):
        self.tokens = np.ascontiguousarray(trace.tokens, dtype=np.int64)
        self.num_steps, self.num_experts = self.tokens.shape
        self.num_gpus = profile.num_gpus
        _check_divisible(self.num_experts, self.num_gpus)
        self.capacity = self.num_experts // self.num_gpus
        self._trace, self._profile = trace, profile
        sizes = [c.num_samples for c in profile.curves]
        self.offsets = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
        self.xs_flat = np.concatenate([c.token_counts for c in profile.curves]).astype(np.int64)
        self.ys_flat = np.concatenate([c.latencies for c in profile.curves]).astype(np.float64)
        self.dense_limits = np.asarray([c.dense_limit for c in profile.curves], dtype=np.int64)
        for a in (self.tokens, self.offsets, self.xs_flat, self.ys_flat, self.dense_limits):
            a.setflags(write=False)

    def curve_args(self) -> tuple:
        return (self.xs_flat, self.ys_flat, self.offsets, self.dense_limits)

    def eval_gpu(self, backend, gpu: int, counts) -> np.ndarray:
        return backend.eval_curve_packed(*self.curve_args(), gpu, counts)

    def load_matrix(self, assignment: np.ndarray) -> np.ndarray:
        """[T, G] int64 tokens per GPU per step (device replay)."""
        from .mapping import replay_loads
        return replay_loads(self._trace, ExpertMapping(np.asarray(assignment, dtype=np.int64), self.num_gpus))

    def latency_matrix(self, backend, loads: np.ndarray) -> np.ndarray:
        lat = np.empty(loads.shape, dtype=np.float64)
        for g in range(self.num_gpus):
            lat[:, g] = self.eval_gpu(backend, g, loads[:, g])
        return lat


def _restart_order(mean_util: np.ndarray, restart_index: int, rng: np.random.Generator,
                   noise_fraction: float) -> np.ndarray:
    keys = np.asarray(mean_util, dtype=np.float64)
    if restart_index > 0:
        eta = rng.uniform(-1.0, 1.0, keys.shape[0])
        keys = keys * (1.0 + noise_fraction * eta)
    return np.lexsort((np.arange(keys.shape[0]), -keys))  # descending key, ascending index on ties


def _thread_count(threads: int | None) -> int:
    """Validates `threads` / GEM_THREADS like the reference (search.py:242-253).
    The device search is independent of it, as the reference's result is."""
    if threads is None:
        raw = os.environ.get("GEM_THREADS", "0")
        try:
            threads = int(raw)
        except ValueError:
            raise ValidationError(f"GEM_THREADS must be an integer, got {raw!r}") from None
    if threads < 0:
        raise ValidationError("thread count must be >= 0")
    return threads or (os.cpu_count() or 1)


def _check_divisible(num_experts: int, num_gpus: int) -> None:
    if num_experts % num_gpus != 0:
        raise ValidationError(f"{num_experts} experts cannot be split evenly across {num_gpus} GPUs")


@dataclass
class RunBatch:
    """Device inputs for a batch of search runs."""

    run_layer: np.ndarray     # [R] int32
    needs_greedy: np.ndarray  # [R] uint8
    order: np.ndarray | None  # [R, E] int16 (greedy expert order; ignored for seeded runs)
    assign: np.ndarray        # [R, E] int8  (seed mapping; output for greedy runs)
    provenance: list[str]
    keys: np.ndarray | None = None  # [R, E] f64 order keys, sorted on the device when order is None


def layer_jobs(mean_util: np.ndarray, num_gpus: int, config: SearchConfig, layer: int) -> RunBatch:
    """The reference's job list for one layer (search.py:276-287): greedy:0..K-1
    (noise from default_rng(seed ^ i)), then the linear and EPLB seeds."""
    E = mean_util.shape[0]
    orders, assigns, greedy, prov = [], [], [], []
    for i in range(config.restarts):
        rng = np.random.default_rng(config.rng_seed ^ i)
        orders.append(_restart_order(mean_util, i, rng, config.noise_fraction))
        assigns.append(np.zeros(E, dtype=np.int64))
        greedy.append(1)
        prov.append(f"greedy:{i}")
    if config.seed_with_baselines:
        for name, asg in (("baseline:linear", linear_assignment(E, num_gpus)),
                          ("baseline:eplb", eplb_assignment(mean_util, num_gpus))):
            orders.append(np.arange(E))
            assigns.append(asg)
            greedy.append(0)
            prov.append(name)
    R = len(prov)
    return RunBatch(np.full(R, layer, dtype=np.int32), np.asarray(greedy, dtype=np.uint8),
                    np.asarray(orders, dtype=np.int16), np.asarray(assigns, dtype=np.int8), prov)


def all_layer_jobs(mean_util: np.ndarray, num_gpus: int, config: SearchConfig,
                   device_order: bool = False) -> RunBatch:
    """layer_jobs for every layer of mean_util [L, E] at once, in the same run
    order. The restart noise comes from default_rng(seed ^ i) -- the same draw
    for every layer -- so it is drawn once per restart; the keys are the same
    fp64 products and a stable argsort of -key is the reference's lexsort
    (descending key, ascending expert index on ties). device_order: leave the
    sort to gem_restart_order (run_search_device) and ship the keys."""
    mu = np.asarray(mean_util, dtype=np.float64)
    L, E = mu.shape
    K = config.restarts
    nb = 2 if config.seed_with_baselines else 0
    per = K + nb
    keys_all = np.zeros((L, per, E))  # seeded runs: all-equal keys, identity order (unused)
    assign = np.zeros((L, per, E), dtype=np.int8)
    for i in range(K):
        keys = mu
        if i > 0:
            eta = np.random.default_rng(config.rng_seed ^ i).uniform(-1.0, 1.0, E)
            keys = mu * (1.0 + config.noise_fraction * eta)
        keys_all[:, i] = keys
    order = None
    if not device_order:
        order = np.empty((L, per, E), dtype=np.int16)
        order[:, :K] = np.argsort(-keys_all[:, :K], axis=2, kind="stable")
        order[:, K:] = np.arange(E, dtype=np.int16)
        order = order.reshape(L * per, E)
    prov = [f"greedy:{i}" for i in range(K)]
    if nb:
        assign[:, K] = linear_assignment(E, num_gpus)
        assign[:, K + 1] = eplb_assignments(mu, num_gpus)
        prov += ["baseline:linear", "baseline:eplb"]
    greedy = np.zeros(per, dtype=np.uint8)
    greedy[:K] = 1
    return RunBatch(np.repeat(np.arange(L, dtype=np.int32), per), np.tile(greedy, L), order,
                    assign.reshape(L * per, E), prov * L, keys=keys_all.reshape(L * per, E))


def concat_batches(batches: list[RunBatch]) -> RunBatch:
    return RunBatch(np.concatenate([b.run_layer for b in batches]),
                    np.concatenate([b.needs_greedy for b in batches]),
                    np.concatenate([b.order for b in batches]),
                    np.concatenate([b.assign for b in batches]),
                    [p for b in batches for p in b.provenance])


@dataclass
class RunResults:
    assign: np.ndarray        # [R, E] int64
    final_score: np.ndarray   # [R] fp64
    swaps: np.ndarray         # [R] int32
    trajectory: np.ndarray    # [R, max swaps + 1] fp64 (columns past a run's swaps are unused)

    def record(self, r: int, provenance: str) -> RestartRecord:
        if "_lists" not in self.__dict__:  # python floats/ints of every run, converted once
            width = int(self.swaps.max(initial=0)) + 1
            self._lists = (self.trajectory[:, :width].tolist(), self.final_score.tolist(), self.swaps.tolist())
        trajs, finals, swaps = self._lists
        s = swaps[r]
        traj = tuple(trajs[r][: s + 1])
        return RestartRecord(provenance, traj[0], finals[r], s, traj)


TRAJ_INITIAL_WIDTH = 256  # trajectory columns allocated up front (runs measured: <= 16 swaps at C4)


@_device.nvtx("gem.K6-K8 search runs")
def run_search_device(hist: torch.Tensor, nmax: int, profile: VariabilityProfile, batch: RunBatch,
                      threshold: float, swap_cap: int) -> RunResults:
    """Run greedy + refinement for every run of `batch` on the device."""
    L, T, E = hist.shape
    G = profile.num_gpus
    if G > 127:
        # assignments are int8 on the device (the reference takes any G; 127 GPUs per mapping here)
        raise ValidationError(f"the device search supports at most 127 GPUs per mapping, got {G}")
    _check_divisible(E, G)
    R = len(batch.provenance)
    dc = _device.DeviceCurves.from_profile(profile)
    lut = dc.lut(nmax)
    traj_cap = swap_cap + 1
    run_layer = _device.upload(batch.run_layer, torch.int32)
    needs = _device.upload(batch.needs_greedy, torch.uint8)
    if batch.order is None:  # restart orders sorted on the device from the host-drawn keys
        keys = _device.upload(batch.keys, torch.float64)
        order = _device.empty((R, E), torch.int16)
        _lib.call("gem_restart_order", ptr(keys), R, E, ptr(order), stream())
    else:
        order = _device.upload(batch.order, torch.int16)
    assign0 = _device.upload(batch.assign, torch.int8)
    swaps = _device.zeros((R,), torch.int32)
    final = _device.empty((R,), torch.float64)
    ws_bytes = int(_lib.lib().gem_search_workspace_bytes(R, T, E, G))
    ws = _device.empty((max(ws_bytes, 1),), torch.uint8)
    # swap_cap only bounds the loop (search.py:56-59, possibly "unlimited"); the
    # trajectory buffer starts at a bounded width and, in the rare case a run
    # outgrows it, the (deterministic) search is repeated at the exact width
    width_cap = min(traj_cap, TRAJ_INITIAL_WIDTH)
    while True:
        assign = assign0.clone()
        traj = _device.zeros((R, width_cap), torch.float64)
        _lib.call("gem_search_runs", ptr(hist), L, T, E, G, ptr(lut), dc.lut_nmax, R, ptr(run_layer), ptr(needs),
                  ptr(order), ptr(assign), float(threshold), int(swap_cap), int(width_cap), ptr(traj), ptr(swaps),
                  ptr(final), ptr(ws), ws_bytes, stream())
        swaps_h = _device.host(swaps)
        width = int(swaps_h.max(initial=0)) + 1  # only the used trajectory columns cross PCIe
        if width <= width_cap:
            break
        width_cap = width
    return RunResults(_device.host(assign).astype(np.int64), _device.host(final), swaps_h,
                      _device.host(traj[:, :width].contiguous()))


def _pick_best(final_scores, lo: int, hi: int) -> int:
    best = lo
    for k in range(lo + 1, hi):
        if final_scores[k] < final_scores[best]:
            best = k
    return best


# ---------------------------------------------------------------------------
# public API


def initial_mapping(stats: TraceStats, restart_index: int, trace: ExpertTrace, profile: VariabilityProfile,
                    rng: np.random.Generator, noise_fraction: float = DEFAULT_NOISE_FRACTION) -> ExpertMapping:
    """Greedy utilization-ordered seed mapping for one restart (search.py:167-184)."""
    _check_divisible(trace.num_experts, profile.num_gpus)
    order = _restart_order(stats.mean_utilization, restart_index, rng, noise_fraction)
    E = trace.num_experts
    batch = RunBatch(np.zeros(1, dtype=np.int32), np.ones(1, dtype=np.uint8), order[None].astype(np.int16),
                     np.zeros((1, E), dtype=np.int8), [f"greedy:{restart_index}"])
    hist, nmax = trace.device_counts()
    res = run_search_device(hist.view(1, *hist.shape), nmax, profile, batch, DEFAULT_CONVERGENCE_THRESHOLD, 0)
    return ExpertMapping(res.assign[0], profile.num_gpus)


def refine(mapping: ExpertMapping, trace: ExpertTrace, profile: VariabilityProfile,
           config: SearchConfig) -> tuple[ExpertMapping, int]:
    """Best-swap refinement until convergence; returns (mapping, swap count)."""
    _check_dimensions(trace, profile, mapping)
    _check_divisible(trace.num_experts, profile.num_gpus)
    E = trace.num_experts
    batch = RunBatch(np.zeros(1, dtype=np.int32), np.zeros(1, dtype=np.uint8), np.arange(E)[None].astype(np.int16),
                     mapping.assignment[None].astype(np.int8), ["refine"])
    hist, nmax = trace.device_counts()
    res = run_search_device(hist.view(1, *hist.shape), nmax, profile, batch, config.convergence_threshold,
                            config.swap_cap(E))
    return ExpertMapping(res.assign[0], profile.num_gpus), int(res.swaps[0])


def search(trace: ExpertTrace, profile: VariabilityProfile, config: SearchConfig | None = None,
           threads: int | None = None) -> SearchResult:
    """All restarts plus the baseline-seeded refinements; keep the best (search.py:256-312)."""
    if config is None:
        config = SearchConfig()
    _thread_count(threads)
    _check_divisible(trace.num_experts, profile.num_gpus)
    return search_layers([trace], profile, config)[0]


def search_layers(traces, profile: VariabilityProfile, config: SearchConfig | None = None) -> list[SearchResult]:
    """Independent per-layer searches with the same config and seed (the CLI's
    multi-layer loop, cli.py:412-416), all layers' runs batched into one device job."""
    if config is None:
        config = SearchConfig()
    traces = list(traces)
    if not traces:
        return []
    for tr in traces:
        _check_divisible(tr.num_experts, profile.num_gpus)
    # layers of equal (num_steps, num_experts) share one batched device job;
    # mixed shapes (e.g. CSV layers whose last step is all zeros) form several
    groups: dict[tuple[int, int], list[int]] = {}
    for i, tr in enumerate(traces):
        groups.setdefault(tr.tokens.shape, []).append(i)
    out: list[SearchResult | None] = [None] * len(traces)
    for members in groups.values():
        stacked = np.stack([traces[i].tokens for i in members])
        hist, nmax = _device.counts_to_device_int32(stacked)
        for i, res in zip(members, search_hist(hist, nmax, profile, config)):
            out[i] = res
    return out


@_device.nvtx("gem.search_hist")
def search_hist(hist: torch.Tensor, nmax: int, profile: VariabilityProfile, config: SearchConfig,
                mean_util: np.ndarray | None = None) -> list[SearchResult]:
    """Search every layer of a device histogram [L,T,E] int32."""
    L, T, E = hist.shape
    G = profile.num_gpus
    _check_divisible(E, G)
    if mean_util is None:
        ds = device_stats(hist, with_gram=False)
        mu_dev, _, _ = finalize_stats(ds, with_corr=False)
        mean_util = _device.host(mu_dev)
    batch = all_layer_jobs(np.asarray(mean_util).reshape(L, E), G, config, device_order=True)
    res = run_search_device(hist, nmax, profile, batch, config.convergence_threshold, config.swap_cap(E))
    out = []
    per = len(batch.provenance) // L
    for l in range(L):
        lo, hi = l * per, (l + 1) * per
        best = _pick_best(res.final_score, lo, hi)
        records = tuple(res.record(r, batch.provenance[r]) for r in range(lo, hi))
        out.append(SearchResult(best_mapping=ExpertMapping(res.assign[best], G),
                                best_score=float(res.final_score[best]), per_restart=records,
                                provenance=batch.provenance[best]))
    return out


def aggregate_score(results: list[SearchResult]) -> float:
    """Multi-layer aggregate: serial fp64 sum in layer order (cli.py:427)."""
    return serial_sum(r.best_score for r in results)
