"""GEM data-parallel core benchmark (BASELINE.json: Qwen3-235B-shaped trace).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

One timed step = the statistics phase over the whole synthetic router trace
(94 layers x 2^24 tokens x top-8 int16 ids, 25.2 GB resident in HBM):
K1 ids->histograms, K2 step co-activation Gram, K3 stats finalize, K3b classes.
`value` = trace tokens/s (whole job). Secondary numbers on the same line:
candidate mappings/s (10k candidate [94,128] mappings scored on the full
trace) and time-to-mapping (statistics + GEM-Place search of all 94 layers on
all 16,384 steps, 32 runs per layer). Multi-GPU: token-range shards, one NCCL
all-reduce of the exact integer statistics (colsum, active counts, Gram).
Inputs exceed L2 (126 MB) by 200x, so no explicit L2 flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "trace tokens/s (stats) + candidate mappings/s; time-to-mapping, Qwen3-235B"

CONFIGS = {
    # name: (L, N, k, E, B, G, C)
    "mixtral": (32, 65536, 2, 8, 1024, 8, 10000),
    "olmoe": (16, 1 << 20, 8, 64, 1024, 8, 10000),
    "qwen3-30b": (48, 1 << 22, 8, 128, 1024, 8, 10000),
    "qwen3-235b": (94, 1 << 24, 8, 128, 1024, 8, 10000),
    "deepseek-v3": (58, 1 << 24, 8, 256, 1024, 32, 10000),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="qwen3-235b", choices=sorted(CONFIGS))
    ap.add_argument("--candidates", type=int, default=None, help="override C (candidate mappings)")
    ap.add_argument("--no-search", action="store_true", help="skip the time-to-mapping leg")
    ap.add_argument("--no-candidates", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-coselect", action="store_true", help="skip the K2b co-selection leg")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--search-steps", type=int, default=None, help="search window (default: all steps)")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo: functional check of the N>1 code path with several ranks on one GPU "
                         "(collectives staged through host memory; not a performance number)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the sharded (torch.distributed) code path even on one GPU")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region by an
    `nvidia-smi -lms` child process (a separate process: a sampling thread in
    this interpreter would take the GIL from the launch loop and open host gaps
    between kernels). The first sample is awaited before the timed region starts."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, period_ms: int = 5):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.path = None
        self.samples = []  # (sm_mhz, max_mhz, [active reason names])

    def _gpu_id(self) -> str:
        try:
            import torch

            u = str(torch.cuda.get_device_properties(self.index).uuid)
            return u if u.startswith("GPU-") else "GPU-" + u
        except Exception:
            return str(self.index)

    def _lines(self):
        try:
            return [ln for ln in Path(self.path).read_text().splitlines() if ln.strip()]
        except OSError:
            return []

    def __enter__(self):
        import tempfile

        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self._gpu_id(), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t_end = time.time() + 10.0
            while time.time() < t_end and not self._lines() and self.proc.poll() is None:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        for ln in self._lines():
            f = [x.strip() for x in ln.split(",")]
            try:
                self.samples.append((float(f[0]), float(f[1]),
                                     [n for n, v in zip(self.NAMES, f[2:6]) if v.lower() == "active"]))
            except (ValueError, IndexError):
                continue
        try:
            os.unlink(self.path)
        except OSError:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0,
                    "source": "nvidia-smi -lms"}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvidia-smi -lms %d (child process)" % self.period_ms}


# ---------------------------------------------------------------------------


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def tensor_peaks():
    """int8 / fp16 / fp64 GEMM peaks measured on a B200 of this pool by tools/peaks.py (cuBLAS)."""
    p = ROOT / "profiles" / "r02_peaks.json"
    try:
        return json.loads(p.read_text())
    except (OSError, ValueError):
        return {}


def ncu_traffic():
    """dram bytes/launch of the dominant kernel from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "ncu_topk_hist.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_19945_b200 as gem
    from paper_2605_19945_b200 import _device, _lib, ingest
    from paper_2605_19945_b200 import dist as dist_mod
    from paper_2605_19945_b200 import mapping as gm
    from paper_2605_19945_b200.search import aggregate_score, search_hist
    from paper_2605_19945_b200.trace import DeviceStats, finalize_stats

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % max(torch.cuda.device_count(), 1)  # gloo check: several ranks may share a GPU
    torch.cuda.set_device(dev)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev), rank=rank, world_size=world)
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
    L, N, k, E, B, G, C = CONFIGS[args.config]
    if args.candidates:
        C = args.candidates
    T = N // B
    # planted structure: 3 consistent experts + 2 temporal pairs; Mixtral's 8 experts (top-2) leave room
    # for 2 consistent + 1 pair next to the top_k always-on background experts
    planted = {} if E >= 16 else {"consistent": 2, "num_groups": 1}
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=0,
                                **planted)
    # token-range shard of this rank (step aligned)
    steps_per = -(-T // world)
    t0, t1 = rank * steps_per, min(T, (rank + 1) * steps_per)
    n_local = (t1 - t0) * B
    ids = ingest.generate_topk_ids(spec, dtype=torch.int16, token_offset=t0 * B, num_tokens=n_local)
    hist = torch.empty((L, t1 - t0, E), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    kev = []  # (start, end) events around K1 per timed step

    phases = ("K1 topk_hist", "K2 step_gram", "all-reduce", "K3 finalize", "K3b classify")
    pev = []  # per timed step: events bracketing each phase

    # steady-state buffers, allocated once (a serving loop reuses them; no
    # allocator traffic inside the timed region)
    ds = DeviceStats.allocate(L, E, T)  # colsum/active/heavy/Gram: one int64 buffer, one all-reduce
    dropped = torch.zeros((L,), dtype=torch.int64, device="cuda")
    st_out = (torch.empty((L, E), dtype=torch.float64, device="cuda"),
              torch.empty((L, E), dtype=torch.float64, device="cuda"),
              torch.empty((L, E, E), dtype=torch.float64, device="cuda"))
    cls_out = ingest.ExpertClasses(torch.empty((L, E), dtype=torch.int8, device="cuda"),
                                   torch.empty((L, E), dtype=torch.int16, device="cuda"),
                                   torch.zeros((1,), dtype=torch.int32, device="cuda"))

    def stats_step(timed: bool):
        ds.pack.zero_()
        dropped.zero_()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(phases) + 1)] if timed else None

        def mark(i):
            if timed:
                evs[i].record(stream)

        torch.cuda.nvtx.range_push("bench.stats_step")
        mark(0)
        _lib.call("gem_topk_hist", ids.data_ptr(), 2, L, n_local, k, B, E, hist.data_ptr(), ds.colsum.data_ptr(),
                  ds.active.data_ptr(), ds.heavy.data_ptr(), dropped.data_ptr(), stream.cuda_stream)
        mark(1)
        _lib.call("gem_step_gram", hist.data_ptr(), L, t1 - t0, E, B * k, ds.gram.data_ptr(), stream.cuda_stream)
        mark(2)
        if use_dist:
            dist.all_reduce(ds.pack)
        mark(3)
        mu, af, corr = finalize_stats(ds, with_corr=True, out=st_out)
        mark(4)
        cls = ingest.classify_device(ds.colsum, ds.heavy, ds.gram, T, out=cls_out)
        mark(5)
        torch.cuda.nvtx.range_pop()
        if timed:
            kev.append((evs[0], evs[1]))
            pev.append(evs)
        return mu, af, corr, cls

    for _ in range(args.warmup):
        stats_step(False)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            out = stats_step(True)
        ev1.record(stream)
        torch.cuda.synchronize()
    out[3].check()  # K3b's asynchronous range flag (checked outside the timed region)
    ms = ev0.elapsed_time(ev1) / args.steps
    if use_dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    k1_ms = sum(a.elapsed_time(b) for a, b in kev) / len(kev)
    tokens_per_s = N / (ms / 1e3)
    result = {
        "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int16 ids / int32+int64 counts / f64 stats", "data": "synthetic",
        "config": {"workload": f"{args.config}: stats phase over the full router trace", "layers": L,
                   "tokens": N, "top_k": k, "experts": E, "tokens_per_step": B, "steps_per_layer": T,
                   "virtual_gpus": G, "id_dtype": "int16", "l2": "inputs 25 GB >> 126 MB L2 (no flush needed)",
                   "parallelism": f"token-range shards x{world}, NCCL all-reduce of integer stats"},
        # K1 (+ its heavy-row pass above 160 experts), K2, K3, K3b
        "gpu_launches": (4 + (E > 160)) * args.steps,
        "step_breakdown_ms": {name: sum(e[i].elapsed_time(e[i + 1]) for e in pev) / len(pev)
                              for i, name in enumerate(phases)},
        "clocks": clk.summary(),
    }
    # roofline of the dominant kernel (K1 = gem_topk_hist): ids read + histogram
    # rows written; above 160 experts (the CTA kernel) + the heavy-step pass's
    # re-read of the rows (the ring kernel counts heavy steps in its reduction)
    hist_passes = 1 if E <= 160 else 2
    algo_bytes = L * n_local * k * 2 + hist_passes * L * (t1 - t0) * E * 4
    k1_name = ("topk_hist_ring_kernel (K1, heavy steps counted in its reduction)" if E <= 160 else
               "gem_topk_hist (K1: topk_hist_creg_kernel + hist_heavy_rows_kernel)")
    peak, peak_src = peaks()
    achieved = algo_bytes / (k1_ms / 1e3) / 1e9
    result["roofline"] = {"kernel": k1_name,
                          "bound": "hbm", "achieved": achieved, "peak": peak,
                          "unit": "GB/s", "frac": achieved / peak, "traffic": ncu_traffic() if args.config == "qwen3-235b" and world == 1 else None,
                          "algorithmic_bytes_per_launch": algo_bytes, "kernel_ms": k1_ms,
                          "kernel_share_of_step": k1_ms / ms, "peak_source": peak_src}

    # ---- K2b token-level co-selection counts of this rank's token shard (an
    #      optional statistics output, timed on its own): tcgen05 kind::i8 OᵀO
    if not args.no_coselect:
        cs = torch.zeros((L, E, E), dtype=torch.int32, device="cuda")

        def cs_step():
            cs.zero_()
            ingest.token_coselection(ids, E, out=cs)

        cs_step()
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, min(3, args.steps))
        c0.record(stream)
        for _ in range(reps):
            cs_step()
        c1.record(stream)
        torch.cuda.synchronize()
        cs_t = torch.tensor([c0.elapsed_time(c1) / reps], device="cuda")
        if use_dist:
            dist.all_reduce(cs_t, op=dist.ReduceOp.MAX)
        cs_ms = float(cs_t.item())
        useful = 2 * L * N * E * E  # int8 MACs x2 of the one-hot OᵀO (unpadded E)
        tp = tensor_peaks()
        result["coselection"] = {
            "value": N / (cs_ms / 1e3), "unit": "tokens/s", "ms": cs_ms,
            "path": ingest.coselection_path(ids, E),
            "roofline": {"kernel": "coselect_tc_kernel (K2b)", "bound": "tensor", "achieved": useful / cs_ms / 1e9,
                         "peak": tp.get("int8_tops"), "unit": "TOPS",
                         "frac": (useful / cs_ms / 1e9 / tp["int8_tops"]) if tp.get("int8_tops") else None,
                         "peak_source": "profiles/r02_peaks.json (cuBLAS int8 GEMM, 8192^3)" if tp else None,
                         "note": "shared-memory bound in practice: SS-mode MMA operand reads + one-hot build; "
                                 "see DESIGN.md K2b"},
            # built-in check (outside the timed region): diag(OᵀO) == K1's per-expert token totals
            "diag_equals_colsum": bool(torch.equal(torch.diagonal(cs, dim1=1, dim2=2).long(),
                                                   hist.sum(dim=1, dtype=torch.int64)))}
        del cs

    plan = dist_mod.ShardPlan(world, rank, L, T)
    ops = dist_mod.DeviceOps()

    # ---- e2e through the public API with host (pinned) ids: every step copies
    #      this rank's id shard host->device and reads the per-expert results back
    if not args.no_e2e:
        host_ids = torch.empty(ids.shape, dtype=ids.dtype, pin_memory=True)
        host_ids.copy_(ids)
        dev_ids = torch.empty_like(ids)
        torch.cuda.synchronize()

        def e2e_step():
            torch.cuda.nvtx.range_push("bench.e2e_step")
            dev_ids.copy_(host_ids, non_blocking=True)
            if use_dist:
                ss = dist_mod.sharded_statistics(dev_ids, plan, ops, B, E)
                mu, cls = ss.finalized[0], ss.finalized[3]
            else:
                st = ingest.trace_statistics(dev_ids, B, E)
                mu, cls = st.mean_utilization, st.classes.cls
                st.check()
            # the whole TraceStats back to the host: utilisation, active fraction, Pearson, classes
            if use_dist:
                outs = (ss.finalized[0], ss.finalized[1], ss.finalized[2], ss.finalized[3])
            else:
                outs = (st.mean_utilization, st.active_fraction, st.correlation, st.classes.cls)
            res = tuple(t.to("cpu", non_blocking=True) for t in outs if t is not None)
            torch.cuda.current_stream().synchronize()
            torch.cuda.nvtx.range_pop()
            return res

        e2e_step()
        reps = max(1, min(3, args.steps))
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(reps):
            e2e_step()
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = torch.tensor([a0.elapsed_time(a1) / reps], device="cuda")
        if use_dist:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_ms.item()) / 1e3
        result["e2e"] = {"value": N / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": int(ids.numel() * 2),
                         "d2h_bytes_per_step": int(2 * L * E * 8 + L * E * E * 8 + L * E), "ms_per_step": e2e_s * 1e3,
                         "bytes_are": "per rank" if use_dist else "whole job",
                         "path": ("dist.sharded_statistics" if use_dist else "ingest.trace_statistics")
                         + "(ids copied from pinned host memory every step)"}
        del host_ids, dev_ids

    # ---- candidate mappings/s (C candidates x all layers, full trace) and
    #      time-to-mapping (stats + GEM-Place search of every layer, full trace).
    #      Multi-GPU: histogram rows go to the layer owners (one all-to-all),
    #      layers are searched / scored where they live, results all-gathered.
    profile = gem.generate_profile(gem.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64,
                                                            max_tokens=B * k, rng_seed=0))

    def owned_hist():
        return dist_mod.exchange_hist(hist, plan) if use_dist else hist

    def dev_time(fn):
        """CUDA-event time of fn() on this rank, max over ranks (ms)."""
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = fn()
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], device="cuda")
        if use_dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return out, float(t.item())

    if not args.no_candidates:
        rng = np.random.default_rng(0)
        base = np.repeat(np.arange(G, dtype=np.int8), E // G)
        cand = rng.permuted(np.broadcast_to(base, (C * L, E)), axis=1).reshape(C, L, E)
        cand_d = torch.from_numpy(np.ascontiguousarray(cand)).cuda()
        nmax = B * k
        c0, c1 = plan.candidate_range(C)

        def score_all():
            # N>1: candidates split by index; every rank needs every layer's
            # full-length rows (one all-gather of the token-range shards, timed)
            if use_dist:
                hist_full = dist_mod.allgather_hist(hist, plan)
                return dist_mod.sharded_candidate_scores(hist_full, plan, ops, profile, cand_d, nmax)
            return gm.score_candidates_device(hist, nmax, profile, cand_d)

        score_all()  # warm-up (LUT build, module load)
        torch.cuda.nvtx.range_push("bench.candidates")
        (total, _), cms = dev_time(score_all)
        torch.cuda.nvtx.range_pop()
        best = int(torch.argmin(total).item())
        result["candidates"] = {"value": C / (cms / 1e3), "unit": "candidate mappings/s", "ms": cms,
                                "candidates": C, "layers": L, "steps": T, "best_index": best,
                                "best_score": float(total[best].item()),
                                "sharding": f"candidates {c0}..{c1 - 1} on this rank of {world} (all-gather of "
                                            f"the histogram shards + one all-gather of the scores, timed)"
                                if use_dist else "single GPU"}
        # K5 roofline (tensor): the one-hot load GEMM's useful int8 ops --
        # 2 x T steps x (C x G) columns x 2E K bytes (u8 limbs) per layer --
        # over the whole scoring time; the leg is bound by the key gathers
        # (C*L*T*G random shared-memory loads), which DESIGN.md §4 sizes
        tp = tensor_peaks()
        mma_ops = 2.0 * T * (C // world if use_dist else C) * G * 2 * E * L
        if tp.get("int8_tops"):
            ach = mma_ops / (cms / 1e3) / 1e12
            result["candidates"]["roofline"] = {
                "kernel": "maxkey_tc_kernel (K5, tcgen05 kind::i8) + keysum_kernel", "bound": "tensor",
                "achieved": ach, "peak": tp["int8_tops"], "unit": "TOPS", "frac": ach / tp["int8_tops"],
                "peak_source": "profiles/r02_peaks.json (cuBLAS int8 GEMM)",
                "note": "the MMA is a minor share: the leg is bound by C*L*T*G shared-memory key gathers "
                        "(floor ~34 ms at C4, DESIGN.md K5 bound)"}
        del cand_d

    if not args.no_search:
        cfg = gem.SearchConfig(rng_seed=0)

        def ttm(Tw):
            st = stats_step(False)
            h = owned_hist()
            if Tw != T:
                h = h[:, :Tw].contiguous()
            if use_dist:
                return dist_mod.sharded_search(h, plan, ops, profile, cfg, B * k), None
            mu = st[0].cpu().numpy() if Tw == T else None
            return None, search_hist(h, B * k, profile, cfg, mean_util=mu)

        def ttm_info(Tw):
            ttm(Tw)  # warm-up: module load, stream-ordered pool growth (~1.5 GB of search scratch), LUT build
            torch.cuda.nvtx.range_push(f"bench.time_to_mapping[{Tw}]")
            (shm, results), tms = dev_time(lambda: ttm(Tw))
            torch.cuda.nvtx.range_pop()
            info = {"value": tms / 1e3, "unit": "s", "steps_searched": Tw, "layers": L,
                    "runs_per_layer": cfg.restarts + 2, "timing": "CUDA events on the launching stream, max over ranks",
                    "includes": "K1..K3b statistics, all-to-all to layer owners (N>1), greedy + refinement of every run"}
            if results is not None:
                swaps = [r.swap_count for res in results for r in res.per_restart]
                info.update({"runs": len(swaps), "swaps_median": float(np.median(swaps)),
                             "swaps_max": int(max(swaps)), "aggregate_score": aggregate_score(results),
                             "layer0_best_score": results[0].best_score})
            else:
                info["aggregate_score"] = shm.aggregate
            return info

        result["time_to_mapping"] = ttm_info(args.search_steps or T)
        result["time_to_mapping"]["roofline_note"] = (
            "dominated by K6 approx_scan5 (random fp32 table gathers in shared memory, ~84% of the shared-memory "
            "wavefront peak per ncu, profiles/r02_ncu_k6.json); no HBM or tensor-pipe bound applies")
        if not args.search_steps and T > 16:  # the paper's 16-step window (the reference arm measures the same)
            w16 = ttm_info(16)
            w16["includes"] = "K1..K3b statistics of the full trace, search of every layer's first 16 steps"
            result["time_to_mapping_w16"] = w16

    if not args.no_cpu and world == 1 and rank == 0:
        try:
            result["cpu_baseline"] = cpu_stats_baseline(spec, ids)
        except Exception as exc:  # the baseline is reported, never required
            result["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU side: reference compute_stats (oracle/_ref, gemap 0.1.0) + a bincount
# restatement of id ingestion (the reference has no id ingestion)


def _cpu_layer(args):
    ids_l, B, E = args
    import numpy as np

    from oracle import oracle as o

    gemap = o.import_reference()
    n = ids_l.shape[0]
    step = (np.arange(n) // B).repeat(ids_l.shape[1])
    T = -(-n // B)
    hist = np.bincount(step * E + ids_l.ravel().astype(np.int64), minlength=T * E).reshape(T, E)
    st = gemap.compute_stats(gemap.ExpertTrace(hist))
    return float(st.mean_utilization[0])


def _single_thread_env():
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"


def cpu_stats_run(ids_np, B, E, cores):
    """Reference statistics for every layer of ids_np [l, n, k], one process per layer -> seconds."""
    from concurrent.futures import ProcessPoolExecutor

    work = [(ids_np[l], B, E) for l in range(ids_np.shape[0])]
    s0 = time.perf_counter()
    if cores > 1:
        with ProcessPoolExecutor(max_workers=cores, initializer=_single_thread_env) as ex:
            list(ex.map(_cpu_layer, work))
    else:
        for w in work:
            _cpu_layer(w)
    return time.perf_counter() - s0


def cpu_stats_baseline(spec, ids_dev):
    """Bounded sample: `cores` layer-slices of 4096 steps (4M tokens) each, one process per core."""
    cores = len(os.sched_getaffinity(0)) or 1  # every host core this process may use
    steps = min(spec.num_steps, 4096)
    n = steps * spec.tokens_per_step
    layers = min(spec.num_layers, cores)
    ids_np = ids_dev[:layers, :n].cpu().numpy()
    secs = cpu_stats_run(ids_np, spec.tokens_per_step, spec.num_experts, layers)
    tokens_equiv = n * layers / spec.num_layers
    return {"value": tokens_equiv / secs, "unit": "tokens/s", "cores": layers, "kind": "reference",
            "sample": f"{layers} layers x {n} tokens ({steps} steps), one process per layer: np.bincount "
                      f"ingestion (restatement; the reference has none) + reference gemap.compute_stats "
                      f"(oracle/_ref Cython build), {secs:.2f} s"}


# ---- the benchmark's own synthetic router trace (K9) for the reference arm,
#      generated on the host by the C oracle (oracle/gem_oracle.c, the exact
#      restatement of gem_gen_topk): the reference arm sees the same ids as ours

def k9_params(config):
    """(weight [L,E] u32, role [L,E] i8, p_cons, p_burst, burst_mult, seed) of bench.CONFIGS[config]:
    the planted layout of ingest.TopkTraceSpec/planted_layout restated in numpy (tests/test_host.py
    pins the equality) so the reference arm never imports this package."""
    import numpy as np

    L, N, k, E, B, G, C = CONFIGS[config]
    zipf_s, seed = 1.1, 0
    consistent, num_groups, group_size = (3, 2, 2) if E >= 16 else (2, 1, 2)
    weight = np.zeros((L, E), dtype=np.uint32)
    role = np.zeros((L, E), dtype=np.int8)
    base = np.maximum(1, np.rint((1 << 20) / np.power(np.arange(E) + 1.0, zipf_s))).astype(np.uint32)
    for l in range(L):
        perm = np.random.default_rng([seed, l]).permutation(E)
        weight[l, perm] = base
        r = 0
        for _ in range(consistent):
            role[l, perm[r]] = 1
            r += 1
        for g in range(num_groups):
            for _ in range(group_size):
                role[l, perm[r]] = 2 + g
                r += 1
    prob = lambda x: min(int(round(x * 4294967296.0)), 0xFFFFFFFF)  # noqa: E731
    return weight, role, prob(0.85), prob(0.17), 3, seed


def _k9_ids(args):
    """ids [n, k] of layer l, global tokens [t0, t0 + n) (C oracle)."""
    config, l, t0, n = args
    from oracle import oracle as o

    L, N, k, E, B, G, C = CONFIGS[config]
    weight, role, pc, pb, bm, seed = k9_params(config)
    return o.gen_topk(1, n, k, B, E, weight[l:l + 1], role[l:l + 1], pc, pb, bm, seed, token_offset=t0,
                      layer_offset=l)[0]


def _hist(ids, B, E):
    import numpy as np

    step = (np.arange(ids.shape[0]) // B).repeat(ids.shape[1])
    T = -(-ids.shape[0] // B)
    return np.bincount(step * E + ids.ravel().astype(np.int64), minlength=T * E).reshape(T, E)


def _ref_stats_layer(args):
    """Generate one layer's sample (untimed), then time the reference statistics on it."""
    config, l, n = args
    from oracle import oracle as o

    L, N, k, E, B, G, C = CONFIGS[config]
    ids = _k9_ids((config, l, 0, n))
    gemap = o.import_reference()
    s0 = time.perf_counter()
    st = gemap.compute_stats(gemap.ExpertTrace(_hist(ids, B, E)))
    secs = time.perf_counter() - s0
    return secs, float(st.mean_utilization[0])


def _ref_profile(gemap, G, nmax):
    return gemap.generate_profile(gemap.VariabilitySetupSpec(num_gpus=G, setup="moderate", tile_size=64,
                                                             max_tokens=nmax, rng_seed=0))


def _cpu_search_layer(args):
    """Reference gemap.search of one layer's window (default config, seed 0: the CLI's multi-layer)."""
    hist, G, nmax = args
    from oracle import oracle as o

    gemap = o.import_reference()
    res = gemap.search(gemap.ExpertTrace(hist), _ref_profile(gemap, G, nmax), gemap.SearchConfig(rng_seed=0),
                       threads=1)
    return res.best_score


def _cpu_score_sample(args):
    """Seconds per reference gemap.score_mapping call on one full-length layer."""
    hist, G, nmax, maps = args
    from oracle import oracle as o

    gemap = o.import_reference()
    prof, tr = _ref_profile(gemap, G, nmax), gemap.ExpertTrace(hist)
    mappings = [gemap.ExpertMapping(m, G) for m in maps]
    gemap.score_mapping(tr, prof, mappings[0])  # first-call overheads
    s0 = time.perf_counter()
    for m in mappings:
        gemap.score_mapping(tr, prof, m)
    return (time.perf_counter() - s0) / len(mappings)


def _cpu_run_units(args):
    """Seconds of one reference greedy placement and one best_swap scan on a full-length layer."""
    hist, G, nmax = args
    import numpy as np

    from oracle import oracle as o

    gemap = o.import_reference()
    import importlib

    kernels = importlib.import_module("gemap.kernels")
    rs = importlib.import_module("gemap.search")  # the module (gemap.search the name is the function)

    inst = rs._Instance(gemap.ExpertTrace(hist), _ref_profile(gemap, G, nmax))
    backend = kernels.active()
    order = np.arange(inst.num_experts)
    s0 = time.perf_counter()
    assignment = rs._greedy_assignment(inst, backend, order)
    t_greedy = time.perf_counter() - s0
    loads = inst.load_matrix(assignment)
    lat = inst.latency_matrix(backend, loads)
    s0 = time.perf_counter()
    backend.best_swap(inst.tokens, assignment, loads, lat, *inst.curve_args())
    return t_greedy, time.perf_counter() - s0


def cpu_search_and_scoring(config, L, k, E, B, G, C, T, cores):
    """The reference's search (16-step window: all L layers measured; full T: one
    layer measured, x L) and candidate scoring (full T, extrapolated from a
    timed sample), on every host core, on the benchmark's own K9 trace."""
    import numpy as np
    from concurrent.futures import ProcessPoolExecutor

    rng = np.random.default_rng(1)
    nmax = B * k
    out = {}
    with ProcessPoolExecutor(max_workers=cores, initializer=_single_thread_env) as ex:
        # every layer's first 16 steps (the window the GPU arm's time_to_mapping_w16 searches)
        w16 = [(_hist(ids, B, E), G, nmax) for ids in ex.map(_k9_ids, [(config, l, 0, 16 * B) for l in range(L)])]
        list(ex.map(_cpu_search_layer, w16[:cores]))  # warm-up: imports in every worker
        s0 = time.perf_counter()
        best = list(ex.map(_cpu_search_layer, w16))
        secs = time.perf_counter() - s0
        agg = 0.0
        for b in best:  # the multi-layer aggregate: serial fp64 sum in layer order (cli.py:427)
            agg = agg + b
        out["time_to_mapping_w16"] = {
            "value": secs, "unit": "s", "steps_searched": 16, "layers": L, "cores": cores, "aggregate_score": agg,
            "sample": f"all {L} layers measured: reference gemap.search (default SearchConfig, seed 0) on every "
                      f"layer's first 16 steps of the benchmark's K9 trace, one process per layer, {cores} "
                      f"processes (statistics of the full trace not included); aggregate_score equals the GPU "
                      f"arm's time_to_mapping_w16.aggregate_score when both compute the same mappings"}
        # layer 0 in full (token ranges generated in parallel)
        chunk = -(-T // cores) * B
        parts = list(ex.map(_k9_ids, [(config, 0, t0, min(chunk, T * B - t0)) for t0 in range(0, T * B, chunk)]))
        full = _hist(np.concatenate(parts), B, E).astype(np.int64)
        base = np.repeat(np.arange(G), E // G)
        per = 2
        work = [(full, G, nmax, [rng.permutation(base) for _ in range(per)]) for _ in range(cores)]
        s0 = time.perf_counter()
        per_call = float(np.median(list(ex.map(_cpu_score_sample, work))))
        wall = time.perf_counter() - s0
        total = C * L * per_call / cores
        units = list(ex.map(_cpu_run_units, [(full, G, nmax)] * cores))
        t_greedy = float(np.median([u[0] for u in units]))
        t_scan = float(np.median([u[1] for u in units]))
        restarts = 30  # SearchConfig default: 30 greedy restarts + 2 baseline seeds, each refined
        lower = L * (restarts * t_greedy + (restarts + 2) * t_scan) / cores
        out["candidates"] = {
            "value": C / total, "unit": "candidate mappings/s", "cores": cores, "kind": "extrapolated",
            "sample": f"{cores * per} reference gemap.score_mapping calls on one {T}-step layer, "
                      f"{per_call * 1e3:.1f} ms each on {cores} processes ({wall:.1f} s); "
                      f"{C} candidates x {L} layers = {C * L} calls / {cores} cores"}
    # one whole layer through the reference's own search (restarts on every
    # core, as GEM_THREADS does), extrapolated to L layers searched one after
    # another (the CLI's multi-layer)
    from oracle import oracle as o

    gemap = o.import_reference()
    s0 = time.perf_counter()
    res = gemap.search(gemap.ExpertTrace(full), _ref_profile(gemap, G, nmax), gemap.SearchConfig(rng_seed=0),
                       threads=cores)
    t_layer = time.perf_counter() - s0
    swaps = [r.swap_count for r in res.per_restart]
    out["time_to_mapping"] = {
        "value": L * t_layer, "unit": "s", "steps_searched": T, "layers": L, "cores": cores,
        "kind": "extrapolated from one measured layer", "layer0_best_score": res.best_score,
        "sample": f"reference gemap.search of one {T}-step layer (default SearchConfig, seed 0, restarts on "
                  f"{cores} threads): {t_layer:.1f} s, swaps per run median {float(np.median(swaps)):.0f} max "
                  f"{max(swaps)}; x {L} layers. Lower bound from unit costs (greedy {t_greedy:.2f} s, best_swap "
                  f"scan {t_scan:.2f} s, every run's final scan only, {cores} cores): {lower:.0f} s"}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as o

    if o.import_reference() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference build) missing"}))
        return
    L, N, k, E, B, G, C = CONFIGS[args.config]
    T = N // B
    # the benchmark's own K9 ids (C oracle on the host), one process per layer:
    # each generates its layer's sample (untimed) and times the reference's
    # bincount ingestion + compute_stats; the layers run concurrently, so the
    # step time is the slowest layer's
    cores = len(os.sched_getaffinity(0)) or 1  # every host core this process may use
    layers = min(L, cores)
    sample_tokens = min(N, 4096 * B)
    from concurrent.futures import ProcessPoolExecutor

    with ProcessPoolExecutor(max_workers=layers, initializer=_single_thread_env) as ex:
        list(ex.map(_ref_stats_layer, [(args.config, l, 16 * B) for l in range(layers)]))  # warm-up: imports
        times = []
        for _ in range(max(1, min(args.steps, 3))):
            times.append(max(t for t, _ in ex.map(_ref_stats_layer, [(args.config, l, sample_tokens)
                                                                      for l in range(layers)])))
    secs = float(np.median(times))
    value = sample_tokens * layers / L / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 1,
        "steps": len(times), "warmup": 1, "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64 counts / f64 stats", "data": "synthetic",
        "config": {"workload": f"{args.config}: stats phase (bounded CPU sample)", "layers": L, "tokens": N,
                   "top_k": k, "experts": E},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": min(cores, layers), "kind": "reference",
                         "sample": f"{layers} layers x {sample_tokens} tokens of the benchmark's own K9 trace "
                                   "(generated by the C oracle, untimed); np.bincount ingestion restatement + "
                                   "reference gemap.compute_stats (Cython build in oracle/_ref), one process per "
                                   "layer, step = the slowest layer"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_search:
        try:
            line.update(cpu_search_and_scoring(args.config, L, k, E, B, G, C, T, cores))
        except Exception as exc:  # reported next to the headline, never required
            line["search_error"] = repr(exc)
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
