"""CPU ORACLE for the GEM hot path — test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker. The product package never imports it and
fails loudly when its CUDA library is missing.

The numeric kernels live in gem_oracle.c (a scalar C restatement, built with
-ffp-contract=off into oracle/build/liboracle.so); this file binds them with
ctypes and restates the host-side orchestration of the reference search:
  restart order      /root/reference/pkg/src/gemap/search.py:187-193
  search job order   /root/reference/pkg/src/gemap/search.py:256-312
  baselines          /root/reference/pkg/src/gemap/baselines.py:14-53
  statistics         /root/reference/pkg/src/gemap/trace.py:87-114 (exact form)
Pinning: tests/test_oracle.py checks this oracle against the reference's golden
fixtures (tests/golden/, generated from the reference by
tests/golden/make_golden.py) and, when oracle/_ref is present, against the
reference package itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
i16p = np.ctypeslib.ndpointer(dtype=np.int16, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
I64 = ctypes.c_int64
F64 = ctypes.c_double


def build() -> Path:
    """Compile gem_oracle.c (gcc) if the shared object is missing or stale."""
    src = _HERE / "gem_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(str(_LIB_PATH))
    L.or_eval_one.restype = F64
    L.or_eval_one.argtypes = [i64p, f64p, I64, I64, I64]
    L.or_eval_curve_packed.restype = None
    L.or_eval_curve_packed.argtypes = [i64p, f64p, i64p, i64p, I64, i64p, I64, f64p]
    L.or_score.restype = F64
    L.or_score.argtypes = [i64p, I64, I64, I64, i64p, i64p, f64p, i64p, i64p]
    L.or_replay.restype = None
    L.or_replay.argtypes = [i64p, I64, I64, I64, i64p, i64p, f64p, i64p, i64p, i64p, f64p, f64p, i32p,
                            ctypes.POINTER(F64), f64p]
    L.or_swap_candidate_score.restype = F64
    L.or_swap_candidate_score.argtypes = [i64p, I64, I64, i64p, i64p, f64p, I64, i64p, f64p, i64p, i64p, I64, I64]
    L.or_best_swap.restype = ctypes.c_int
    L.or_best_swap.argtypes = [i64p, I64, I64, i64p, i64p, f64p, I64, i64p, f64p, i64p, i64p,
                               ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(F64)]
    L.or_greedy.restype = None
    L.or_greedy.argtypes = [i64p, I64, I64, I64, i64p, f64p, i64p, i64p, i64p, i64p]
    L.or_refine.restype = I64
    L.or_refine.argtypes = [i64p, I64, I64, I64, i64p, f64p, i64p, i64p, i64p, F64, I64, f64p, I64,
                            ctypes.POINTER(F64)]
    L.or_colstats.restype = None
    L.or_colstats.argtypes = [i64p, I64, I64, i64p, i64p, i64p]
    L.or_gram.restype = None
    L.or_gram.argtypes = [i64p, I64, I64, i64p]
    L.or_classify.restype = ctypes.c_int
    L.or_classify.argtypes = [i64p, i64p, i64p, I64, I64, I64, I64, I64, I64, i8p, i16p]
    L.or_topk_hist.restype = None
    L.or_topk_hist.argtypes = [ctypes.c_void_p, ctypes.c_int, I64, I64, I64, I64, I64, i64p, i64p]
    L.or_philox4x32_10.restype = None
    L.or_philox4x32_10.argtypes = [u32p, ctypes.c_uint32, ctypes.c_uint32, u32p]
    L.or_gen_topk.restype = None
    L.or_gen_topk.argtypes = [I64, I64, I64, I64, I64, u32p, i8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                              ctypes.c_uint64, I64, ctypes.c_int, ctypes.c_void_p]
    L.or_gen_topk_l.restype = None
    L.or_gen_topk_l.argtypes = [I64, I64, I64, I64, I64, I64, u32p, i8p, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.c_uint32, ctypes.c_uint64, I64, ctypes.c_int, ctypes.c_void_p]
    _lib = L
    return L


# ---------------------------------------------------------------------------
# curves


class Curves:
    """Packed curve arrays in the reference's _Instance layout (search.py:110-114)."""

    def __init__(self, curves):
        """curves: iterable of (token_counts, latencies, dense_limit)."""
        curves = list(curves)
        xs = [np.asarray(c[0], dtype=np.int64) for c in curves]
        ys = [np.asarray(c[1], dtype=np.float64) for c in curves]
        self.G = len(curves)
        self.offsets = np.concatenate(([0], np.cumsum([x.size for x in xs]))).astype(np.int64)
        self.xs = np.ascontiguousarray(np.concatenate(xs))
        self.ys = np.ascontiguousarray(np.concatenate(ys))
        self.dense = np.asarray([int(c[2]) for c in curves], dtype=np.int64)

    @classmethod
    def from_profile(cls, profile):
        return cls((c.token_counts, c.latencies, c.dense_limit) for c in profile.curves)

    def args(self):
        return self.xs, self.ys, self.offsets, self.dense

    def eval(self, gpu: int, counts) -> np.ndarray:
        ns = np.ascontiguousarray(np.asarray(counts, dtype=np.int64).ravel())
        out = np.empty(ns.size, dtype=np.float64)
        lib().or_eval_curve_packed(*self.args(), int(gpu), ns, ns.size, out)
        return out.reshape(np.shape(counts))

    def lut(self, nmax: int) -> np.ndarray:
        ns = np.arange(nmax + 1, dtype=np.int64)
        return np.stack([self.eval(g, ns) for g in range(self.G)])


def _tok(tokens) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))


def load_matrix(tokens, assignment, G) -> np.ndarray:
    tok = _tok(tokens)
    loads = np.zeros((tok.shape[0], G), dtype=np.int64)
    for g in range(G):
        loads[:, g] = tok[:, np.asarray(assignment) == g].sum(axis=1)
    return loads


def latency_matrix(curves: Curves, loads) -> np.ndarray:
    loads = np.asarray(loads, dtype=np.int64)
    return np.stack([curves.eval(g, loads[:, g]) for g in range(curves.G)], axis=1)


# ---------------------------------------------------------------------------
# scoring / search primitives (C)


def score(tokens, assignment, curves: Curves) -> float:
    tok = _tok(tokens)
    a = np.ascontiguousarray(np.asarray(assignment, dtype=np.int64))
    return float(lib().or_score(tok, tok.shape[0], tok.shape[1], curves.G, a, *curves.args()))


def replay(tokens, assignment, curves: Curves) -> dict:
    tok = _tok(tokens)
    T, E = tok.shape
    G = curves.G
    a = np.ascontiguousarray(np.asarray(assignment, dtype=np.int64))
    loads = np.zeros((T, G), dtype=np.int64)
    lat = np.zeros((T, G))
    step_max = np.zeros(T)
    strag = np.zeros(T, dtype=np.int32)
    busy = np.zeros(G)
    total = F64()
    lib().or_replay(tok, T, E, G, a, *curves.args(), loads, lat, step_max, strag, ctypes.byref(total), busy)
    return {"loads": loads, "lat": lat, "step_max": step_max, "straggler": strag, "total": total.value,
            "busy": busy, "gpu_tokens": loads.sum(axis=0)}


def swap_candidate_score(tokens, assignment, loads, lat, curves: Curves, i, j) -> float:
    tok = _tok(tokens)
    return float(lib().or_swap_candidate_score(
        tok, tok.shape[0], tok.shape[1], np.ascontiguousarray(assignment, dtype=np.int64),
        np.ascontiguousarray(loads, dtype=np.int64), np.ascontiguousarray(lat, dtype=np.float64), curves.G,
        *curves.args(), int(i), int(j)))


def best_swap(tokens, assignment, loads, lat, curves: Curves):
    tok = _tok(tokens)
    bi, bj, bc = I64(), I64(), F64()
    found = lib().or_best_swap(tok, tok.shape[0], tok.shape[1], np.ascontiguousarray(assignment, dtype=np.int64),
                               np.ascontiguousarray(loads, dtype=np.int64),
                               np.ascontiguousarray(lat, dtype=np.float64), curves.G, *curves.args(),
                               ctypes.byref(bi), ctypes.byref(bj), ctypes.byref(bc))
    if not found:
        return False, -1, -1, float("inf")
    return True, bi.value, bj.value, bc.value


def greedy(tokens, order, curves: Curves) -> np.ndarray:
    tok = _tok(tokens)
    out = np.empty(tok.shape[1], dtype=np.int64)
    lib().or_greedy(tok, tok.shape[0], tok.shape[1], curves.G, *curves.args(),
                    np.ascontiguousarray(order, dtype=np.int64), out)
    return out


def refine(tokens, assignment, curves: Curves, threshold: float, cap: int):
    """-> (assignment, final_score, swaps, trajectory)."""
    tok = _tok(tokens)
    a = np.array(assignment, dtype=np.int64, copy=True)
    traj = np.zeros(cap + 1)
    fs = F64()
    swaps = lib().or_refine(tok, tok.shape[0], tok.shape[1], curves.G, *curves.args(), a, float(threshold), int(cap),
                            traj, cap + 1, ctypes.byref(fs))
    if swaps < 0:
        raise AssertionError("oracle refine: incremental score != full rescore")
    return a, fs.value, int(swaps), tuple(float(x) for x in traj[: swaps + 1])


# ---------------------------------------------------------------------------
# statistics, baselines, search orchestration


def colstats3(tokens):
    """(colsum, active, heavy) of one layer's [T, E] counts (gem_oracle.c or_colstats)."""
    tok = _tok(tokens)
    cs = np.zeros(tok.shape[1], dtype=np.int64)
    ac = np.zeros(tok.shape[1], dtype=np.int64)
    hv = np.zeros(tok.shape[1], dtype=np.int64)
    lib().or_colstats(tok, tok.shape[0], tok.shape[1], cs, ac, hv)
    return cs, ac, hv


def colstats(tokens):
    cs, ac, _ = colstats3(tokens)
    return cs, ac


def heavy_counts(tokens) -> np.ndarray:
    """#steps with h > 0 and h*E >= row total, per expert (numpy twin of or_colstats' heavy)."""
    tok = _tok(tokens)
    row = tok.sum(axis=1, keepdims=True)
    return ((tok > 0) & (tok * tok.shape[1] >= row)).sum(axis=0).astype(np.int64)


def gram(tokens) -> np.ndarray:
    tok = _tok(tokens)
    out = np.zeros((tok.shape[1], tok.shape[1]), dtype=np.int64)
    lib().or_gram(tok, tok.shape[0], tok.shape[1], out)
    return out


def mean_utilization(tokens) -> np.ndarray:
    cs, _ = colstats(tokens)
    return cs / int(cs.sum())  # trace.py:95-97 (int64 / int -> IEEE division)


def stats(tokens):
    """(mean_utilization, active_fraction, correlation) from exact integer statistics."""
    tok = _tok(tokens)
    T, E = tok.shape
    cs, ac = colstats(tok)
    g = gram(tok)
    mu = cs / int(cs.sum())
    af = ac / T
    corr = np.eye(E)
    for a in range(E):
        for b in range(a + 1, E):
            va = T * int(g[a, a]) - int(cs[a]) ** 2
            vb = T * int(g[b, b]) - int(cs[b]) ** 2
            if va == 0 or vb == 0:
                v = 0.0
            else:
                num = T * int(g[a, b]) - int(cs[a]) * int(cs[b])
                v = float(num) / (np.sqrt(float(va)) * np.sqrt(float(vb)))
                v = min(1.0, max(-1.0, v))
            corr[a, b] = corr[b, a] = v
    return mu, af, corr


def classify(tokens, cons=(4, 5), corr=(4, 5)):
    tok = _tok(tokens)
    T, E = tok.shape
    cs, _, hv = colstats3(tok)
    g = gram(tok)
    cls = np.zeros(E, dtype=np.int8)
    grp = np.zeros(E, dtype=np.int16)
    err = lib().or_classify(cs, hv, g, T, E, cons[0], cons[1], corr[0], corr[1], cls, grp)
    if err:
        raise OverflowError("oracle classify: statistics out of exact range")
    return cls, grp


def classify_from_stats(colsum, heavy, gram, T, cons=(4, 5), corr=(4, 5)):
    """Classification from (already reduced) integer statistics of one layer."""
    colsum = np.ascontiguousarray(colsum, dtype=np.int64)
    heavy = np.ascontiguousarray(heavy, dtype=np.int64)
    gram = np.ascontiguousarray(gram, dtype=np.int64)
    E = colsum.size
    cls = np.zeros(E, dtype=np.int8)
    grp = np.zeros(E, dtype=np.int16)
    if lib().or_classify(colsum, heavy, gram, int(T), E, cons[0], cons[1], corr[0], corr[1], cls, grp):
        raise OverflowError("oracle classify: statistics out of exact range")
    return cls, grp


def restart_order(mean_util, restart_index, rng, noise_fraction):
    keys = np.asarray(mean_util, dtype=np.float64)
    if restart_index > 0:
        eta = rng.uniform(-1.0, 1.0, keys.shape[0])
        keys = keys * (1.0 + noise_fraction * eta)
    return np.lexsort((np.arange(keys.shape[0]), -keys))


def linear_assignment(E, G):
    return np.arange(E, dtype=np.int64) * G // E


def eplb_assignment(mean_util, G):
    w = np.asarray(mean_util, dtype=np.float64)
    E = w.size
    cap = E // G
    order = np.lexsort((np.arange(E), -w))
    out = np.empty(E, dtype=np.int64)
    totals = [0.0] * G
    counts = [0] * G
    for e in order:
        bg, bt = -1, float("inf")
        for g in range(G):
            if counts[g] < cap and totals[g] < bt:
                bt, bg = totals[g], g
        out[e] = bg
        totals[bg] = totals[bg] + float(w[e])
        counts[bg] += 1
    return out


def search(tokens, curves: Curves, restarts=30, noise_fraction=0.2, threshold=1e-3, rng_seed=0,
           seed_with_baselines=True, max_swaps=None):
    """Restatement of search.py:256-312 -> dict(best_assignment, best_score, provenance, records)."""
    tok = _tok(tokens)
    E = tok.shape[1]
    G = curves.G
    cap = max_swaps if max_swaps is not None else 10 * E
    mu = mean_utilization(tok)
    jobs = [(f"greedy:{i}", None, i) for i in range(restarts)]
    if seed_with_baselines:
        jobs.append(("baseline:linear", linear_assignment(E, G), 0))
        jobs.append(("baseline:eplb", eplb_assignment(mu, G), 0))
    records = []
    for prov, seed_asg, idx in jobs:
        if seed_asg is None:
            rng = np.random.default_rng(rng_seed ^ idx)
            asg = greedy(tok, restart_order(mu, idx, rng, noise_fraction), curves)
        else:
            asg = seed_asg.copy()
        asg, final, swaps, traj = refine(tok, asg, curves, threshold, cap)
        records.append({"provenance": prov, "assignment": asg, "final_score": final, "swap_count": swaps,
                        "trajectory": traj, "initial_score": traj[0]})
    best = 0
    for k in range(1, len(records)):
        if records[k]["final_score"] < records[best]["final_score"]:
            best = k
    return {"best_assignment": records[best]["assignment"], "best_score": records[best]["final_score"],
            "provenance": records[best]["provenance"], "records": records}


# ---------------------------------------------------------------------------
# top-k ids


def topk_hist(ids, B: int, E: int):
    """ids [L,N,k] int16/int32 -> (hist [L,T,E] int64, dropped [L])."""
    ids = np.ascontiguousarray(ids)
    assert ids.dtype in (np.int16, np.int32)
    L, N, k = ids.shape
    T = (N + B - 1) // B
    hist = np.zeros((L, T, E), dtype=np.int64)
    dropped = np.zeros(L, dtype=np.int64)
    lib().or_topk_hist(ids.ctypes.data, ids.dtype.itemsize, L, N, k, B, E, hist, dropped)
    return hist, dropped


def coselect(ids, E: int) -> np.ndarray:
    """Token-level co-selection counts C[l,a,b] = #tokens choosing both a and b (int64 [L,E,E]).

    No reference counterpart ("parity unpinned by the
    reference"); restated from its definition OᵀO over the 0/1 selection
    indicator O[n,e] = [e in ids[n]] (ids outside [0,E) ignored, a repeated id
    counts once). Its diagonal is the number of tokens choosing e, i.e.
    topk_hist's column sums when ids are distinct -- the link to the pinned K1."""
    ids = np.asarray(ids)
    L, N, k = ids.shape
    out = np.zeros((L, E, E), dtype=np.int64)
    for l in range(L):
        x = ids[l].astype(np.int64)
        ok = (x >= 0) & (x < E)
        onehot = np.zeros((N, E + 1), dtype=np.int64)
        onehot[np.repeat(np.arange(N), k), np.where(ok, x, E).ravel()] = 1  # assignment: duplicates set once
        o = onehot[:, :E]
        out[l] = o.T @ o
    return out


def coselect_loops(ids, E: int) -> np.ndarray:
    """The same by explicit per-token pair loops (pure Python; small cases only)."""
    ids = np.asarray(ids)
    L, N, k = ids.shape
    out = np.zeros((L, E, E), dtype=np.int64)
    for l in range(L):
        for n in range(N):
            s = sorted({int(v) for v in ids[l, n] if 0 <= int(v) < E})
            for a in s:
                for b in s:
                    out[l, a, b] += 1
    return out


def philox4x32_10(counter, key):
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(np.ascontiguousarray(counter, dtype=np.uint32), int(key[0]), int(key[1]), out)
    return out


def gen_topk(L, N, k, B, E, weight, role, p_cons, p_burst, burst_mult, seed, token_offset=0, id_bytes=2,
             layer_offset=0):
    """ids [L, N, k] of layers [layer_offset, layer_offset + L) (weight/role: those layers' rows)."""
    ids = np.zeros((L, N, k), dtype=np.int16 if id_bytes == 2 else np.int32)
    lib().or_gen_topk_l(L, int(layer_offset), N, k, B, E, np.ascontiguousarray(weight, dtype=np.uint32),
                        np.ascontiguousarray(role, dtype=np.int8), int(p_cons), int(p_burst), int(burst_mult),
                        int(seed), int(token_offset), id_bytes, ids.ctypes.data)
    return ids


def reference_path() -> Path | None:
    """oracle/_ref: the reference package installed by oracle/build_ref.sh (if present)."""
    p = _HERE / "_ref"
    return p if (p / "gemap" / "__init__.py").exists() else None


def import_reference():
    """Import the real reference (`gemap`) from oracle/_ref, or None."""
    p = reference_path()
    if p is None:
        return None
    import sys

    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    os.environ.setdefault("GEM_BACKEND", "auto")
    import gemap  # noqa: F401

    return gemap
