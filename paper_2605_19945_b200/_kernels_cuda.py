"""The CUDA backend module of the reference's kernel-backend protocol.

Drop-in for `gemap._kernels` (/root/reference/pkg/src/gemap/_kernels.pyx:58-160):
same three functions, same argument meaning (caller-owned host arrays, results
freshly allocated), same results bit for bit, same (False, -1, -1, inf)
convention. Each call goes through tier 1 of the C ABI (gem_ref_*), which
stages the host arrays on the GPU, runs the sm_100a kernels and copies back.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

BACKEND = "cuda"


def _c(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def eval_curve_packed(xs_flat, ys_flat, offsets, dense_limits, gpu, counts):
    """Evaluate GPU `gpu`'s curve from the packed profile arrays."""
    xs, ys, off, dl = _c(xs_flat, np.int64), _c(ys_flat, np.float64), _c(offsets, np.int64), _c(dense_limits, np.int64)
    ns = _c(np.asarray(counts, dtype=np.int64).ravel(), np.int64)
    out = np.empty(ns.shape[0], dtype=np.float64)
    _lib.call("gem_ref_eval_curve_packed", _p(xs), _p(ys), _p(off), _p(dl), dl.shape[0], int(gpu), _p(ns),
              ns.shape[0], _p(out))
    return out.reshape(np.shape(counts))


def swap_candidate_score(tokens, assignment, loads, lat, xs_flat, ys_flat, offsets, dense_limits, i, j):
    """Total score after swapping experts i and j, from cached loads/latencies."""
    tok = _c(tokens, np.int64)
    asg, ld, lt = _c(assignment, np.int64), _c(loads, np.int64), _c(lat, np.float64)
    xs, ys, off, dl = _c(xs_flat, np.int64), _c(ys_flat, np.float64), _c(offsets, np.int64), _c(dense_limits, np.int64)
    out = ctypes.c_double()
    _lib.call("gem_ref_swap_candidate_score", _p(tok), tok.shape[0], tok.shape[1], _p(asg), _p(ld), _p(lt),
              lt.shape[1], _p(xs), _p(ys), _p(off), _p(dl), int(i), int(j), ctypes.addressof(out))
    return float(out.value)


def best_swap(tokens, assignment, loads, lat, xs_flat, ys_flat, offsets, dense_limits):
    """Scan all cross-GPU expert pairs; return (found, i, j, candidate_score)."""
    tok = _c(tokens, np.int64)
    asg, ld, lt = _c(assignment, np.int64), _c(loads, np.int64), _c(lat, np.float64)
    xs, ys, off, dl = _c(xs_flat, np.int64), _c(ys_flat, np.float64), _c(offsets, np.int64), _c(dense_limits, np.int64)
    found, bi, bj, bc = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    _lib.call("gem_ref_best_swap", _p(tok), tok.shape[0], tok.shape[1], _p(asg), _p(ld), _p(lt), ld.shape[1],
              _p(xs), _p(ys), _p(off), _p(dl), ctypes.addressof(found), ctypes.addressof(bi),
              ctypes.addressof(bj), ctypes.addressof(bc))
    if not found.value:
        return False, -1, -1, float("inf")
    return True, int(bi.value), int(bj.value), float(bc.value)
