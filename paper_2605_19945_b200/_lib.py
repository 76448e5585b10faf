"""ctypes binding of libgemcore.so (include/gemcore.h).

The package has exactly one compute backend: the sm_100a kernels in this
library. There is no CPU fallback — if the library is missing or no CUDA
device is present, every compute entry point raises instead of degrading.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

from .errors import GemapError

_PKG = Path(__file__).resolve().parent
# GEM_LIB_VARIANT=<name> loads _lib/libgemcore-<name>.so (kernel experiments built by tools/)
LIB_PATH = _PKG / "_lib" / ("libgemcore-%s.so" % os.environ["GEM_LIB_VARIANT"] if os.environ.get("GEM_LIB_VARIANT")
                            else "libgemcore.so")
CSRC = _PKG / "csrc"

GEM_OK = 0
GEM_ERR_INVALID = -1
GEM_ERR_CUDA = -2
GEM_ERR_MISMATCH = -3
GEM_ERR_RANGE = -4

GEM_CLASS_OTHER = 0
GEM_CLASS_CONSISTENT = 1
GEM_CLASS_TEMPORAL = 2


class KernelError(GemapError):
    """A libgemcore entry point reported a failure."""


class NativeLibraryMissing(GemapError, RuntimeError):
    """libgemcore.so is not built; run __graft_entry__.build() or `make -C csrc`."""


def build(force: bool = False) -> Path:
    """Compile libgemcore.so for sm_100a with nvcc (in-tree)."""
    if force or not LIB_PATH.exists():
        subprocess.run(["make", "-s", "-C", str(CSRC), "-j", str(min(8, os.cpu_count() or 1))], check=True)
    return LIB_PATH


P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U32 = ctypes.c_uint32
U64 = ctypes.c_uint64
F64 = ctypes.c_double
SZ = ctypes.c_size_t

# name -> argtypes (all return int status unless noted)
_SIGNATURES = {
    "gem_device_info": [P, P, P],
    "gem_ref_eval_curve_packed": [P, P, P, P, I64, I64, P, I64, P],
    "gem_ref_swap_candidate_score": [P, I64, I64, P, P, P, I64, P, P, P, P, I64, I64, P],
    "gem_ref_best_swap": [P, I64, I64, P, P, P, I64, P, P, P, P, P, P, P, P],
    "gem_gen_topk": [I64, I64, I32, I32, I32, P, P, U32, U32, U32, U64, I64, I32, P, P],
    "gem_topk_hist": [P, I32, I64, I64, I32, I32, I32, P, P, P, P, P, P],
    "gem_topk_hist_rows": [P, I32, I64, I64, I32, I32, I32, P, I64, P, P, P, P, P],
    "gem_scale_gaps": [P, I64, I64, P, I32, P, P],
    "gem_restart_order": [P, I64, I32, P, P],
    "gem_hist_colstats": [P, I64, I64, I32, P, P, P, P],
    "gem_step_gram": [P, I64, I64, I32, I64, P, P],
    "gem_step_gram_path": [I32, I64],
    "gem_step_gram_cc": [P, I64, I64, I32, P, P],
    "gem_step_gram_tc": [P, I64, I64, I32, P, P],
    "gem_coselect": [P, I32, I64, I64, I32, I32, P, P],
    "gem_coselect_path": [P, I32, I64, I32, I32],
    "gem_coselect_tc": [P, I32, I64, I64, I32, I32, P, P],
    "gem_coselect_scatter": [P, I32, I64, I64, I32, I32, P, P],
    "gem_stats_finalize": [P, P, P, I64, I64, I32, P, P, P, P],
    "gem_classify": [P, P, P, I64, I64, I32, I64, I64, I64, I64, P, P, P, P],
    "gem_eval_curve": [P, P, P, P, I32, P, I64, P, P, P],
    "gem_equal_latency_load": [P, P, P, P, I32, I32, I64, I64, P, P],
    "gem_curve_lut": [P, P, P, P, I32, I64, P, P],
    "gem_score_batch": [P, I64, I64, I32, I32, P, I64, P, I64, P, P, P, P],
    "gem_layer_sum": [P, I64, I64, P, P],
    "gem_score_batch_tc": [P, I64, I64, I32, I32, P, I64, P, I64, P, P, P],
    "gem_score_batch_v1": [P, I64, I64, I32, I32, P, I64, P, I64, P, P, P],
    "gem_replay": [P, I64, I32, I32, P, P, I64, P, P, P, P, P, P, P, P, P],
    "gem_search_runs": [P, I64, I64, I32, I32, P, I64, I64, P, P, P, P, F64, I64, I64, P, P, P, P, SZ, P],
    "gem_best_swap_runs": [P, I64, I64, I32, I32, P, I64, I64, P, P, P, P, P, P, P, SZ, P],
}

_lib = None


def lib():
    """Load libgemcore.so (raises NativeLibraryMissing if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: the CUDA library is required (no CPU fallback). "
            "Build it with `python -c 'import __graft_entry__ as g; g.build()'`."
        )
    L = ctypes.CDLL(str(LIB_PATH))
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    L.gem_version.restype = ctypes.c_char_p
    L.gem_version.argtypes = []
    L.gem_last_error.restype = ctypes.c_char_p
    L.gem_last_error.argtypes = []
    L.gem_search_workspace_bytes.restype = SZ
    L.gem_search_workspace_bytes.argtypes = [I64, I64, I32, I32]
    _lib = L
    return L


def exported_symbols() -> list[str]:
    return sorted(list(_SIGNATURES) + ["gem_version", "gem_last_error", "gem_search_workspace_bytes"])


def check(rc: int, what: str) -> None:
    if rc != GEM_OK:
        msg = lib().gem_last_error().decode(errors="replace")
        raise KernelError(f"{what} failed (status {rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
