"""Device plumbing: torch owns device memory and streams; libgemcore does the math.

Nothing here computes results; it moves arrays and hands raw pointers plus the
current torch stream to the C ABI.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import GemapError, ValidationError


class NoDeviceError(GemapError, RuntimeError):
    """A CUDA device is required: this package has no CPU compute path."""


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NoDeviceError("no CUDA device visible: the B200 kernels are the only compute path")
    _lib.lib()  # fail loudly if the native library is missing
    return torch.device("cuda", torch.cuda.current_device())


def nvtx(name: str):
    """Decorator: an NVTX range around the call (visible in Nsight Systems / ncu --nvtx)."""
    def wrap(fn):
        import functools

        @functools.wraps(fn)
        def inner(*a, **kw):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **kw)
            finally:
                torch.cuda.nvtx.range_pop()
        return inner
    return wrap


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def upload(arr, dtype: torch.dtype) -> torch.Tensor:
    """numpy/array-like -> contiguous device tensor of `dtype`."""
    if isinstance(arr, torch.Tensor):
        return arr.to(device=device(), dtype=dtype).contiguous()
    np_dtype = {torch.int64: np.int64, torch.int32: np.int32, torch.int16: np.int16, torch.int8: np.int8,
                torch.float64: np.float64, torch.uint8: np.uint8}[dtype]
    a = np.ascontiguousarray(np.asarray(arr, dtype=np_dtype))
    return torch.from_numpy(a).to(device(), non_blocking=False)


def empty(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


INT32_MAX = (1 << 31) - 1


def counts_to_device_int32(tokens: np.ndarray) -> tuple[torch.Tensor, int]:
    """[..., T, E] int64 counts -> device int32, plus max row total (the LUT bound).

    Every load the kernels form is a sum of one step's counts, so the largest
    step total bounds every LUT index and must fit int32.
    """
    tok = np.asarray(tokens)
    if tok.size and int(tok.max()) > INT32_MAX:
        raise ValidationError("token counts above 2^31-1 are outside the device int32 range")
    row_tot = tok.sum(axis=-1, dtype=np.int64) if tok.size else np.zeros(1, dtype=np.int64)
    nmax = int(row_tot.max()) if row_tot.size else 0
    if nmax > INT32_MAX:
        raise ValidationError("a step's total token count exceeds the device int32 range")
    return upload(tok, torch.int32), nmax


# ---------------------------------------------------------------------------
# curves on the device

LUT_MAX_ENTRIES = 1 << 28  # 2 GiB of fp64 per LUT


class DeviceCurves:
    """Packed profile arrays on the device (the _Instance layout, search.py:110-114)
    plus a cached exact LUT  lut[g][n] = C_g(n), n in [0, nmax]."""

    def __init__(self, token_counts, latencies, dense_limits):
        xs = [np.asarray(x, dtype=np.int64) for x in token_counts]
        self.num_gpus = len(xs)
        sizes = [x.size for x in xs]
        self.offsets_h = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
        self.xs = upload(np.concatenate(xs), torch.int64)
        self.ys = upload(np.concatenate([np.asarray(y, dtype=np.float64) for y in latencies]), torch.float64)
        self.offsets = upload(self.offsets_h, torch.int64)
        self.dense = upload(np.asarray(dense_limits, dtype=np.int64), torch.int64)
        self._lut: torch.Tensor | None = None
        self._lut_nmax = -1

    @classmethod
    def from_profile(cls, profile) -> "DeviceCurves":
        cached = getattr(profile, "_device_curves", None)
        if cached is not None and cached.xs.device == device():
            return cached
        dc = cls([c.token_counts for c in profile.curves], [c.latencies for c in profile.curves],
                 [c.dense_limit for c in profile.curves])
        try:
            object.__setattr__(profile, "_device_curves", dc)
        except (AttributeError, TypeError):
            pass
        return dc

    def eval(self, gpu: int, counts: torch.Tensor, err: torch.Tensor | None = None) -> torch.Tensor:
        """C_gpu(counts) on the device, asynchronously (err: optional int32 flag, set on an empty curve)."""
        counts = counts.to(device=device(), dtype=torch.int64).contiguous()
        out = torch.empty(counts.shape, dtype=torch.float64, device=counts.device)
        _lib.call("gem_eval_curve", ptr(self.xs), ptr(self.ys), ptr(self.offsets), ptr(self.dense), int(gpu),
                  ptr(counts), counts.numel(), ptr(out), ptr(err), stream())
        return out

    def equal_latency_load(self, gpu_a: int, gpu_b: int, n_a: int, max_search: int) -> int:
        """profiles.equal_latency_load on one device thread (one result read back)."""
        out = torch.empty((1,), dtype=torch.int64, device=device())
        _lib.call("gem_equal_latency_load", ptr(self.xs), ptr(self.ys), ptr(self.offsets), ptr(self.dense),
                  int(gpu_a), int(gpu_b), int(n_a), int(max_search), ptr(out), stream())
        return int(out.item())

    def lut(self, nmax: int) -> torch.Tensor:
        """[G, nmax+1] fp64 table (grown on demand; a larger table serves smaller nmax)."""
        if nmax < 0:
            nmax = 0
        if self._lut is None or self._lut_nmax < nmax:
            if (nmax + 1) * self.num_gpus > LUT_MAX_ENTRIES:
                raise ValidationError(
                    f"step loads up to {nmax} tokens need a {(nmax + 1) * self.num_gpus}-entry latency table; "
                    f"the device scorer supports up to {LUT_MAX_ENTRIES}")
            lut = torch.empty((self.num_gpus, nmax + 1), dtype=torch.float64, device=device())
            _lib.call("gem_curve_lut", ptr(self.xs), ptr(self.ys), ptr(self.offsets), ptr(self.dense),
                      self.num_gpus, nmax, ptr(lut), stream())
            self._lut, self._lut_nmax = lut, nmax
        return self._lut

    @property
    def lut_nmax(self) -> int:
        return self._lut_nmax


def c_i32() -> ctypes.c_int32:
    return ctypes.c_int32()
