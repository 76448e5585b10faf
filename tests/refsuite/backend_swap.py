"""pytest plugin (-p refsuite.backend_swap): the reference package's ACTIVE
kernel backend -- what its search(), refine() and the acceptance criteria call
through kernels.active() (/root/reference/pkg/src/gemap/kernels.py:37-45) --
is replaced by this package's CUDA backend before any test runs. Tests that
pick "python"/"cython" explicitly still get those modules (they are the
comparators), so every reference test that exercises the active backend
drives the sm_100a kernels through the tier-1 C ABI."""

import gemap.kernels as _ref_kernels

from paper_2605_19945_b200 import kernels as _ours

_ref_kernels._active = _ours.get_backend("cuda")
assert _ref_kernels.active_name() == "cuda"
