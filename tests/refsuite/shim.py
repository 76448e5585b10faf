"""Build a `gemap` shim package that IS this package (module aliases only), so
the reference's own tests -- and its `python -m gemap` subprocesses -- import
paper_2605_19945_b200 under the reference's name. Generated at test time
into a scratch directory; nothing of the reference is copied."""

from __future__ import annotations

from pathlib import Path

_INIT = '''"""gemap -> paper_2605_19945_b200 (test shim)."""
import importlib as _il
import sys as _sys

import paper_2605_19945_b200 as _pkg
from paper_2605_19945_b200 import *  # noqa: F401,F403
from paper_2605_19945_b200 import __all__, __version__  # noqa: F401

for _m in ("search", "kernels", "mapping", "cli", "trace", "profiles", "baselines", "scale", "errors", "_util"):
    _sys.modules["gemap." + _m] = _il.import_module("paper_2605_19945_b200." + _m)
    if _m not in globals():  # gemap.search is the function, as in the reference
        globals()[_m] = _sys.modules["gemap." + _m]
'''

_MAIN = '''import sys

from paper_2605_19945_b200.cli import main

sys.exit(main())
'''


def build(root: Path) -> Path:
    d = Path(root) / "gemap"
    d.mkdir(parents=True, exist_ok=True)
    (d / "__init__.py").write_text(_INIT)
    (d / "__main__.py").write_text(_MAIN)
    return Path(root)
