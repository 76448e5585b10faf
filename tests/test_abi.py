"""CPU checks of the C ABI: the library exists, loads, and exports every
function include/gemcore.h declares (no compute calls without a GPU)."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "gemcore.h"
LIB = ROOT / "paper_2605_19945_b200" / "_lib" / "libgemcore.so"


def declared() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(gem_[a-z_0-9]+)\s*\(", text, flags=re.M))


def _ensure_lib():
    if not LIB.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "paper_2605_19945_b200" / "csrc")], check=True)


def test_header_declares_protocol_and_device_tiers():
    names = declared()
    for n in ("gem_ref_eval_curve_packed", "gem_ref_swap_candidate_score", "gem_ref_best_swap", "gem_topk_hist",
              "gem_step_gram", "gem_stats_finalize", "gem_classify", "gem_curve_lut", "gem_score_batch",
              "gem_search_runs", "gem_gen_topk", "gem_replay"):
        assert n in names, n


def test_library_exports_every_declared_symbol():
    _ensure_lib()
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = declared() - exported
    assert not missing, missing


def test_ctypes_binding_covers_header():
    import sys

    _ensure_lib()
    sys.path.insert(0, str(ROOT))
    from paper_2605_19945_b200 import _lib

    assert set(_lib.exported_symbols()) == declared()
    L = _lib.lib()  # dlopen works without a GPU
    assert L.gem_version().decode().startswith("gemcore")


def test_sass_is_sm100a():
    _ensure_lib()
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
