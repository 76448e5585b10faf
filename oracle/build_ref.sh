#!/usr/bin/env bash
# Build the real reference (`gemap`, /root/reference/pkg) into oracle/_ref/ —
# a strengthening oracle and the CPU arm of bench.py --impl reference.
# Runs only where /root/reference exists (this container); oracle/_ref is
# git-ignored but travels to the GPU box with the gpurun snapshot.
# The reference's setup.py compiles its Cython kernels with -O3 -ffp-contract=off.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no /root/reference: keeping existing oracle/_ref" >&2; exit 0; }
# the reference's own test suite + fixtures, run against this package by
# tests/test_reference_suite.py (git-ignored like the rest of oracle/_ref)
if [ ! -f "$HERE/_ref/ref_tests/conftest.py" ]; then
  mkdir -p "$HERE/_ref/ref_tests"
  cp -r "$SRC/tests/." "$HERE/_ref/ref_tests/"
fi
if [ -f "$HERE/_ref/gemap/__init__.py" ] && ls "$HERE"/_ref/gemap/_kernels*.so >/dev/null 2>&1; then exit 0; fi
TMP="$(mktemp -d /tmp/gemref.XXXXXX)"
cp -r "$SRC" "$TMP/pkg"          # the build writes into its source tree; /root/reference is read-only
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg" >/dev/null
rm -rf "$TMP"
echo "built reference into $HERE/_ref"
