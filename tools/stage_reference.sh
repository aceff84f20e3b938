#!/usr/bin/env bash
# Stage the unmodified reference (pure Python `binfec`) into the git-ignored
# baseline/_ref/ so that it travels to the GPU box with gpurun:
#   baseline/_ref/binfec/     the installed package (bench.py --impl reference
#                              secondary leg, tests/test_reference_suite.py)
#   baseline/_ref/ref_tests/  the reference's own test suite, re-run through
#                              the shim by tests/test_reference_suite.py
# Needs /root/reference (this container only).
set -euo pipefail
HERE="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
test -d "$SRC" || { echo "no reference at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"   # the build writes into its source tree
rm -rf "$HERE/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$HERE/baseline/_ref/ref_tests"
rm -rf "$TMP"
echo "staged reference into $HERE/baseline/_ref"
