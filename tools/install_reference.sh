#!/bin/bash
# Offline install of the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot).  The reference's own test suite,
# demos and configs are copied next to it (baseline/_ref/greengate_suite/) so
# tests/test_reference_suite_gpu.py can run the reference's tests against the
# patched-in device controller on a box where /root/reference does not exist.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"                      # the build may write into the tree
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/greengate_suite"
cp -r "$SRC/tests" "$SRC/demos" "$SRC/configs" "$ROOT/baseline/_ref/greengate_suite/"
rm -rf "$TMP"
echo "reference installed: $ROOT/baseline/_ref"
