#!/usr/bin/env bash
# Install the UNMODIFIED reference (viscache 0.1.0) into baseline/_ref for the
# bench's reference arm and the drop-in tests (tests/test_gpu_dropin.py).
# baseline/_ref is git-ignored but travels to the GPU box with the snapshot.
# The reference tree is read-only, so pip builds from a scratch copy; only
# dependency resolution fails offline, hence --no-deps (numpy/numba/scipy are
# in the image).  The reference's own test suite is copied next to the package
# (baseline/_ref/viscache_tests) so it can run on the GPU box against the
# injected CUDA cache.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}"
TMP="$(mktemp -d)"
cp -r "$SRC/pkg" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/pkg/tests" "$ROOT/baseline/_ref/viscache_tests"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
