#!/usr/bin/env bash
# Install the read-only reference package into baseline/_ref (git-ignored, not
# gpurun-ignored: it travels to the GPU box) and stage its test directory
# beside it, so tests/test_reference_suite_gpu.py can run the reference's own
# test files against the device engine there. Run in this container, where
# /root/reference exists. Nothing here is committed.
set -euo pipefail
REPO=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
tmp=$(mktemp -d)
cp -r "$SRC" "$tmp/pkg"  # the build writes into the source tree; the reference is read-only
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$tmp/pkg" >/dev/null
cp -r "$SRC/tests" "$REPO/baseline/_ref/tests"
cp "$SRC/pyproject.toml" "$REPO/baseline/_ref/pyproject.toml"
rm -rf "$tmp"
echo "staged $(ls "$REPO/baseline/_ref/tests" | wc -l) test files into baseline/_ref"
