#!/usr/bin/env bash
# Install the unmodified reference (prefixdec) into baseline/_ref -- the
# one offline install the task allows -- and put its own test files beside
# it so integration/plugin.py can run them against the B200 path on the GPU
# box (where /root/reference does not exist). baseline/_ref is git-ignored
# and travels with gpurun snapshots. Build from a /tmp copy: the build
# writes into its source tree and /root/reference is read-only.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import prefixdec, prefixdec._kernels; print('prefixdec', prefixdec.__file__)"
