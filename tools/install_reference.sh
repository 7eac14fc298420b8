#!/usr/bin/env bash
# Install the unmodified reference (swarm-rl, /root/reference/pkg) into baseline/_ref, the
# one offline install the task allows, so the reference's package AND its own test files
# travel to the GPU box with the gpurun snapshot (baseline/_ref is git-ignored, not
# gpurun-ignored).  tests/refpath.py finds them there when /root/reference is absent.
#   bash tools/install_reference.sh
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$ROOT/baseline/_ref/swarm_ref_tests"   # the reference's own suites, unmodified
echo "installed: $(ls "$ROOT/baseline/_ref")"
