#!/bin/bash
# Install the UNMODIFIED reference package (lfbp, /root/reference/pkg) into
# baseline/_ref -- git-ignored, but it travels to the GPU box with the gpurun
# snapshot -- together with the reference's own test files
# (baseline/_ref/tests), so the GPU box can run them against the drop-in
# (tests/test_reference_suite.py) and time the reference as shipped
# (bench.py cpu_baseline).  /root/reference is read-only, so the wheel is
# built from a copy under /tmp.  Nothing here is committed.
set -euo pipefail
REPO=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$REPO/baseline/_ref/tests"
rm -rf "$TMP"
echo "installed $(ls "$REPO/baseline/_ref")"
