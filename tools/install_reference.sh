#!/bin/bash
# Install the UNMODIFIED reference package (approx8) into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot), the one offline install the task
# allows.  The build writes egg-info into its source tree, so it runs from a copy
# under /tmp (/root/reference is read-only).  The reference's own test directory is
# copied next to it (baseline/_ref/approx8_tests, also git-ignored) so that
# tests/test_dropin_reference.py can run the reference's tests against the B200
# drop-in on the GPU box, where /root/reference does not exist.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --no-deps --upgrade "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/approx8_tests" "$ROOT/baseline/_ref/approx8_configs"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/approx8_tests"
cp -r "$SRC/configs" "$ROOT/baseline/_ref/approx8_configs"  # the perf-model tests read configs/*.toml
rm -rf "$TMP"
echo "installed approx8 into $ROOT/baseline/_ref"
