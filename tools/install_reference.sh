#!/usr/bin/env bash
# Install the UNMODIFIED reference package (arXiv 2602.04936 `lcpsearch`,
# /root/reference/pkg) into baseline/_ref, plus a copy of its own test files
# under baseline/_ref/lcpsearch_tests.  baseline/_ref is git-ignored (not
# product source) but not gpurun-ignored, so it travels to the GPU box, where
# /root/reference does not exist.  Used by:
#   - bench.py (cpu_baseline.python_reference: the reference's own
#     _query_stream timed on the box's host cores),
#   - tests/test_reference_suite.py (the reference's own query tests run
#     against the GPU package through tests/refsuite/lcpsearch_gpu_shim.py).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"   # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/lcpsearch_tests"
cp "$TMP"/pkg/tests/*.py "$ROOT/baseline/_ref/lcpsearch_tests/"
echo "installed lcpsearch into $ROOT/baseline/_ref"
