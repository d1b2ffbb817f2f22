#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with gpurun) for the --impl reference bench arm, and
# place the reference's own test suite next to it (baseline/_ref/ref_tests)
# so tests/test_gpu_reference_suite.py can run it against the B200 engine.
# Needs /root/reference (this container only).  Offline, no dependency
# resolution (numpy/scipy/numba/PyYAML are already in the image).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 1; }
rm -rf /tmp/refpkg && cp -r "$SRC" /tmp/refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/refpkg --upgrade >/dev/null
rm -rf "$ROOT/baseline/_ref/ref_tests" && cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
echo "reference installed: $ROOT/baseline/_ref (tests: baseline/_ref/ref_tests)"
