#!/usr/bin/env bash
# Run the reference's own engine tests + acceptance criteria 1-2 against the
# B200 engine (tests/ref_shim.py routes parallel_loglik to the GPU).
set -uo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="$ROOT/baseline/_ref"
export PYTHONPATH="$REF:$REF/ref_tests:$ROOT/tests:$ROOT:${PYTHONPATH:-}"
export NUMBA_CACHE_DIR="${NUMBA_CACHE_DIR:-/tmp/numba_cache_ref}"
cd "$REF/ref_tests"
python -m pytest -v -p no:cacheprovider -p ref_shim --rootdir . test_engine.py 2>&1 | grep -E "PASSED|FAILED|ERROR|passed|failed|ref_shim"
python -m pytest -q -s -p no:cacheprovider -p ref_shim --rootdir . test_acceptance.py -k "criterion_1 or criterion_2" 2>&1 | grep -E "criterion|passed|failed|ref_shim"
