"""The reference's OWN tests for the path, run against the B200 engine -- needs a B200.

tools/install_reference.sh installs the unmodified reference package into
baseline/_ref (git-ignored; it travels to the GPU box) together with its test
suite.  Here pytest runs the reference's test_engine.py (TestParallelLoglik
and the rest of the engine tests: 1e-9 vs the serial oracle, segment-count
invariance 1e-10, renorm-schedule tracking 1e-11, float32 1e-4, bitwise
worker invariance, state cap, config rejects) and acceptance criteria 1-2
(200 random instances vs serial and brute force < 1e-10; K=25 N=1e5 segment
spread < 1e-10) with ``parallel_loglik`` / ``_parallel_loglik_arrays`` routed
to the GPU by the tests/ref_shim.py plugin.  Skipped when the reference
install is absent.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")


def _run(args, timeout):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REF_TESTS, os.path.join(ROOT, "tests"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_shim", "--rootdir", REF_TESTS,
           *args]
    return subprocess.run(cmd, env=env, cwd=REF_TESTS, capture_output=True, text=True, timeout=timeout)


def _passed(out):
    m = re.search(r"(\d+) passed", out.stdout)
    return int(m.group(1)) if m else 0


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not installed (tools/install_reference.sh)")
def test_reference_engine_suite_on_b200():
    out = _run(["test_engine.py"], 900)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert _passed(out) >= 25, out.stdout[-2000:]
    calls = int(re.search(r"ref_shim: (\d+) likelihood calls", out.stdout).group(1))
    assert calls > 0


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not installed (tools/install_reference.sh)")
def test_reference_acceptance_criteria_1_2_on_b200():
    out = _run(["test_acceptance.py", "-k", "criterion_1 or criterion_2", "-s"], 900)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "criterion 1 (oracle equivalence): PASS" in out.stdout, out.stdout[-3000:]
    assert "criterion 2 (segment invariance): PASS" in out.stdout, out.stdout[-3000:]
