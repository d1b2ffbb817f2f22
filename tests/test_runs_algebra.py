"""CPU check of the run-absorbing chain's algebra and step rule (no GPU).

The device kernel (csrc/thmm_runs.cuh) replaces r consecutive absent records
by one product with T_r = (Gamma diag(1-p))^r.  Here the same step program
(present record, or absent chunk starting at a run position that is a
multiple of R, runs restarting every 32 records of a segment) is evaluated
with numpy, scaled per step, and compared with the serial forward oracle;
and bench.py's exact step counter is checked against a literal loop over
the rule.
"""

import importlib.util
import os

import numpy as np
import pytest

import fixtures as fx
from oracle import thmm_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _steps(present, lo, hi, R, W=32):
    """The kernel's step program over [lo, hi): list of (record, code)."""
    out = []
    for w0 in range(lo, hi, W):
        rs = 0
        wlen = min(W, hi - w0)
        for i in range(wlen):
            t = w0 + i
            if present[t]:
                out.append((t, 0))
                rs = i + 1
            elif (i - rs) % R == 0:
                run = 0
                while i + run < wlen and not present[w0 + i + run]:
                    run += 1
                out.append((t, min(run, R)))
    return out


def _runs_loglik(params, present, lon, lat, R, segments):
    """log L by the run-absorbing steps, segment products folded in order."""
    gamma = np.asarray(params.gamma)
    q = np.array([1.0 - s.p for s in params.states])
    e = orc.emission_columns(params, present, lon, lat)
    t1 = gamma * q[None, :]
    powers = [np.eye(len(q)), t1]
    for _ in range(2, R + 1):
        powers.append(powers[-1] @ t1)
    v = np.asarray(params.delta, dtype=np.float64).copy()
    acc = 0.0
    for lo, hi in orc.segment_bounds(present.size, segments):
        m = np.eye(len(q))
        ls = 0.0
        for t, code in _steps(present, lo, hi, R):
            m = (m @ gamma) * e[t][None, :] if code == 0 else m @ powers[code]
            mx = m.max()
            m /= mx
            ls += np.log(mx)
        v = v @ m
        acc += ls
        mx = v.max()
        acc += np.log(mx)
        v /= mx
    return float(np.log(v.sum()) + acc)


@pytest.mark.parametrize("k,prob,R,segments", [(3, 0.1, 8, 1), (5, 0.3, 16, 4), (9, 0.05, 8, 7), (25, 0.13, 16, 3)])
def test_run_absorbing_steps_reproduce_the_forward_algorithm(k, prob, R, segments):
    rng = np.random.default_rng(100 + k)
    p = fx.random_params(rng, k)
    n = 1500
    pr = rng.random(n) < prob
    lo = np.where(pr, rng.uniform(-1.5, 1.5, n), 0.0)
    la = np.where(pr, rng.uniform(-1.5, 1.5, n), 0.0)
    want = orc.forward_loglik_arrays(p, pr, lo, la)
    got = _runs_loglik(p, pr, lo, la, R, segments)
    assert abs(got - want) <= 1e-11 * abs(want), (got, want)
    steps = sum(len(_steps(pr, a, b, R)) for a, b in orc.segment_bounds(n, segments))
    assert steps < n * (prob + 0.5)  # far fewer steps than records on sparse streams


def test_bench_step_counter_matches_the_kernel_rule():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    rng = np.random.default_rng(1)
    for n, nseg, R in ((1000, 7, 8), (777, 3, 16), (64, 64, 8), (5000, 1, 16), (33, 2, 16)):
        pr = rng.random(n) < 0.2
        want = sum(len(_steps(pr, a, b, R)) for a, b in orc.segment_bounds(n, nseg))
        assert bench.runs_steps(pr, nseg, R) == want, (n, nseg, R)
