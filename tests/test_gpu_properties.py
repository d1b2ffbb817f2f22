"""Size-independent properties of the likelihood at full BASELINE sizes -- needs a B200.

The reference pins these on small inputs (test_core.py:177-241); here they
are checked on the device path up to N = 10^6..10^7 where no CPU oracle run
is cheap:

* all-absent chain with a common event probability p: every emission is
  q = 1 - p and Gamma is row-stochastic, so logL = N log(1 - p) exactly in
  real arithmetic (reference test_core.py "all absent" closed form);
* relabelling the hidden states (Gamma -> P Gamma P', delta -> P delta,
  states permuted) leaves the likelihood unchanged (test_core.py
  permutation invariance);
* records far out in the tails (emissions down to ~1e-200, far below the
  FP32 range) stay exact against the C oracle: the power-of-two row scaling
  keeps the products in range.
"""

import math

import numpy as np
import pytest

import fixtures as fx
from oracle import coracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


def _with_common_p(eng, p, prob):
    states = tuple(eng.StateEmission(prob, np.asarray(s.mu), np.asarray(s.sigma)) for s in p.states)
    return eng.HmmParams(gamma=np.asarray(p.gamma), delta=np.asarray(p.delta), states=states)


@pytest.mark.parametrize("k,n", [(5, 10_000), (25, 1_000_000), (50, 2_000_000), (80, 500_000)])
def test_all_absent_closed_form(eng, k, n):
    rng = np.random.default_rng(900 + k)
    p = _with_common_p(eng, fx.random_params(rng, k), 0.3)
    pr = np.zeros(n, dtype=bool)
    lo = np.zeros(n)
    la = np.zeros(n)
    want = n * math.log(1.0 - 0.3)
    dev = eng.DeviceObservations(pr, lo, la)
    got = dev.loglik(p, eng.EngineConfig())
    assert abs(got - want) <= 1e-12 * abs(want), (got, want)
    got32 = dev.loglik(p, eng.EngineConfig(precision="tf32x3"))
    assert abs(got32 - want) <= 1e-6 * abs(want)


@pytest.mark.parametrize("k,n", [(7, 20_000), (25, 1_000_000), (33, 300_000)])
def test_state_permutation_invariance(eng, k, n):
    rng = np.random.default_rng(950 + k)
    p = fx.random_params(rng, k)
    pr, lo, la = fx.random_obs_arrays(rng, n)
    perm = rng.permutation(k)
    g = np.asarray(p.gamma)[np.ix_(perm, perm)]
    d = np.asarray(p.delta)[perm]
    q = eng.HmmParams(gamma=g, delta=d, states=tuple(p.states[i] for i in perm))
    dev = eng.DeviceObservations(pr, lo, la)
    a, b = dev.loglik_batch([p, q], eng.EngineConfig())
    assert abs(a - b) <= 1e-12 * abs(a), (a, b)


def test_far_tail_records_match_oracle(eng):
    rng = np.random.default_rng(77)
    for k in (3, 25, 80):
        p = fx.random_params(rng, k, sigma_scale=0.05)
        pr, lo, la = fx.random_obs_arrays(rng, 4000)
        # a few records ~20-30 sigma from every state mean: emissions ~1e-90..1e-200
        idx = rng.choice(4000, 40, replace=False)
        pr[idx] = True
        lo[idx] = 2.0 + rng.uniform(0.0, 0.5, 40)
        la[idx] = -2.0 - rng.uniform(0.0, 0.5, 40)
        want = coracle.forward_loglik(p, pr, lo, la)
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())
        assert abs(got - want) <= 1e-9 * abs(want), (k, got, want)
        assert abs(got - want) <= 1e-11 * abs(want), (k, got, want)
