"""Vectorised prior / block proposals of the many-chain sampler vs the
reference's scalar ones (CPU; the GPU run is in test_gpu_parity.py)."""

import math

import numpy as np
import pytest

from conftest import needs_reference
from paper_2003_03508_b200 import mcmc, proposals, synth


def _ref():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from tremorhmm import bayes

    return bayes


@needs_reference
@pytest.mark.parametrize("k", [1, 3, 8])
def test_log_prior_matches_reference(k):
    bayes = _ref()
    rng = np.random.default_rng(100 + k)
    vecs, want = [], []
    for _ in range(4):
        p = synth.sample_prior_params(k, rng)
        p = synth.HmmParams(gamma=0.999 * p.gamma + 0.001 / k, delta=p.delta, states=p.states)
        v = proposals.params_to_vectors([p])[0]
        rp = bayes.params_from_vector(k, v, delta_mode="uniform")
        vecs.append(v)
        want.append(bayes.log_prior(rp, bayes.PriorSpec.default_for(k)))
    got = mcmc.log_prior_batch(k, np.stack(vecs))
    np.testing.assert_allclose(got, want, rtol=1e-12)


@needs_reference
def test_block_proposals_match_reference_stream():
    bayes = _ref()
    k = 4
    rng0 = np.random.default_rng(7)
    p = synth.sample_prior_params(k, rng0)
    p = synth.HmmParams(gamma=0.999 * p.gamma + 0.001 / k, delta=p.delta, states=p.states)
    v = proposals.params_to_vectors([p])[None][0]
    rp = bayes.params_from_vector(k, v[0], delta_mode="uniform")
    for (name, fn), step in zip(mcmc.BLOCKS, (0.1, 0.1, 0.005, 0.02)):
        r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
        cand, jac, ok = fn(k, v, step, r1)
        ref_p, ref_jac = bayes._propose_block(rp, name, step, r2, "uniform")
        np.testing.assert_allclose(cand[0], bayes.params_to_vector(ref_p), rtol=1e-13, atol=1e-15)
        assert math.isclose(jac[0], ref_jac, rel_tol=1e-10, abs_tol=1e-12)
        assert ok[0]


def test_log_prior_support():
    k = 2
    rng = np.random.default_rng(3)
    p = synth.sample_prior_params(k, rng)
    p = synth.HmmParams(gamma=0.9 * p.gamma + 0.05, delta=p.delta, states=p.states)
    v = proposals.params_to_vectors([p])
    assert np.isfinite(mcmc.log_prior_batch(k, v)[0])
    w = v.copy()
    w[0, k * k + k] = 100.0              # mu outside the Shikoku box
    assert mcmc.log_prior_batch(k, w)[0] == -np.inf
