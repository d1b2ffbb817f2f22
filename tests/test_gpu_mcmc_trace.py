"""The many-chain sampler (mcmc.run_chains) pinned to the reference sampler.

With one chain and the reference's seed, ``run_chains`` must reproduce
``bayes.run_chain`` (bayes.py:690-796) exactly: same initial prior draw, the
four random-walk blocks, the rejuvenation move every 4th iteration
(``_RejuvenationKernel``, bayes.py:472-604), the same random stream, hence the
same accept decisions.  Both samplers get the same likelihood: on the GPU the
B200 engine (the reference through its ``loglik_fn`` hook, ours through the
batched entry), on CPU the C oracle.

Bound (stated): parameter vectors, log-likelihoods and log-priors of every
kept row agree to <= 1e-12 (relative; the vectorised prior and proposal
arithmetic may differ from the reference's scalar code by a few ulp), and the
acceptance rate of every block is equal.
"""

import os
import sys

import numpy as np
import pytest

from conftest import reference_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-12


def _reference():
    """The reference package: /root/reference here, baseline/_ref on the GPU box."""
    for path in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(path, "tremorhmm")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import tremorhmm  # noqa: F401
            from tremorhmm import bayes, core
            return bayes, core
    return None


def _compare(k, n, iters, seed, single_ll, batch_obs, alpha=0.01):
    from paper_2003_03508_b200 import mcmc, synth

    ref = _reference()
    if ref is None:
        pytest.skip("reference package not installed")
    bayes, core = ref
    _, pr, lo, la = synth.make_workload("k5_n1e4" if k == 5 else "k25_n1e6", n=n)
    obs = [core.Observation((float(x), float(y))) if f else core.Observation(None) for f, x, y in zip(pr, lo, la)]
    spec = bayes.PriorSpec.default_for(k)
    if alpha != 0.01:  # a flatter transition prior: the rejuvenation move gets accepted, and at K=25
        # prior draws have no exact-zero transitions (Dirichlet(0.01) rows of 25 almost surely do, and the
        # reference's initialisation then never finds a finite prior)
        from dataclasses import replace
        spec = replace(spec, dirichlet_alpha=alpha)
    steps = bayes.StepSizes(0.1, 0.1, 0.005, 0.02)
    cfg = bayes.McmcConfig(iterations=iters, thin=1, seed=seed, steps=steps)
    trace = bayes.run_chain(k, obs, spec, cfg, None, delta_mode="uniform", loglik_fn=single_ll)

    rng = np.random.default_rng(seed)
    ours = mcmc.PriorSpec(dirichlet_alpha=alpha)
    init, init_ll = mcmc.init_from_prior(k, 1, batch_obs, rng, spec=ours)
    res = mcmc.run_chains(k, batch_obs, init, iters, steps=(0.1, 0.1, 0.005, 0.02), delta_mode="uniform",
                          rng=rng, points=(pr, lo, la), init_loglik=init_ll, spec=ours)
    assert list(res.iterations) == list(trace.iterations)
    np.testing.assert_allclose(res.vectors[:, 0, :], trace.params, rtol=TOL, atol=1e-300)
    np.testing.assert_allclose(res.log_likelihood[:, 0], trace.log_likelihood, rtol=TOL, atol=0)
    np.testing.assert_allclose(res.log_prior[:, 0], trace.log_prior, rtol=TOL, atol=1e-12)
    for block, rate in trace.stats["acceptance_by_block"].items():
        assert res.acceptance[block][0] == rate, (block, res.acceptance[block][0], rate)
    n_rejuv = res.proposed["rejuvenate"]
    assert n_rejuv >= 4
    moved = np.any(res.vectors[1:, 0] != res.vectors[:-1, 0], axis=1).sum()
    return n_rejuv, int(res.accepted["rejuvenate"][0]), int(moved)


class _OracleObs:
    """Batched likelihood over the C oracle (CPU stand-in for the device)."""

    def __init__(self, pr, lo, la):
        self.arrays = (pr, lo, la)

    def loglik_batch(self, pack, cfg):
        from types import SimpleNamespace

        from oracle import coracle
        from paper_2003_03508_b200.model import STATE_FIELDS

        out = []
        for b in range(pack.B):
            p = SimpleNamespace(gamma=pack.gamma[b], delta=pack.delta[b],
                                **{f: pack.states[i, b] for i, f in enumerate(STATE_FIELDS)})
            out.append(coracle.forward_loglik(p, *self.arrays))
        return np.array(out)


@pytest.mark.skipif(not reference_available(), reason="reference package not mounted")
def test_run_chains_reproduces_reference_trace_cpu():
    """CPU: both samplers on the C oracle's likelihood, K=5, N=400."""
    from oracle import coracle
    from paper_2003_03508_b200 import synth

    _, pr, lo, la = synth.make_workload("k5_n1e4", n=40)
    nr, na, moved = _compare(5, 40, 81, 2, lambda p: coracle.forward_loglik(p, pr, lo, la),
                             _OracleObs(pr, lo, la), alpha=1.0)
    assert moved > 0 and nr == 20 and na >= 1  # a rejuvenation move accepted on both sides


@pytest.mark.gpu
@pytest.mark.parametrize("k,n,iters,seed,alpha", [(5, 40, 81, 2, 1.0), (5, 2000, 25, 3, 0.01),
                                                  (5, 2000, 41, 7, 0.01), (25, 3000, 21, 5, 1.0)])
def test_run_chains_reproduces_reference_trace_gpu(k, n, iters, seed, alpha):
    """GPU: the reference sampler with the B200 engine in its loglik_fn hook
    vs run_chains(C=1) on the batched B200 entry point."""
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native, synth

    _native.require_device()
    _, pr, lo, la = synth.make_workload("k5_n1e4" if k == 5 else "k25_n1e6", n=n)
    dev = eng.DeviceObservations(pr, lo, la)
    nr, na, moved = _compare(k, n, iters, seed, lambda p: dev.loglik(p, eng.EngineConfig()), dev, alpha=alpha)
    print(f"K={k}: {iters} iterations, {nr} rejuvenation moves ({na} accepted), {moved} rows moved")
    assert moved > 0
    if alpha == 1.0 and k == 5:
        assert na >= 1
    dev.close()
