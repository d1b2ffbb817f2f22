"""Synthetic tremor-like inputs at the benchmark sizes.

The reference benchmark (reference bench.py:60-64) draws parameters from the
prior and simulates a path, one ``Observation`` object per hour.  At
N = 10^7..10^8 that object path is infeasible, so this module restates the
same recipe at array level and consumes the numpy ``Generator`` in exactly the
same order, which makes the arrays bit-identical to
``observation_arrays(simulate_path(params, n, rng)[1])`` (checked against the
reference in tests/test_synth.py and pinned by the checksums in
tests/golden/bench_configs.json):

* ``sample_prior_params`` -- reference bayes.py:661-687 with
  ``PriorSpec.default_for(k)`` (bayes.py:175-190, moment_match_gamma
  bayes.py:57-71): Dirichlet(0.01) rows, truncated-Gamma event probabilities
  (first ceil(K/2) states low, bayes.py:193-195), uniform means on the Shikoku
  box, inverse-Wishart(max(K, 2), I) covariances.
* ``simulate_arrays`` -- reference simforecast.py:21-61 without the objects.
* ``propose`` -- reference bayes.py:397-456, 609-653 (uniform delta), used for
  the batched-proposal workload.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import HmmParams, StateEmission

MU_BOX = (132.0, 135.0, 32.0, 35.0)


def _moment_match(mean: float, var: float):
    rate = mean / var
    return rate * mean, rate


def sample_prior_params(k: int, rng: np.random.Generator, alpha: float = 0.01) -> HmmParams:
    """Prior draw with uniform delta (the reference bench's ``delta_mode``);
    ``alpha`` = the spec's Dirichlet concentration (default_for: 0.01)."""
    from scipy.stats import invwishart

    if k < 1:
        raise ValueError("k must be a positive integer")
    gamma = np.vstack([rng.dirichlet(np.full(k, alpha)) for _ in range(k)])
    n_low = (k + 1) // 2
    low, high = _moment_match(0.1, 0.001), _moment_match(0.9, 0.001)
    lon_min, lon_max, lat_min, lat_max = MU_BOX
    df = float(max(k, 2))
    states = []
    for j in range(k):
        shape, rate = low if j < n_low else high
        while True:
            p = rng.gamma(shape, 1.0 / rate)
            if 0.0 < p < 1.0:
                break
        mu = np.array([rng.uniform(lon_min, lon_max), rng.uniform(lat_min, lat_max)])
        sigma = invwishart.rvs(df=df, scale=np.eye(2), random_state=rng)
        states.append(StateEmission(p, mu, np.asarray(sigma)))
    return HmmParams(gamma=gamma, delta=np.full(k, 1.0 / k), states=tuple(states))


def simulate_arrays(params, n: int, rng: np.random.Generator):
    """``(states, present, lon, lat)`` for an n-step path, same RNG stream as
    the reference simulator: state uniforms, event uniforms, then the
    standard-normal location noise."""
    n = int(n)
    if n < 1:
        raise ValueError("n must be a positive integer")
    k = len(params._p)
    cum_start = np.cumsum(params.delta)
    cum_rows = np.cumsum(params.gamma, axis=1)
    u_state = rng.random(n)
    u_event = rng.random(n)
    z = rng.standard_normal((n, 2))
    states = _walk(cum_start, cum_rows, u_state, k)
    present = u_event < np.asarray(params._p)[states]
    xy = np.zeros((n, 2))
    # The reference's per-state pass (simforecast.py:51-54) builds
    # `present & (states == j)` over the whole path for every state (K full
    # passes: ~60 s at K=80, N=10^8).  One stable sort of the present
    # records by state yields the same row sets in the same order, so each
    # state's `mu + z[idx] @ chol.T` is the identical BLAS call on the
    # identical matrix -- bit-identical output in one pass.
    pidx = np.flatnonzero(present)
    pst = states[pidx].astype(np.int16 if k < 32768 else np.int64)
    order = np.argsort(pst, kind="stable")
    bounds = np.searchsorted(pst[order], np.arange(k + 1), side="left")
    for j, st in enumerate(params.states):
        if bounds[j + 1] > bounds[j]:
            idx = pidx[order[bounds[j]:bounds[j + 1]]]
            xy[idx] = st.mu + z[idx] @ st.chol.T
    lon = np.where(present, xy[:, 0], 0.0)
    lat = np.where(present, xy[:, 1], 0.0)
    return states, present, np.ascontiguousarray(lon), np.ascontiguousarray(lat)


def _walk(cum_start, cum_rows, u, k):
    """Inverse-CDF state walk, ``min(searchsorted(right), K-1)`` per step.

    Sequential by nature; vectorised over a per-state lookup so 10^8 steps
    stay in numpy: for each step we only need the row of the previous state.
    """
    n = u.size
    states = np.empty(n, dtype=np.int64)
    s = min(int(np.searchsorted(cum_start, u[0], side="right")), k - 1)
    states[0] = s
    if n == 1:
        return states
    try:
        from numba import njit  # noqa: F401
        return _walk_numba(cum_rows, u, s, k, states)
    except ImportError:  # pragma: no cover - numba is in the image
        for t in range(1, n):
            s = min(int(np.searchsorted(cum_rows[s], u[t], side="right")), k - 1)
            states[t] = s
        return states


_WALK_JIT = None


def _walk_numba(cum_rows, u, s0, k, states):
    global _WALK_JIT
    if _WALK_JIT is None:
        from numba import njit

        @njit(cache=False, nogil=True)
        def walk(cum_rows, u, s0, k, states):
            s = s0
            for t in range(1, u.size):
                row = cum_rows[s]
                # searchsorted(side="right"): first index with row[i] > x
                lo, hi = 0, k
                x = u[t]
                while lo < hi:
                    mid = (lo + hi) >> 1
                    if row[mid] <= x:
                        lo = mid + 1
                    else:
                        hi = mid
                s = lo if lo < k - 1 else k - 1
                states[t] = s
            return states

        _WALK_JIT = walk
    return _WALK_JIT(np.ascontiguousarray(cum_rows), u, s0, k, states)


@dataclass(frozen=True)
class StepSizes:
    """Random-walk step sizes per block (reference bayes.py StepSizes)."""

    gamma: float = 0.25
    p: float = 0.25
    mu: float = 0.01
    sigma: float = 0.05


def _prop_gamma(gamma, step, rng):
    k = gamma.shape[0]
    logg = np.log(gamma)
    z = logg - logg.mean(axis=1, keepdims=True)
    z = z + step * rng.standard_normal((k, k))
    z -= z.max(axis=1, keepdims=True)
    new = np.exp(z)
    new /= new.sum(axis=1, keepdims=True)
    if np.any(new <= 0.0):
        raise ValueError("proposed transition row underflowed to the simplex boundary")
    return new


def _prop_p(ps, step, rng):
    u = np.log(ps) - np.log1p(-ps) + step * rng.standard_normal(ps.size)
    new = 1.0 / (1.0 + np.exp(-u))
    if np.any(new <= 0.0) or np.any(new >= 1.0):
        raise ValueError("proposed event probability left (0, 1)")
    return new


def _prop_sigma(states, step, rng):
    noise = step * rng.standard_normal((len(states), 3))
    out = []
    for st, eps in zip(states, noise):
        l00 = math.exp(math.log(st.chol[0, 0]) + eps[0])
        b = st.chol[1, 0] + eps[1]
        l11 = math.exp(math.log(st.chol[1, 1]) + eps[2])
        out.append(np.array([[l00 * l00, l00 * b], [l00 * b, b * b + l11 * l11]]))
    return out


def propose(params: HmmParams, steps: StepSizes, rng: np.random.Generator) -> HmmParams:
    """One full-sweep random-walk proposal (blocks gamma, p, mu, sigma in
    that order), uniform delta; the Jacobian term is not needed here."""
    out = params
    if steps.gamma != 0.0:
        g = _prop_gamma(out.gamma, steps.gamma, rng)
        out = HmmParams(gamma=g, delta=np.full(g.shape[0], 1.0 / g.shape[0]), states=out.states)
    if steps.p != 0.0:
        ps = _prop_p(np.asarray(out._p), steps.p, rng)
        out = HmmParams(gamma=out.gamma, delta=out.delta,
                        states=tuple(StateEmission(p, s.mu, s.sigma) for p, s in zip(ps, out.states)))
    if steps.mu != 0.0:
        mus = np.stack([s.mu for s in out.states])
        mus = mus + steps.mu * rng.standard_normal(mus.shape)
        out = HmmParams(gamma=out.gamma, delta=out.delta,
                        states=tuple(StateEmission(s.p, m, s.sigma) for m, s in zip(mus, out.states)))
    if steps.sigma != 0.0:
        sig = _prop_sigma(out.states, steps.sigma, rng)
        out = HmmParams(gamma=out.gamma, delta=out.delta,
                        states=tuple(StateEmission(s.p, s.mu, sg) for sg, s in zip(sig, out.states)))
    return out


# Benchmark workloads of BASELINE.json "configs" (seed per K as in SURVEY.md §8d).
WORKLOADS = {
    "k5_n1e4": dict(k=5, n=10_000, seed=0, batch=1),
    "k25_n1e6": dict(k=25, n=1_000_000, seed=25, batch=1),
    "k50_n1e7": dict(k=50, n=10_000_000, seed=50, batch=1),
    "k80_n1e8": dict(k=80, n=100_000_000, seed=80, batch=1),
    "k25_n1e6_b256": dict(k=25, n=1_000_000, seed=256, batch=256),
}

BATCH_STEPS = StepSizes(0.1, 0.1, 0.005, 0.02)


def make_workload(name: str, n: int | None = None):
    """``(params_list, present, lon, lat)`` for a named workload.

    Single-eval workloads: one prior draw then the simulated path from the
    same generator.  The batched workload mixes the draw to strict positivity
    (``0.999 Gamma + 0.001/K``, needed by the log-ratio proposal), simulates
    the path from it, then draws ``batch`` proposals around it.
    """
    w = WORKLOADS[name]
    k, seed, batch = w["k"], w["seed"], w["batch"]
    n = w["n"] if n is None else int(n)
    rng = np.random.default_rng(seed)
    base = sample_prior_params(k, rng)
    if batch == 1:
        _, present, lon, lat = simulate_arrays(base, n, rng)
        return [base], present, lon, lat
    mixed = HmmParams(gamma=0.999 * base.gamma + 0.001 / k, delta=base.delta, states=base.states)
    _, present, lon, lat = simulate_arrays(mixed, n, rng)
    props = [propose(mixed, BATCH_STEPS, rng) for _ in range(batch)]
    return props, present, lon, lat
