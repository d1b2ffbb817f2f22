"""Seeded random instances, restating the reference test fixtures.

``random_params`` / ``random_obs_arrays`` follow reference
pkg/tests/test_core.py:25-47 (``random_spd``, ``random_params``,
``random_obs``) and consume the numpy Generator in the same order, so a seed
gives the same instance as the reference test suite.  tests/test_oracle.py
checks the equality against the reference when it is importable, and the
golden files pin the generated inputs by checksum so the GPU box (which has
no reference) regenerates exactly the instances the goldens were made from.
"""

from __future__ import annotations

import hashlib

import numpy as np

from paper_2003_03508_b200.model import HmmParams, StateEmission


def random_spd(rng, scale=1.0):
    a = rng.standard_normal((2, 2))
    return scale * (a @ a.T + 0.3 * np.eye(2))


def random_params(rng, k, p_range=(0.05, 0.95), sigma_scale=0.5):
    gamma = rng.dirichlet(np.full(k, 5.0), size=k)
    delta = rng.dirichlet(np.full(k, 5.0))
    states = tuple(
        StateEmission(rng.uniform(*p_range), rng.uniform(-1.0, 1.0, size=2), random_spd(rng, sigma_scale))
        for _ in range(k))
    return HmmParams(gamma=gamma, delta=delta, states=states)


def random_obs_arrays(rng, n, present_prob=0.6, spread=1.5):
    """Array form of reference ``random_obs`` (same RNG consumption)."""
    present = np.zeros(n, dtype=bool)
    lon = np.zeros(n)
    lat = np.zeros(n)
    for i in range(n):
        if rng.random() < present_prob:
            x = rng.uniform(-spread, spread, size=2)
            present[i] = True
            lon[i], lat[i] = float(x[0]), float(x[1])
    return present, lon, lat


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()[:24]


def params_digest(p) -> str:
    return digest(np.asarray(p.gamma), np.asarray(p.delta), np.asarray(p._p), np.asarray(p._mu0),
                  np.asarray(p._mu1), np.asarray(p._l00), np.asarray(p._l10), np.asarray(p._l11))


def criterion1_instances():
    """The 200 seeded instances of reference acceptance criterion 1
    (test_acceptance.py:93-122): yields (k, n, segments, params, present, lon, lat)."""
    import math

    rng = np.random.default_rng(20260814)
    for _ in range(200):
        k = int(rng.integers(2, 51))
        n = min(10_000, max(1, int(round(math.exp(rng.uniform(0.0, math.log(1e4)))))))
        params = random_params(rng, k)
        present, lon, lat = random_obs_arrays(rng, n)
        segments = int(rng.integers(1, min(8, n) + 1))
        yield k, n, segments, params, present, lon, lat
