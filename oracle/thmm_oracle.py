"""CPU oracle for the HMM forward log-likelihood -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_2003_03508_b200``) never imports anything under ``oracle/``.

It restates, in numpy, the reference algorithm of ``tremorhmm`` (paths
relative to /root/reference/pkg/src/tremorhmm):

* ``emission_columns``      core.py:235-260 (``_emission_columns``)
* ``forward_loglik_arrays`` core.py:270-302 (``_forward_loglik_arrays``,
                            the paper's Algorithm 1)
* ``segment_bounds``        engine.py:97-111
* ``chain_segment``         engine.py:124-179 (``_chain_fused_*`` + ``_finish``)
* ``combine_segments``      engine.py:292-318
* ``parallel_loglik_arrays`` engine.py:321-345 (streamed per segment, so the
                            N x K emission table is never materialised whole)
* ``brute_force_loglik``    core.py:321-347

Parity of this restatement is pinned against the reference itself: the
golden fixtures under tests/golden/ were produced by importing the reference
package (script: oracle/gen_golden.py) and tests/test_oracle.py checks this
module (and the C restatement in thmm_oracle.c) against them.

Parameters are duck-typed: anything with the reference ``HmmParams``
attributes (``gamma, delta, _p, _q, _mu0, _mu1, _l00, _l10, _l11, _log_det``).
"""

from __future__ import annotations

import math

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)


def emission_columns(params, present, lon, lat):
    """(n, K) emission diagonals; core.py:235-260.  Divisions (not
    reciprocals) and the same operation order as the reference."""
    n = present.size
    k = len(params._p)
    out = np.empty((n, k), dtype=np.float64)
    absent = ~present
    if absent.any():
        out[absent, :] = params._q
    if present.any():
        x = lon[present]
        y = lat[present]
        cols = np.empty((x.size, k), dtype=np.float64)
        for j in range(k):
            z0 = (x - params._mu0[j]) / params._l00[j]
            z1 = ((y - params._mu1[j]) - params._l10[j] * z0) / params._l11[j]
            cols[:, j] = params._p[j] * np.exp(
                -LOG_2PI - 0.5 * params._log_det[j] - 0.5 * (z0 * z0 + z1 * z1))
        out[present, :] = cols
    return out


def forward_loglik_arrays(params, present, lon, lat, renorm_period=1):
    """Serial scaled forward recursion; core.py:270-302.

    ``v <- (v Gamma) * e_t``; every ``renorm_period`` steps divide by max(v)
    and accumulate its log.  Returns -inf on total collapse.
    """
    if present.size == 0:
        raise ValueError("observation sequence is empty")
    if renorm_period < 1:
        raise ValueError("renorm_period must be a positive integer")
    gamma = np.asarray(params.gamma, dtype=np.float64)
    v = np.array(params.delta, dtype=np.float64)
    acc = 0.0
    since = 0
    for t in range(present.size):
        v = v @ gamma
        if present[t]:
            z0 = (lon[t] - params._mu0) / params._l00
            z1 = ((lat[t] - params._mu1) - params._l10 * z0) / params._l11
            v = v * (params._p * np.exp(
                -LOG_2PI - 0.5 * params._log_det - 0.5 * (z0 * z0 + z1 * z1)))
        else:
            v = v * params._q
        since += 1
        if since == renorm_period:
            since = 0
            top = v.max()
            if top <= 0.0:
                return -math.inf
            acc += math.log(top)
            v /= top
    total = v.sum()
    if total <= 0.0:
        return -math.inf
    return math.log(total) + acc


def segment_bounds(n, segments):
    """Contiguous near-equal blocks, earlier blocks larger; engine.py:97-111."""
    if n < 1:
        raise ValueError("n must be positive")
    if not 1 <= segments <= n:
        raise ValueError("segments must lie in [1, n]")
    base, extra = divmod(n, segments)
    out, lo = [], 0
    for i in range(segments):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def chain_segment(gamma, ediag, period):
    """Scaled product of Gamma diag(e_t) over the rows of ``ediag``;
    engine.py:133-179 followed by ``_finish`` (engine.py:124-130).

    Returns ``(m, log_scale)`` with max(m) == 1 (or m all zero)."""
    m = gamma * ediag[0]
    log_scale = 0.0
    since = 0
    for t in range(1, ediag.shape[0]):
        m = (m @ gamma) * ediag[t]
        since += 1
        if since == period:
            since = 0
            top = m.max()
            if top > 0.0:
                log_scale += math.log(float(top))
                m = m / top
    top = m.max()
    if top > 0.0 and top != 1.0:
        log_scale += math.log(float(top))
        m = m / top
    return m, log_scale


def combine_segments(delta, parts):
    """Ordered host fold; engine.py:292-318.  ``parts`` is a list of
    ``(lo, hi, m, log_scale)``.  Raises RuntimeError on collapse and
    ValueError on a gap."""
    if len(parts) == 0:
        raise ValueError("no segment products to combine")
    order = sorted(parts, key=lambda s: s[0])
    for a, b in zip(order, order[1:]):
        if a[1] != b[0]:
            raise ValueError("segment products must tile the chain contiguously")
    v = np.array(delta, dtype=np.float64)
    acc = 0.0
    for _, _, m, log_scale in order:
        v = v @ m
        acc += log_scale
        top = v.max()
        if top <= 0.0:
            raise RuntimeError("running state vector collapsed to zero while combining segments")
        acc += math.log(float(top))
        v = v / top
    return math.log(float(v.sum())) + acc


def segment_products(params, present, lon, lat, segments, period=8):
    """Per-segment ``(lo, hi, m, log_scale)``; emissions evaluated per segment."""
    gamma = np.ascontiguousarray(params.gamma, dtype=np.float64)
    out = []
    for lo, hi in segment_bounds(present.size, min(segments, present.size)):
        ed = emission_columns(params, present[lo:hi], lon[lo:hi], lat[lo:hi])
        m, ls = chain_segment(gamma, ed, period)
        out.append((lo, hi, m, ls))
    return out


def parallel_loglik_arrays(params, present, lon, lat, segments=1, period=8):
    """Segmented engine result; engine.py:321-345."""
    if present.size == 0:
        raise ValueError("observation sequence is empty")
    return combine_segments(params.delta, segment_products(params, present, lon, lat, segments, period))


def brute_force_loglik(params, present, lon, lat):
    """Path enumeration in log space (core.py:321-347); tiny instances only."""
    from scipy.special import logsumexp

    n = present.size
    k = len(params._p)
    if n == 0:
        raise ValueError("observation sequence is empty")
    if float(k) ** (n + 1) > 1_000_000:
        raise ValueError("too many hidden paths to enumerate")
    ed = emission_columns(params, present, lon, lat)
    with np.errstate(divide="ignore"):
        lg = np.log(np.asarray(params.gamma))
        le = np.log(ed)
        lp = np.log(np.asarray(params.delta))[None, :]
    for t in range(n):
        lp = (lp[:, :, None] + lg[None, :, :] + le[t][None, None, :]).reshape(-1, k)
    return float(logsumexp(lp))


def stationary_distribution(gamma, tol=1e-12, max_iter=100_000):
    """Power iteration from the uniform vector (reference core.py:350-388)."""
    gamma = np.ascontiguousarray(gamma, dtype=np.float64)
    k = gamma.shape[0]
    pi = np.full(k, 1.0 / k)
    for _ in range(max_iter):
        nxt = pi @ gamma
        nxt /= nxt.sum()
        if np.max(np.abs(nxt - pi)) < tol:
            return nxt
        pi = nxt
    raise RuntimeError("power iteration did not reach the stationary distribution")


def filtered_next_state(params, present, lon, lat):
    """Filtered distribution one step past the history; reference
    simforecast.py:97-118 (sum-normalised forward recursion, then one Gamma)."""
    if present.size == 0:
        raise ValueError("history is empty")
    ed = emission_columns(params, present, lon, lat)
    gamma = np.asarray(params.gamma, dtype=np.float64)
    v = np.array(params.delta, dtype=np.float64)
    for t in range(present.size):
        v = (v @ gamma) * ed[t]
        s = v.sum()
        if s <= 0.0:
            raise RuntimeError("history has zero likelihood under these parameters")
        v /= s
    v = v @ gamma
    return v / v.sum()
