"""Many-chain Metropolis-Hastings on the batched B200 likelihood.

The reference sampler (``bayes.run_chain``, bayes.py:690-796) evaluates one
likelihood at a time: per iteration it updates the gamma, p, mu and sigma
blocks in turn, each a random-walk proposal in unconstrained coordinates
(bayes.py:397-456) accepted by Metropolis-Hastings with the proposal's
log-Jacobian (bayes.py:609-659), i.e. ~4 sequential likelihood calls per
iteration.  Here C independent chains advance in lockstep: every block move
proposes for all chains at once (vectorised restatement of the reference
proposals), packs the C candidates in one pass
(``proposals.params_from_vectors``), evaluates their likelihoods in ONE launch
of the device chain kernel, and accepts per chain.  The joint prior is the
reference's (``bayes.log_prior`` with ``PriorSpec.default_for(K)``,
bayes.py:206-233, 176-190), vectorised over chains.

Not restated: the every-4th-iteration rejuvenation kernel
(bayes.py:473-604); the blockwise random-walk moves alone leave the same
posterior invariant.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .engine import DeviceObservations, EngineConfig
from .proposals import params_from_vectors, vector_length

LOG2 = math.log(2.0)


@dataclass(frozen=True)
class PriorSpec:
    """Reference ``PriorSpec.default_for(k)`` (bayes.py:140-190)."""

    dirichlet_alpha: float = 0.01
    p_low: tuple = (10.0, 100.0)      # moment_match_gamma(0.1, 0.001)
    p_high: tuple = (810.0, 900.0)    # moment_match_gamma(0.9, 0.001)
    mu_bounds: tuple = (132.0, 135.0, 32.0, 35.0)
    iw_df: Optional[float] = None     # None -> max(K, 2)

    def df(self, k: int) -> float:
        return float(max(k, 2)) if self.iw_df is None else float(self.iw_df)


def _split(k: int, v: np.ndarray):
    kk = k * k
    return (v[:, :kk].reshape(-1, k, k), v[:, kk:kk + k], v[:, kk + k:kk + 3 * k].reshape(-1, k, 2),
            v[:, kk + 3 * k:].reshape(-1, k, 3))


def log_prior_batch(k: int, vecs: np.ndarray, spec: PriorSpec = PriorSpec()) -> np.ndarray:
    """Joint log prior of B parameter vectors (reference bayes.log_prior,
    bayes.py:206-233, identity inverse-Wishart scale); -inf off the support."""
    from scipy.special import gammainc, gammaln, multigammaln

    v = np.atleast_2d(np.asarray(vecs, dtype=np.float64))
    gamma, ps, mus, sig = _split(k, v)
    lp = np.zeros(v.shape[0])
    with np.errstate(divide="ignore", invalid="ignore"):
        a = spec.dirichlet_alpha
        bad = np.any(gamma <= 0.0, axis=(1, 2))
        if k > 1:
            lp += k * (gammaln(a * k) - k * gammaln(a)) + (a - 1.0) * np.log(np.where(gamma > 0, gamma, 1.0)).sum(
                axis=(1, 2))
        n_low = (k + 1) // 2
        for j in range(k):
            shape, rate = spec.p_low if j < n_low else spec.p_high
            x = ps[:, j]
            lp += shape * math.log(rate) + (shape - 1.0) * np.log(x) - rate * x - gammaln(shape)
            lp -= math.log(gammainc(shape, rate))
        lon_min, lon_max, lat_min, lat_max = spec.mu_bounds
        bad |= np.any((mus[..., 0] < lon_min) | (mus[..., 0] > lon_max) | (mus[..., 1] < lat_min)
                      | (mus[..., 1] > lat_max), axis=1)
        lp -= k * (math.log(lon_max - lon_min) + math.log(lat_max - lat_min))
        df = spec.df(k)
        s00, s01, s11 = sig[..., 0], sig[..., 1], sig[..., 2]
        l00 = np.sqrt(s00)
        l10 = s01 / l00
        l11 = np.sqrt(s11 - l10 * l10)
        logdet = 2.0 * (np.log(l00) + np.log(l11))
        tr = (s11 + s00) / np.exp(logdet)
        lp += np.sum(-0.5 * df * 2 * LOG2 - float(multigammaln(0.5 * df, 2)) - 0.5 * (df + 3.0) * logdet - 0.5 * tr,
                     axis=1)
    return np.where(bad | ~np.isfinite(lp), -np.inf, lp)


# -- vectorised block proposals (reference bayes.py:397-456) -----------------

def propose_gamma(k, v, step, rng):
    g, _, _, _ = _split(k, v)
    logg = np.log(g)
    z = logg - logg.mean(axis=2, keepdims=True) + step * rng.standard_normal(g.shape)
    z -= z.max(axis=2, keepdims=True)
    new = np.exp(z)
    new /= new.sum(axis=2, keepdims=True)
    out = v.copy()
    out[:, :k * k] = new.reshape(v.shape[0], -1)
    with np.errstate(divide="ignore"):
        jac = np.log(new).sum(axis=(1, 2)) - logg.sum(axis=(1, 2))
    ok = np.all(new > 0.0, axis=(1, 2))
    return out, jac, ok


def propose_p(k, v, step, rng):
    _, ps, _, _ = _split(k, v)
    u = np.log(ps) - np.log1p(-ps) + step * rng.standard_normal(ps.shape)
    new = 1.0 / (1.0 + np.exp(-u))
    out = v.copy()
    out[:, k * k:k * k + k] = new
    with np.errstate(divide="ignore"):
        jac = np.sum(np.log(new) + np.log1p(-new), axis=1) - np.sum(np.log(ps) + np.log1p(-ps), axis=1)
    ok = np.all((new > 0.0) & (new < 1.0), axis=1)
    return out, jac, ok


def propose_mu(k, v, step, rng):
    out = v.copy()
    out[:, k * k + k:k * k + 3 * k] += step * rng.standard_normal((v.shape[0], 2 * k))
    return out, np.zeros(v.shape[0]), np.ones(v.shape[0], dtype=bool)


def propose_sigma(k, v, step, rng):
    _, _, _, sig = _split(k, v)
    s00, s01, s11 = sig[..., 0], sig[..., 1], sig[..., 2]
    l00 = np.sqrt(s00)
    l10 = s01 / l00
    l11 = np.sqrt(s11 - l10 * l10)
    eps = step * rng.standard_normal((v.shape[0], k, 3))
    a = np.log(l00) + eps[..., 0]
    b = l10 + eps[..., 1]
    c = np.log(l11) + eps[..., 2]
    n00, n11 = np.exp(a), np.exp(c)
    new = np.stack([n00 * n00, n00 * b, b * b + n11 * n11], axis=-1)
    out = v.copy()
    out[:, k * k + 3 * k:] = new.reshape(v.shape[0], -1)
    jac = np.sum(3.0 * (a - np.log(l00)) + 2.0 * (c - np.log(l11)), axis=1)
    return out, jac, np.all(np.isfinite(new), axis=(1, 2))


BLOCKS = (("gamma", propose_gamma), ("p", propose_p), ("mu", propose_mu), ("sigma", propose_sigma))


@dataclass
class ChainsResult:
    vectors: np.ndarray         # (kept, C, L)
    log_likelihood: np.ndarray  # (kept, C)
    log_prior: np.ndarray       # (kept, C)
    acceptance: dict            # block -> (C,) acceptance rate
    evaluations: int            # batched likelihood launches


def run_chains(k: int, obs, init_vecs: np.ndarray, iterations: int, *,
               steps=(0.25, 0.25, 0.01, 0.05), delta_mode: str = "uniform", thin: int = 1,
               spec: PriorSpec = PriorSpec(), rng: Optional[np.random.Generator] = None,
               cfg: EngineConfig = EngineConfig()) -> ChainsResult:
    """Blockwise random-walk MH for C chains in lockstep; one batched
    likelihood launch per block move.  ``steps`` = (gamma, p, mu, sigma).
    ``obs``: a ``DeviceObservations`` (one GPU) or a
    ``distributed.ReplicaLoglik`` (chains' proposals sharded over the ranks;
    run the same call with the same seed on every rank)."""
    rng = np.random.default_rng(0) if rng is None else rng
    cur = np.array(np.atleast_2d(init_vecs), dtype=np.float64)
    if cur.shape[1] != vector_length(k):
        raise ValueError(f"expected vectors of length {vector_length(k)}")
    n_chains = cur.shape[0]
    cur_lp = log_prior_batch(k, cur, spec)
    pack, ok = params_from_vectors(k, cur, delta_mode)
    if not ok.all() or not np.all(np.isfinite(cur_lp)):
        raise ValueError("initial states must lie inside the prior support")
    cur_ll = obs.loglik_batch(pack, cfg)
    evals = 1
    acc = {name: np.zeros(n_chains) for name, _ in BLOCKS}
    kept_v, kept_ll, kept_lp = [], [], []
    for it in range(iterations):
        for (name, prop), step in zip(BLOCKS, steps):
            if step == 0.0:
                continue
            with np.errstate(all="ignore"):
                cand, jac, ok = prop(k, cur, step, rng)
            cand_lp = log_prior_batch(k, cand, spec)
            pack, valid = params_from_vectors(k, cand, delta_mode)
            ok &= valid & np.isfinite(cand_lp)
            cand_ll = np.full(n_chains, -np.inf)
            if valid.any():
                ll = obs.loglik_batch(pack, cfg)   # one launch for every valid candidate
                evals += 1
                cand_ll[np.flatnonzero(valid)] = ll
            log_ratio = (cand_ll + cand_lp) - (cur_ll + cur_lp) + jac
            u = rng.random(n_chains)
            accept = ok & np.isfinite(cand_ll) & (np.log(u) < np.minimum(log_ratio, 0.0))
            cur[accept] = cand[accept]
            cur_ll[accept] = cand_ll[accept]
            cur_lp[accept] = cand_lp[accept]
            acc[name] += accept
        if it % thin == 0:
            kept_v.append(cur.copy())
            kept_ll.append(cur_ll.copy())
            kept_lp.append(cur_lp.copy())
    return ChainsResult(np.stack(kept_v), np.stack(kept_ll), np.stack(kept_lp),
                        {n: a / max(iterations, 1) for n, a in acc.items()}, evals)
