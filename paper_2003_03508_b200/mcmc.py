"""Many-chain Metropolis-Hastings on the batched B200 likelihood.

The reference sampler (``bayes.run_chain``, bayes.py:690-796) evaluates one
likelihood at a time: per iteration it updates the gamma, p, mu and sigma
blocks in turn, each a random-walk proposal in unconstrained coordinates
(bayes.py:397-456) accepted by Metropolis-Hastings with the proposal's
log-Jacobian (bayes.py:609-659), and every REJUVENATE_PERIOD-th iteration a
joint independence move for one state (``_RejuvenationKernel``,
bayes.py:472-604, 746-754), i.e. ~4.25 sequential likelihood calls per
iteration.  Here C chains advance in lockstep: every move proposes for all
chains at once (vectorised restatement of the reference proposals), packs the
C candidates in one pass (``proposals.params_from_vectors``), evaluates their
likelihoods in ONE launch of the device chain kernel, and accepts per chain.
The joint prior is the reference's (``bayes.log_prior`` with
``PriorSpec.default_for(K)``, bayes.py:206-233, 176-190), vectorised over
chains.

Schedule and random stream follow ``run_chain`` exactly: iteration 0 is the
initial state, sweeps run for it = 1 .. iterations-1, the rejuvenation move
for state (it // 4) % K follows the four blocks when it % 4 == 0, and the
shared generator is consumed in the reference's order (chain by chain where
the reference draws per chain; an accept uniform only for candidates that
reach the Metropolis-Hastings test).  With C = 1 and the reference's seed the
trace is the reference's (tests/test_gpu_mcmc_trace.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .engine import DeviceObservations, EngineConfig
from .proposals import params_from_vectors, vector_length

LOG2 = math.log(2.0)
LOG_2PI = math.log(2.0 * math.pi)
REJUVENATE_PERIOD = 4       # reference bayes.py:54
INIT_MAX_REDRAWS = 1000     # reference bayes.py:44


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


# -- batched rejuvenation move (reference _RejuvenationKernel, bayes.py:472-604) --

def _logsumexp(x, axis):
    m = np.max(x, axis=axis, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore"):
        return np.squeeze(m, axis=axis) + np.log(np.sum(np.exp(x - m), axis=axis))


def _iw_logpdf(s00, s01, s11, df, scale):
    """Reference invwishart_logpdf (bayes.py:112-140) over arrays of 2x2 SPD
    matrices given by (s00, s01, s11)."""
    from scipy.special import multigammaln

    l00 = np.sqrt(s00)
    l10 = s01 / l00
    l11 = np.sqrt(s11 - l10 * l10)
    logdet = 2.0 * (np.log(l00) + np.log(l11))
    c00 = math.sqrt(scale[0, 0])
    c10 = scale[1, 0] / c00
    c11 = math.sqrt(scale[1, 1] - c10 * c10)
    logdet_scale = 2.0 * (math.log(c00) + math.log(c11))
    det = np.exp(logdet)
    tr = (scale[0, 0] * s11 - scale[0, 1] * s01 - scale[1, 0] * s01 + scale[1, 1] * s00) / det
    return (0.5 * df * logdet_scale - 0.5 * df * 2 * LOG2 - float(multigammaln(0.5 * df, 2))
            - 0.5 * (df + 3.0) * logdet - 0.5 * tr)


class Rejuvenator:
    """Joint independence proposal for one state's (p, mu, Sigma) plus the
    whole transition matrix, for C chains at once (reference
    ``_RejuvenationKernel``, bayes.py:472-604, same mixture components,
    constants and draw order).  Draws are per chain in chain order from the
    shared generator (the reference's sequence at C = 1); the log q-ratios of
    all chains are evaluated together."""

    GAMMA_CONC = 20.0
    GAMMA_DIAG_BOOST = 6.0
    GAMMA_WEIGHTS = (0.4, 0.3, 0.3)  # uniform, diagonal-boosted, concentrated
    MU_KDE_WEIGHT = 0.7
    MU_KDE_BW = 0.15
    MU_POINTS = 512
    SIGMA_SHARP_DF = 6.0
    SIGMA_BROAD_DF = 2.1

    def __init__(self, spec: "PriorSpec", points: Optional[tuple] = None):
        self.spec = spec
        lon_min, lon_max, lat_min, lat_max = spec.mu_bounds
        self.log_area = math.log(lon_max - lon_min) + math.log(lat_max - lat_min)
        pts = np.zeros((0, 2))
        if points is not None:  # (present, lon, lat): the observed event locations
            pr, lo, la = (np.asarray(a) for a in points)
            pr = pr.astype(bool)
            pts = np.stack([lo[pr], la[pr]], axis=1).astype(np.float64)
            if len(pts) > self.MU_POINTS:
                stride = len(pts) / self.MU_POINTS
                pts = pts[(np.arange(self.MU_POINTS) * stride).astype(int)]
        self.points = pts
        scale = 0.05 * min(lon_max - lon_min, lat_max - lat_min)
        self.sigma_sharp_scale = (self.SIGMA_SHARP_DF - 3.0) * scale * scale * np.eye(2)
        self.sigma_broad_scale = np.eye(2)
        self._cumw = np.cumsum(self.GAMMA_WEIGHTS)

    # -- draws (per chain, reference order) ---------------------------------
    def _draw_gamma(self, old, rng):
        k = old.shape[0]
        rows = []
        for i in range(k):
            which = int(np.searchsorted(self._cumw, rng.random(), side="right"))
            which = min(which, 2)
            if which == 0:
                alpha = np.ones(k)
            elif which == 1:
                alpha = np.ones(k)
                alpha[i] += self.GAMMA_DIAG_BOOST
            else:
                alpha = self.GAMMA_CONC * old[i] + 1.0
            rows.append(rng.dirichlet(alpha))
        return np.vstack(rows)

    def _draw_mu(self, rng):
        lon_min, lon_max, lat_min, lat_max = self.spec.mu_bounds
        if len(self.points) > 0 and rng.random() < self.MU_KDE_WEIGHT:
            center = self.points[rng.integers(len(self.points))]
            return center + self.MU_KDE_BW * rng.standard_normal(2)
        return np.array([rng.uniform(lon_min, lon_max), rng.uniform(lat_min, lat_max)])

    def _draw_sigma(self, rng):
        from scipy.stats import invwishart

        if rng.random() < 0.5:
            return np.asarray(invwishart.rvs(df=self.SIGMA_SHARP_DF, scale=self.sigma_sharp_scale,
                                             random_state=rng))
        return np.asarray(invwishart.rvs(df=self.SIGMA_BROAD_DF, scale=self.sigma_broad_scale, random_state=rng))

    def _draw_p(self, j, k, rng):
        shape, rate = self.spec.p_low if j < (k + 1) // 2 else self.spec.p_high
        while True:
            p = rng.gamma(shape, 1.0 / rate)
            if 0.0 < p < 1.0:
                return p

    # -- proposal densities (all chains at once) ----------------------------
    def _log_q_gamma(self, new, old):
        """sum_i logsumexp_c(log w_c + Dirichlet(new_i; alpha_c(i, old_i))), (C,)"""
        from scipy.special import gammaln

        c, k, _ = new.shape
        alphas = np.empty((c, k, 3, k))
        alphas[:, :, 0, :] = 1.0
        alphas[:, :, 1, :] = 1.0
        alphas[:, np.arange(k), 1, np.arange(k)] += self.GAMMA_DIAG_BOOST
        alphas[:, :, 2, :] = self.GAMMA_CONC * old + 1.0
        x = new[:, :, None, :]
        with np.errstate(divide="ignore", invalid="ignore"):
            terms = np.where(alphas == 1.0, 0.0, (alphas - 1.0) * np.log(x))
        logpdf = gammaln(alphas.sum(axis=3)) - gammaln(alphas).sum(axis=3) + terms.sum(axis=3)
        comps = np.log(np.asarray(self.GAMMA_WEIGHTS))[None, None, :] + logpdf
        return _logsumexp(comps, axis=2).sum(axis=1)

    def _log_q_mu(self, mu):
        log_uniform = -self.log_area
        if len(self.points) == 0:
            return np.full(mu.shape[0], log_uniform)
        d = (self.points[None, :, :] - mu[:, None, :]) / self.MU_KDE_BW
        comps = -LOG_2PI - 2.0 * math.log(self.MU_KDE_BW) - 0.5 * (d * d).sum(axis=2)
        log_kde = _logsumexp(comps, axis=1) - math.log(len(self.points))
        return np.logaddexp(math.log(self.MU_KDE_WEIGHT) + log_kde, math.log1p(-self.MU_KDE_WEIGHT) + log_uniform)

    def _log_q_sigma(self, sig):
        s00, s01, s11 = sig[:, 0], sig[:, 1], sig[:, 2]
        sharp = _iw_logpdf(s00, s01, s11, self.SIGMA_SHARP_DF, self.sigma_sharp_scale)
        broad = _iw_logpdf(s00, s01, s11, self.SIGMA_BROAD_DF, self.sigma_broad_scale)
        return np.logaddexp(sharp, broad) - LOG2

    def _log_q_p(self, p, j, k):
        from scipy.special import gammainc, gammaln

        shape, rate = self.spec.p_low if j < (k + 1) // 2 else self.spec.p_high
        return (shape * math.log(rate) + (shape - 1.0) * np.log(p) - rate * p - float(gammaln(shape))
                - math.log(float(gammainc(shape, rate))))

    def propose(self, k: int, v: np.ndarray, j: int, rng: np.random.Generator):
        """Candidates for state j of every chain: (cand, log q-ratio, ok)."""
        c = v.shape[0]
        gam, ps, mus, sig = _split(k, v)
        out = v.copy()
        new_g = np.empty((c, k, k))
        new_mu = np.empty((c, 2))
        new_sig = np.empty((c, 3))
        new_p = np.empty(c)
        ok = np.ones(c, dtype=bool)
        for ch in range(c):  # the reference's draw order, chain after chain
            new_g[ch] = self._draw_gamma(gam[ch], rng)
            new_mu[ch] = self._draw_mu(rng)
            s = self._draw_sigma(rng)
            new_sig[ch] = (s[0, 0], s[0, 1], s[1, 1])
            ok[ch] = abs(s[0, 1] - s[1, 0]) <= 1e-12 * max(1.0, abs(s[0, 1]), abs(s[1, 0]))
            new_p[ch] = self._draw_p(j, k, rng)
        gv, pv, mv, sv = _split(k, out)
        gv[:] = new_g
        pv[:, j] = new_p
        mv[:, j] = new_mu
        sv[:, j] = new_sig
        with np.errstate(all="ignore"):
            log_fwd = (self._log_q_gamma(new_g, gam) + self._log_q_mu(new_mu) + self._log_q_sigma(new_sig)
                       + self._log_q_p(new_p, j, k))
            log_rev = (self._log_q_gamma(gam, new_g) + self._log_q_mu(mus[:, j]) + self._log_q_sigma(sig[:, j])
                       + self._log_q_p(ps[:, j], j, k))
        return out, log_rev - log_fwd, ok


# -- the sampler -------------------------------------------------------------

@dataclass
class ChainsResult:
    vectors: np.ndarray         # (kept, C, L); row 0 = the initial states (iteration 0)
    log_likelihood: np.ndarray  # (kept, C)
    log_prior: np.ndarray       # (kept, C)
    acceptance: dict            # block -> (C,) acceptance rate (accepted / proposed)
    evaluations: int            # batched likelihood launches
    iterations: np.ndarray = None  # (kept,) iteration index of each kept row
    accepted: dict = None       # block -> (C,) accepted moves
    proposed: dict = None       # block -> proposals made (same for every chain)


def init_from_prior(k: int, n_chains: int, obs, rng: np.random.Generator, *, spec: "PriorSpec" = None,
                    delta_mode: str = "uniform", cfg: EngineConfig = EngineConfig()):
    """Initial states as the reference draws them (bayes.py:717-733): a prior
    draw per chain, redrawn (up to INIT_MAX_REDRAWS times) until its prior
    and likelihood are finite; the likelihoods of all pending chains are
    evaluated in one launch per round.  Returns (vectors (C, L), log_lik (C,))."""
    from .proposals import params_to_vectors
    from .synth import sample_prior_params

    spec = PriorSpec() if spec is None else spec
    if delta_mode != "uniform":
        raise ValueError("init_from_prior draws delta_mode='uniform' (the reference bench setting)")
    vecs = np.empty((n_chains, vector_length(k)))
    ll = np.full(n_chains, -np.inf)
    pending = np.arange(n_chains)
    for _ in range(INIT_MAX_REDRAWS):
        if spec.iw_df is not None and spec.df(k) != float(max(k, 2)):
            raise ValueError("init_from_prior draws the default inverse-Wishart df = max(K, 2)")
        draws = params_to_vectors([sample_prior_params(k, rng, spec.dirichlet_alpha) for _ in pending])
        lp = log_prior_batch(k, draws, spec)
        pack, valid = params_from_vectors(k, draws, delta_mode)
        cand_ll = np.full(len(pending), -np.inf)
        sel = valid & np.isfinite(lp)
        if sel.any():
            pk, _ = params_from_vectors(k, draws[sel], delta_mode)
            cand_ll[sel] = obs.loglik_batch(pk, cfg)
        good = np.isfinite(cand_ll)
        vecs[pending[good]] = draws[good]
        ll[pending[good]] = cand_ll[good]
        pending = pending[~good]
        if pending.size == 0:
            return vecs, ll
    raise RuntimeError(f"no prior draw with finite posterior after {INIT_MAX_REDRAWS} attempts")


def run_chains(k: int, obs, init_vecs: np.ndarray, iterations: int, *,
               steps=(0.25, 0.25, 0.01, 0.05), delta_mode: str = "uniform", thin: int = 1,
               spec: PriorSpec = PriorSpec(), rng: Optional[np.random.Generator] = None,
               cfg: EngineConfig = EngineConfig(), rejuvenate: bool = True, points=None,
               init_loglik: Optional[np.ndarray] = None) -> ChainsResult:
    """Blockwise random-walk MH (+ the rejuvenation move every
    REJUVENATE_PERIOD-th iteration) for C chains in lockstep, on the schedule
    of the reference ``run_chain`` (bayes.py:690-796): ``iterations`` counts
    iteration 0 (the initial state), rows are kept when it % thin == 0.  One
    batched likelihood launch per move.  ``steps`` = (gamma, p, mu, sigma).
    ``points`` = (present, lon, lat) for the rejuvenation move's location
    kernel (the reference passes its observations).  ``obs``: a
    ``DeviceObservations`` (one GPU) or a ``distributed.ReplicaLoglik``
    (chains' proposals sharded over the ranks; run the same call with the
    same seed on every rank)."""
    rng = np.random.default_rng(0) if rng is None else rng
    if int(iterations) != iterations or iterations < 1:
        raise ValueError("iterations must be a positive integer")
    cur = np.array(np.atleast_2d(init_vecs), dtype=np.float64)
    if cur.shape[1] != vector_length(k):
        raise ValueError(f"expected vectors of length {vector_length(k)}")
    n_chains = cur.shape[0]
    cur_lp = log_prior_batch(k, cur, spec)
    pack, ok = params_from_vectors(k, cur, delta_mode)
    if not ok.all() or not np.all(np.isfinite(cur_lp)):
        raise ValueError("initial states must lie inside the prior support")
    evals = 0
    if init_loglik is None:
        cur_ll = obs.loglik_batch(pack, cfg)
        evals += 1
    else:
        cur_ll = np.array(init_loglik, dtype=np.float64)
    rejuv = Rejuvenator(spec, points) if rejuvenate else None
    names = [name for name, _ in BLOCKS] + (["rejuvenate"] if rejuvenate else [])
    acc = {name: np.zeros(n_chains, dtype=np.int64) for name in names}
    proposed = {name: 0 for name in names}
    kept_i, kept_v, kept_ll, kept_lp = [0], [cur.copy()], [cur_ll.copy()], [cur_lp.copy()]
    moves = list(zip(BLOCKS, steps))
    for it in range(1, int(iterations)):
        todo = [(name, prop, step) for (name, prop), step in moves]
        if rejuvenate and it % REJUVENATE_PERIOD == 0:
            todo.append(("rejuvenate", None, None))
        for name, prop, step in todo:
            if name != "rejuvenate" and step == 0.0:
                continue
            with np.errstate(all="ignore"):
                if name == "rejuvenate":
                    cand, jac, ok = rejuv.propose(k, cur, (it // REJUVENATE_PERIOD) % k, rng)
                else:
                    cand, jac, ok = prop(k, cur, step, rng)
            proposed[name] += 1
            cand_lp = log_prior_batch(k, cand, spec)
            pack, valid = params_from_vectors(k, cand, delta_mode)
            ok &= valid
            live = ok & np.isfinite(cand_lp)
            cand_ll = np.full(n_chains, -np.inf)
            if live.any():
                sel = np.flatnonzero(live)
                pk = pack if live.all() else params_from_vectors(k, cand[sel], delta_mode)[0]
                cand_ll[sel] = obs.loglik_batch(pk, cfg)  # one launch for every live candidate
                evals += 1
            test = live & np.isfinite(cand_ll)
            # one uniform per candidate that reaches the MH test, in chain order
            # (the reference's mh_accept, bayes.py:656-658, 767-772)
            log_ratio = (cand_ll + cand_lp) - (cur_ll + cur_lp) + jac
            accept = np.zeros(n_chains, dtype=bool)
            idx = np.flatnonzero(test)
            if idx.size:
                u = rng.random(idx.size)
                accept[idx] = u < np.exp(np.minimum(log_ratio[idx], 0.0))
            cur[accept] = cand[accept]
            cur_ll[accept] = cand_ll[accept]
            cur_lp[accept] = cand_lp[accept]
            acc[name] += accept
        if it % thin == 0:
            kept_i.append(it)
            kept_v.append(cur.copy())
            kept_ll.append(cur_ll.copy())
            kept_lp.append(cur_lp.copy())
    rate = {n: (a / proposed[n] if proposed[n] else np.zeros(n_chains)) for n, a in acc.items()}
    return ChainsResult(np.stack(kept_v), np.stack(kept_ll), np.stack(kept_lp), rate, evals,
                        np.array(kept_i, dtype=np.int64), acc, proposed)
