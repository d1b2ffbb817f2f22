"""Host-side model types for the zero-inflated bivariate-Gaussian HMM.

These mirror the reference's domain types so that callers of
``tremorhmm.engine.parallel_loglik`` can switch packages without touching
their code:

* ``Observation``      -- reference core.py:62-83
* ``StateEmission``    -- reference core.py:86-119 (2x2 Cholesky, core.py:33-53)
* ``HmmParams``        -- reference core.py:122-173 (incl. the stacked per-state
                          scalars ``_p,_q,_mu0,_mu1,_l00,_l10,_l11,_log_det``)
* ``ScaledMatrix``     -- reference core.py:176-206
* ``observation_arrays`` -- reference core.py:209-222

The device path never sees these objects: ``pack_params`` flattens one or
more parameter sets (ours or the reference's own ``HmmParams``, which carry
the same attributes) into the structure-of-arrays layout the C-ABI takes
(include/thmm.h, ``thmm_params``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

LOG_2PI = math.log(2.0 * math.pi)


def _readonly(values) -> np.ndarray:
    arr = np.array(values, dtype=np.float64, copy=True)
    arr.setflags(write=False)
    return arr


def cholesky2(sigma: np.ndarray) -> Tuple[float, float, float]:
    """Lower factor (l00, l10, l11) of a 2x2 SPD matrix (reference core.py:33-53).

    Same checks and error messages class as the reference: non-finite,
    asymmetric (beyond 1e-12 relative) or non-positive-definite input raises
    ValueError.
    """
    s00, s01 = float(sigma[0, 0]), float(sigma[0, 1])
    s10, s11 = float(sigma[1, 0]), float(sigma[1, 1])
    if not all(math.isfinite(x) for x in (s00, s01, s10, s11)):
        raise ValueError("covariance entries must be finite")
    if abs(s01 - s10) > 1e-12 * max(1.0, abs(s01), abs(s10)):
        raise ValueError("covariance matrix must be symmetric")
    if s00 <= 0.0:
        raise ValueError("covariance matrix is not positive definite")
    l00 = math.sqrt(s00)
    l10 = s10 / l00
    schur = s11 - l10 * l10
    if schur <= 0.0:
        raise ValueError("covariance matrix is not positive definite")
    return l00, l10, math.sqrt(schur)


@dataclass(frozen=True)
class Observation:
    """One hourly record: ``(lon, lat)`` for a located tremor, ``None`` for a quiet hour."""

    value: Optional[Tuple[float, float]] = None

    def __post_init__(self):
        if self.value is None:
            return
        lon, lat = (float(c) for c in self.value)
        if not (math.isfinite(lon) and math.isfinite(lat)):
            raise ValueError("observation coordinates must be finite")
        object.__setattr__(self, "value", (lon, lat))

    @property
    def present(self) -> bool:
        return self.value is not None


@dataclass(frozen=True)
class StateEmission:
    """Emission law of one hidden state: event probability p in (0, 1),
    mean ``mu`` (2,) and covariance ``sigma`` (2, 2) with its cached lower
    Cholesky factor and log-determinant."""

    p: float
    mu: np.ndarray
    sigma: np.ndarray
    chol: np.ndarray = field(init=False, repr=False, compare=False)
    log_det: float = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        p = float(self.p)
        if not (math.isfinite(p) and 0.0 < p < 1.0):
            raise ValueError("event probability must lie strictly in (0, 1)")
        mu = np.asarray(self.mu, dtype=np.float64)
        if mu.shape != (2,) or not np.all(np.isfinite(mu)):
            raise ValueError("mu must be a finite length-2 vector")
        sigma = np.asarray(self.sigma, dtype=np.float64)
        if sigma.shape != (2, 2):
            raise ValueError("sigma must be a 2x2 matrix")
        l00, l10, l11 = cholesky2(sigma)
        object.__setattr__(self, "p", p)
        object.__setattr__(self, "mu", _readonly(mu))
        object.__setattr__(self, "sigma", _readonly(sigma))
        object.__setattr__(self, "chol", _readonly([[l00, 0.0], [l10, l11]]))
        object.__setattr__(self, "log_det", 2.0 * (math.log(l00) + math.log(l11)))


@dataclass(frozen=True)
class HmmParams:
    """Transition matrix ``gamma`` (K, K), initial law ``delta`` (K,) and the
    K state emissions; validated and frozen at construction (reference
    core.py:135-169), with the same stacked per-state scalars."""

    gamma: np.ndarray
    delta: np.ndarray
    states: Tuple[StateEmission, ...]

    def __post_init__(self):
        states = tuple(self.states)
        if not states:
            raise ValueError("at least one state is required")
        if not all(isinstance(s, StateEmission) for s in states):
            raise ValueError("states must be StateEmission instances")
        k = len(states)
        gamma = np.asarray(self.gamma, dtype=np.float64)
        if gamma.shape != (k, k):
            raise ValueError(f"gamma must have shape ({k}, {k})")
        if not np.all(np.isfinite(gamma)) or np.any(gamma < 0.0):
            raise ValueError("gamma entries must be finite and nonnegative")
        worst = float(np.max(np.abs(gamma.sum(axis=1) - 1.0)))
        if worst > 1e-12:
            raise ValueError(f"gamma rows must sum to 1 (max deviation {worst:.3e})")
        delta = np.asarray(self.delta, dtype=np.float64)
        if delta.shape != (k,):
            raise ValueError(f"delta must have length {k}")
        if not np.all(np.isfinite(delta)) or np.any(delta < 0.0):
            raise ValueError("delta entries must be finite and nonnegative")
        if abs(delta.sum() - 1.0) > 1e-12:
            raise ValueError("delta must sum to 1")
        put = lambda name, val: object.__setattr__(self, name, val)  # noqa: E731
        put("gamma", _readonly(gamma))
        put("delta", _readonly(delta))
        put("states", states)
        put("_p", _readonly([s.p for s in states]))
        put("_q", _readonly([1.0 - s.p for s in states]))
        put("_mu0", _readonly([s.mu[0] for s in states]))
        put("_mu1", _readonly([s.mu[1] for s in states]))
        put("_l00", _readonly([s.chol[0, 0] for s in states]))
        put("_l10", _readonly([s.chol[1, 0] for s in states]))
        put("_l11", _readonly([s.chol[1, 1] for s in states]))
        put("_log_det", _readonly([s.log_det for s in states]))

    @property
    def K(self) -> int:
        return len(self.states)


@dataclass(frozen=True)
class ScaledMatrix:
    """Nonnegative matrix carried as ``exp(log_scale) * m`` (reference core.py:176-206)."""

    m: np.ndarray
    log_scale: float = 0.0

    def __post_init__(self):
        m = np.asarray(self.m)
        if m.ndim != 2:
            raise ValueError("m must be a 2-d matrix")
        if not np.all(np.isfinite(m)) or np.any(m < 0.0):
            raise ValueError("matrix entries must be finite and nonnegative")
        object.__setattr__(self, "m", m)
        object.__setattr__(self, "log_scale", float(self.log_scale))

    def normalized(self) -> "ScaledMatrix":
        top = float(self.m.max())
        if top <= 0.0 or top == 1.0:
            return self
        return ScaledMatrix(self.m / top, self.log_scale + math.log(top))

    def to_dense(self) -> np.ndarray:
        return np.exp(self.log_scale) * np.asarray(self.m, dtype=np.float64)


def observation_arrays(obs: Sequence[Observation]) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """``(present bool[N], lon f64[N], lat f64[N])``; absent records hold 0.0."""
    n = len(obs)
    present = np.zeros(n, dtype=bool)
    lon = np.zeros(n, dtype=np.float64)
    lat = np.zeros(n, dtype=np.float64)
    for i, ob in enumerate(obs):
        if ob.value is not None:
            present[i] = True
            lon[i], lat[i] = ob.value
    return present, lon, lat


# Order of the per-state vectors in the packed parameter block; must match
# thmm_params in include/thmm.h.
STATE_FIELDS = ("_p", "_q", "_mu0", "_mu1", "_l00", "_l10", "_l11", "_log_det")


@dataclass
class ParamPack:
    """Structure-of-arrays view of B parameter sets with a common K.

    gamma (B, K, K), delta (B, K) and ``states`` (8, B, K) in STATE_FIELDS
    order, all C-contiguous float64.
    """

    K: int
    gamma: np.ndarray
    delta: np.ndarray
    states: np.ndarray

    @property
    def B(self) -> int:
        return self.gamma.shape[0]

    def __len__(self) -> int:
        return self.B

    def slice(self, lo: int, hi: int) -> "ParamPack":
        """Parameter sets [lo, hi) as a new contiguous pack."""
        return ParamPack(self.K, np.ascontiguousarray(self.gamma[lo:hi]), np.ascontiguousarray(self.delta[lo:hi]),
                         np.ascontiguousarray(self.states[:, lo:hi]))


def pack_params(params_list) -> ParamPack:
    """Flatten one HmmParams (or a sequence of them, common K) for the C-ABI.

    Accepts any object with the reference HmmParams attributes, so the
    reference's own frozen parameter objects work unchanged.
    """
    if hasattr(params_list, "gamma"):
        params_list = [params_list]
    params_list = list(params_list)
    if len(params_list) == 1:  # the MCMC hot call: one concatenate instead of 10 assignments
        p = params_list[0]
        k = len(p._p)
        buf = np.concatenate((p.gamma.ravel(), p.delta, p._p, p._q, p._mu0, p._mu1, p._l00, p._l10, p._l11,
                              p._log_det))  # STATE_FIELDS order
        if buf.dtype != np.float64:
            buf = buf.astype(np.float64)
        kk = k * k
        return ParamPack(k, buf[:kk].reshape(1, k, k), buf[kk:kk + k].reshape(1, k), buf[kk + k:].reshape(8, 1, k))
    if not params_list:
        raise ValueError("no parameter sets given")
    k = int(params_list[0].K)
    if any(int(p.K) != k for p in params_list):
        raise ValueError("all parameter sets of a batch must share K")
    b, kk = len(params_list), k * k
    # one contiguous block: gamma | delta | states, filled in place
    buf = np.empty(b * (kk + 9 * k), dtype=np.float64)
    gamma = buf[:b * kk].reshape(b, k, k)
    delta = buf[b * kk:b * (kk + k)].reshape(b, k)
    states = buf[b * (kk + k):].reshape(8, b, k)
    for i, p in enumerate(params_list):
        gamma[i] = p.gamma
        delta[i] = p.delta
        for f, name in enumerate(STATE_FIELDS):
            states[f, i] = getattr(p, name)
    return ParamPack(k, gamma, delta, states)
