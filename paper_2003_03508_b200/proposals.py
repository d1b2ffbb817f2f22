"""Batched per-proposal host work for the MCMC inner loop.

The reference builds one frozen ``HmmParams`` per proposal in Python
(``bayes.params_from_vector``, bayes.py:285-302, validating every state in
``StateEmission.__post_init__``, core.py:103-119) and, with
``delta_mode="stationary"``, runs a power iteration per proposal
(``core.stationary_distribution``, core.py:350-388): 1-9 ms per proposal,
which rivals the GPU likelihood of a whole batch.  Here a batch of B
parameter vectors becomes the packed structure-of-arrays block of the C-ABI
in one vectorised pass, the stationary vectors of all B transition matrices
come from one GPU launch (``thmm_stationary``), and the result feeds
``DeviceObservations.loglik_batch`` directly (no Python objects).

Vector layout (reference ``params_to_vector``, bayes.py:265-282):
``gamma (K*K, row-major) | p (K) | mu (K x 2) | sigma (K x [s00, s01, s11])``.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .model import ParamPack

STATIONARY_TOL = 1e-12        # reference core.py:29
STATIONARY_MAX_ITER = 100_000  # reference core.py:30


def vector_length(k: int) -> int:
    return k * k + 6 * k


def params_to_vectors(params_list) -> np.ndarray:
    """(B, K*K + 6K) vectors of HmmParams-like objects (bayes.py:265-282)."""
    out = []
    for p in params_list:
        k = int(p.K)
        sig = np.stack([[s.sigma[0, 0], s.sigma[0, 1], s.sigma[1, 1]] for s in p.states])
        mus = np.stack([s.mu for s in p.states])
        out.append(np.concatenate([np.asarray(p.gamma).ravel(), np.asarray(p._p), mus.ravel(), sig.ravel()]))
    return np.stack(out)


def stationary_distribution_batch(gammas, device: int = 0, tol: float = STATIONARY_TOL,
                                  max_iter: int = STATIONARY_MAX_ITER) -> np.ndarray:
    """Stationary vectors of B row-stochastic matrices (B, K, K) -> (B, K),
    one GPU launch.  RuntimeError if any power iteration does not converge
    (reference core.py:383-387)."""
    g = np.ascontiguousarray(gammas, dtype=np.float64)
    if g.ndim == 2:
        g = g[None]
    if g.ndim != 3 or g.shape[1] != g.shape[2]:
        raise ValueError("gamma must be a square matrix")
    if not np.all(np.isfinite(g)) or np.any(g < 0.0):
        raise ValueError("gamma entries must be finite and nonnegative")
    if np.max(np.abs(g.sum(axis=2) - 1.0)) > 1e-9:
        raise ValueError("gamma rows must sum to 1")
    b, k = g.shape[0], g.shape[1]
    nat.require_device()
    out = np.empty((b, k), dtype=np.float64)
    status = np.empty(b, dtype=np.int32)
    err = nat.errbuf()
    rc = nat.lib().thmm_stationary(nat.as_ptr(g, nat.c_double), k, b, float(tol), int(max_iter), int(device),
                                   nat.as_ptr(out, nat.c_double), nat.as_ptr(status, nat.c_int32), err, len(err))
    nat.raise_for(rc, err)
    return out


def params_from_vectors(k: int, vecs, delta_mode: str = "stationary", device: int = 0):
    """Pack B parameter vectors for the likelihood in one vectorised pass.

    Returns ``(pack, valid)``: ``pack`` is a ``ParamPack`` for the valid rows
    and ``valid`` a boolean mask over the input -- a row is invalid exactly
    when the reference's ``params_from_vector`` would raise ValueError
    (gamma rows not stochastic to 1e-12 or negative, p outside (0, 1),
    non-finite mu, covariance not SPD), which the MCMC driver treats as a
    rejected proposal (bayes.py:760-762)."""
    v = np.ascontiguousarray(vecs, dtype=np.float64)
    if v.ndim == 1:
        v = v[None]
    if v.shape[1] != vector_length(k):
        raise ValueError(f"expected vectors of length {vector_length(k)}")
    b = v.shape[0]
    kk = k * k
    gamma = v[:, :kk].reshape(b, k, k)
    ps = v[:, kk:kk + k]
    mus = v[:, kk + k:kk + 3 * k].reshape(b, k, 2)
    sig = v[:, kk + 3 * k:].reshape(b, k, 3)
    s00, s01, s11 = sig[..., 0], sig[..., 1], sig[..., 2]
    with np.errstate(invalid="ignore", divide="ignore"):
        ok = np.all(np.isfinite(v), axis=1)
        ok &= np.all(gamma >= 0.0, axis=(1, 2))
        ok &= np.max(np.abs(gamma.sum(axis=2) - 1.0), axis=1) <= 1e-12
        ok &= np.all((ps > 0.0) & (ps < 1.0), axis=1)
        ok &= np.all(s00 > 0.0, axis=1)
        l00 = np.sqrt(s00)
        l10 = s01 / l00
        rem = s11 - l10 * l10
        ok &= np.all(rem > 0.0, axis=1)
        l11 = np.sqrt(rem)
        log_det = 2.0 * (np.log(l00) + np.log(l11))
    idx = np.flatnonzero(ok)
    nb = idx.size
    buf = np.empty(nb * (kk + 9 * k), dtype=np.float64)
    g_out = buf[:nb * kk].reshape(nb, k, k)
    d_out = buf[nb * kk:nb * (kk + k)].reshape(nb, k)
    st = buf[nb * (kk + k):].reshape(8, nb, k)
    g_out[:] = gamma[idx]
    if nb:
        if delta_mode == "stationary":
            d_out[:] = stationary_distribution_batch(g_out, device=device)
        elif delta_mode == "uniform":
            d_out[:] = 1.0 / k
        else:
            raise ValueError("delta_mode must be 'stationary' or 'uniform'")
    st[0] = ps[idx]
    st[1] = 1.0 - ps[idx]
    st[2] = mus[idx, :, 0]
    st[3] = mus[idx, :, 1]
    st[4] = l00[idx]
    st[5] = l10[idx]
    st[6] = l11[idx]
    st[7] = log_det[idx]
    return ParamPack(k, g_out, d_out, st), ok
