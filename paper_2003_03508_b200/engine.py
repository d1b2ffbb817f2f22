"""Drop-in replacement for ``tremorhmm.engine`` backed by sm_100a kernels.

Same names, signatures, argument meaning and error behaviour as the
reference module (/root/reference/pkg/src/tremorhmm/engine.py); the three
stages of engine.py:1-17 run on the GPU behind the C-ABI of include/thmm.h:

1. emission diagonals -- evaluated inside the chain kernel from the raw
   (present, lon, lat) stream, never materialised (reference core.py:235-260);
2. ``Gamma diag(e_t)`` -- applied as the epilogue of each FP64 tensor-core
   step (reference engine.py:136-143);
3. segmented scaled chain products + ordered combine -- one CTA per segment,
   then a log-depth tree of the same MMA machinery, finished against delta
   on the device (reference engine.py:225-231, 292-345).

``EngineConfig.workers`` keeps its reference meaning: it never changes the
value for a given segment count, and ``segments`` defaults to it
(engine.py:61-64; test_engine.py:197-203 compares workers=4 with
workers=1/segments=4 bitwise).  The one deviation: the reference default
(workers=1, one sequential segment) lets the engine cut the chain to fill the
GPU.  An explicit count is honoured.  Results are deterministic.

Additions (no reference counterpart):

* ``DeviceObservations`` -- device-resident observation stream, uploaded
  once and reused by every evaluation (the MCMC inner loop).
* ``parallel_loglik_batch`` -- B parameter proposals per launch.
"""

from __future__ import annotations

import math
import os
import threading
import weakref
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native as nat
from .model import HmmParams, Observation, ParamPack, ScaledMatrix, observation_arrays, pack_params

MAX_PARALLEL_STATES = nat.MAX_STATES
MAX_BATCH = 65535  # parameter sets per launch (thmm_loglik: grid y extent)


@dataclass(frozen=True)
class EngineConfig:
    """Knobs of the parallel backend (reference engine.py:49-81)."""

    workers: int = 1
    segments: Optional[int] = None
    renorm_period: int = 8
    precision: str = "float64"

    def __post_init__(self):
        if int(self.workers) != self.workers or self.workers < 1:
            raise ValueError("workers must be a positive integer")
        if self.segments is not None and (int(self.segments) != self.segments or self.segments < 1):
            raise ValueError("segments must be a positive integer when given")
        if int(self.renorm_period) != self.renorm_period or self.renorm_period < 1:
            raise ValueError("renorm_period must be a positive integer")
        if self.precision not in nat.PRECISION_CODES:
            raise ValueError("precision must be 'float64' or 'float32' (or the tensor-core study modes "
                             "'tf32', 'tf32x2', 'tf32x3')")

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float64 if self.precision == "float64" else np.float32)

    def resolved_segments(self) -> int:
        return self.workers if self.segments is None else self.segments


@dataclass(frozen=True)
class SegmentProduct:
    """Scale-carrying product of the factor sub-chain [lo, hi) (engine.py:84-94)."""

    product: ScaledMatrix
    lo: int
    hi: int

    def __post_init__(self):
        if not (0 <= self.lo < self.hi):
            raise ValueError("segment range must be non-empty with 0 <= lo < hi")


def segment_bounds(n: int, segments: int) -> List[tuple]:
    """Contiguous blocks with sizes differing by at most one, earlier blocks
    larger (engine.py:97-111); the device kernels use the same split."""
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


# ---------------------------------------------------------------------------
# device selection
# ---------------------------------------------------------------------------

_default_device = None


def set_default_device(device: int) -> None:
    """Device used by the array/object entry points (default: $LOCAL_RANK or 0)."""
    global _default_device
    _default_device = int(device)


def default_device() -> int:
    if _default_device is not None:
        return _default_device
    return int(os.environ.get("LOCAL_RANK", "0"))


def _native_config(cfg: EngineConfig, lo: int = 0, hi: int = 0, stream: int = 0,
                   segments: Optional[int] = None) -> nat.ThmmConfig:
    # Reference semantics: ``segments`` defaults to ``workers`` (engine.py:61-64,
    # 80-81), so EngineConfig(workers=4) is EngineConfig(workers=4, segments=4)
    # value for value.  The reference default (workers=1 -> ONE segment, a
    # fully sequential chain) is the one deviation: on the GPU it means "fill
    # the device" (segment count only changes the value at rounding level).
    if segments is None:
        segments = cfg.segments if cfg.segments is not None else (cfg.workers if cfg.workers > 1 else None)
    segs = segments
    return nat.ThmmConfig(int(cfg.renorm_period), nat.PRECISION_CODES[cfg.precision],
                          int(segs or 0), int(lo), int(hi), stream or None)


class _PackedParams:
    """Keeps the packed arrays alive while the C struct points into them."""

    def __init__(self, params_list):
        # an already packed block (proposals.params_from_vectors) passes through
        pack = params_list if isinstance(params_list, ParamPack) else pack_params(params_list)
        if pack.B < 1:
            raise ValueError("no parameter sets given")
        if pack.K > MAX_PARALLEL_STATES:
            raise ValueError(f"parallel engine supports at most {MAX_PARALLEL_STATES} states, got {pack.K}")
        self.pack = pack
        self.struct = nat.ThmmParams(pack.K, pack.B, pack.gamma.ctypes.data, pack.delta.ctypes.data,
                                     pack.states.ctypes.data)


# ---------------------------------------------------------------------------
# device-resident observations
# ---------------------------------------------------------------------------


# Host observation arrays page-locked on first use (thmm_host_register): the
# reference's MCMC driver passes the same arrays on every likelihood call
# (bayes.py:709-715), so after the first call the chain kernels read them in
# place over PCIe (zero-copy) instead of staging a pageable copy.  Keyed by
# (address, bytes); released when the owning array is (weakref.finalize runs
# in numpy's dealloc before the buffer is freed).  THMM_AUTOPIN=0 disables.
AUTOPIN_MIN_BYTES = 1 << 12
_pin_lock = threading.Lock()
_pinned_ranges = {}  # (ptr, nbytes) -> (registered: bool, finalizer)


def _unpin(key, registered):
    with _pin_lock:
        _pinned_ranges.pop(key, None)
    if registered and nat._lib is not None:
        nat.lib().thmm_host_unregister(nat.c_void_p(key[0]))


def _auto_pin(*arrays) -> None:
    if os.environ.get("THMM_AUTOPIN", "1") == "0":
        return
    for a in arrays:
        if a.nbytes < AUTOPIN_MIN_BYTES:
            continue
        key = (a.ctypes.data, a.nbytes)
        if key in _pinned_ranges:  # the common case (same arrays every call): no lock
            continue
        with _pin_lock:
            if key in _pinned_ranges:
                continue
            owner = a
            while isinstance(owner.base, np.ndarray):
                owner = owner.base
            err = nat.errbuf()
            ok = nat.lib().thmm_host_register(nat.c_void_p(key[0]), key[1], err, len(err)) == nat.THMM_OK
            # failures (already pinned, e.g. torch pin_memory; or not lockable) are
            # remembered too, so the registration is not retried every call
            _pinned_ranges[key] = (ok, weakref.finalize(owner, _unpin, key, ok))


def _host_arrays(present, lon, lat):
    present = np.ascontiguousarray(present, dtype=np.bool_).view(np.uint8)
    lon = np.ascontiguousarray(lon, dtype=np.float64)
    lat = np.ascontiguousarray(lat, dtype=np.float64)
    if not (present.shape == lon.shape == lat.shape) or present.ndim != 1:
        raise ValueError("present, lon and lat must be 1-d arrays of equal length")
    return present, lon, lat


class DeviceObservations:
    """An observation stream resident in HBM of one GPU.

    Build it once (``DeviceObservations(present, lon, lat)`` or
    ``DeviceObservations.from_observations(obs)``) and evaluate any number of
    parameter sets against it; this is what the MCMC loop should hold.
    """

    def __init__(self, present, lon, lat, device: Optional[int] = None):
        nat.require_device()
        present, lon, lat = _host_arrays(present, lon, lat)
        if present.size == 0:
            raise ValueError("observation sequence is empty")
        self.device = default_device() if device is None else int(device)
        self._handle = nat.c_void_p()
        err = nat.errbuf()
        rc = nat.lib().thmm_obs_create(nat.as_ptr(present, nat.c_uint8), nat.as_ptr(lon, nat.c_double),
                                       nat.as_ptr(lat, nat.c_double), present.size, self.device,
                                       nat.ctypes.byref(self._handle), err, len(err))
        nat.raise_for(rc, err)
        self.n = int(present.size)

    @classmethod
    def from_observations(cls, obs: Sequence[Observation], device: Optional[int] = None):
        return cls(*observation_arrays(obs), device=device)

    def assign(self, present, lon, lat) -> None:
        """Replace the stream contents (reuses the device allocation)."""
        present, lon, lat = _host_arrays(present, lon, lat)
        if present.size == 0:
            raise ValueError("observation sequence is empty")
        err = nat.errbuf()
        rc = nat.lib().thmm_obs_assign(self._handle, nat.as_ptr(present, nat.c_uint8),
                                       nat.as_ptr(lon, nat.c_double), nat.as_ptr(lat, nat.c_double),
                                       present.size, err, len(err))
        nat.raise_for(rc, err)
        self.n = int(present.size)

    def __len__(self) -> int:
        return self.n

    def close(self) -> None:
        if getattr(self, "_handle", None) is not None and self._handle.value:
            nat.lib().thmm_obs_destroy(self._handle)
            self._handle = nat.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    # -- evaluation -------------------------------------------------------

    def loglik_batch(self, params_list, cfg: EngineConfig, *, lo: int = 0, hi: int = 0,
                     stream: int = 0, raise_on_collapse: bool = False) -> np.ndarray:
        """Log-likelihood of each parameter set; collapsed proposals give -inf
        (or RuntimeError with ``raise_on_collapse``).  Batches beyond one
        launch's proposal limit (MAX_BATCH, the grid's y extent) run as
        consecutive launches."""
        n_sets = len(params_list) if isinstance(params_list, ParamPack) else None
        if n_sets is None:
            params_list = list(params_list)
            n_sets = len(params_list)
        if n_sets > MAX_BATCH:
            parts = []
            for s0 in range(0, n_sets, MAX_BATCH):
                part = (params_list.slice(s0, min(s0 + MAX_BATCH, n_sets)) if isinstance(params_list, ParamPack)
                        else params_list[s0:s0 + MAX_BATCH])
                parts.append(self.loglik_batch(part, cfg, lo=lo, hi=hi, stream=stream,
                                               raise_on_collapse=raise_on_collapse))
            return np.concatenate(parts)
        pp = _PackedParams(params_list)
        out = np.empty(pp.pack.B, dtype=np.float64)
        status = np.empty(pp.pack.B, dtype=np.int32)
        c = _native_config(cfg, lo, hi, stream)
        err = nat.errbuf()
        rc = nat.lib().thmm_loglik(self._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                   out.ctypes.data, status.ctypes.data, err, len(err))
        if rc == nat.THMM_ECOLLAPSE and not raise_on_collapse:
            return out
        nat.raise_for(rc, err)
        return out

    def loglik_host_batch(self, params_list, present, lon, lat, cfg: EngineConfig, *, stream: int = 0,
                          raise_on_collapse: bool = False, mapped: bool = False, _checked: bool = False) -> np.ndarray:
        """Replace the stream with host arrays and evaluate, with the
        host->device copy pipelined against the chain kernels.

        mapped=True: pinned arrays are read in place by the chain kernels
        over PCIe (thmm_loglik_mapped, zero-copy) and the handle's records
        are left unchanged; pageable arrays take the pipelined copy."""
        if not _checked:
            present, lon, lat = _host_arrays(present, lon, lat)
        if present.size == 0:
            raise ValueError("observation sequence is empty")
        if mapped:
            _auto_pin(present, lon, lat)
        pp = _PackedParams(params_list)
        out = np.empty(pp.pack.B, dtype=np.float64)
        status = np.empty(pp.pack.B, dtype=np.int32)
        c = _native_config(cfg, 0, 0, stream)
        err = nat.errbuf()
        fn = nat.lib().thmm_loglik_mapped if mapped else nat.lib().thmm_loglik_host
        rc = fn(self._handle, present.ctypes.data, lon.ctypes.data, lat.ctypes.data, present.size,
                nat.ctypes.byref(pp.struct), nat.ctypes.byref(c), out.ctypes.data, status.ctypes.data, err, len(err))
        self.n = int(nat.lib().thmm_obs_length(self._handle))  # unchanged by a zero-copy call
        if rc == nat.THMM_ECOLLAPSE and not raise_on_collapse:
            return out
        nat.raise_for(rc, err)
        return out

    def loglik(self, params, cfg: EngineConfig, **kw) -> float:
        return float(self.loglik_batch([params], cfg, raise_on_collapse=True, **kw)[0])

    def range_nodes(self, params_list, cfg: EngineConfig, lo: int, hi: int, out_m_ptr: int, out_e_ptr: int,
                    stream: int = 0, sync: bool = True) -> None:
        """Reduce records [lo, hi) to one scaled product node per proposal,
        written to device memory (multi-GPU shard; see distributed.py).
        ``sync=False`` only enqueues the work on ``stream``."""
        pp = _PackedParams(params_list)
        c = _native_config(cfg, lo, hi, stream)
        err = nat.errbuf()
        fn = nat.lib().thmm_range_nodes if sync else nat.lib().thmm_range_nodes_async
        rc = fn(self._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                nat.c_void_p(out_m_ptr), nat.c_void_p(out_e_ptr), err, len(err))
        nat.raise_for(rc, err)

    def range_nodes_host(self, params_list, present, lon, lat, cfg: EngineConfig, out_m_ptr: int,
                         out_e_ptr: int, stream: int = 0) -> None:
        """Replace the stream with host arrays and enqueue the reduction of
        the whole stream to one node per proposal, the copy pipelined against
        the chain (``thmm_range_nodes_host``).  Nothing is synchronised: the
        host arrays must stay alive and unmodified until ``stream`` has
        passed this point (the fold that consumes the nodes)."""
        present, lon, lat = _host_arrays(present, lon, lat)
        if present.size == 0:
            raise ValueError("observation sequence is empty")
        _auto_pin(present, lon, lat)
        pp = _PackedParams(params_list)
        c = _native_config(cfg, 0, 0, stream)
        err = nat.errbuf()
        rc = nat.lib().thmm_range_nodes_host(self._handle, nat.as_ptr(present, nat.c_uint8),
                                             nat.as_ptr(lon, nat.c_double), nat.as_ptr(lat, nat.c_double),
                                             present.size, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                             nat.c_void_p(out_m_ptr), nat.c_void_p(out_e_ptr), err, len(err))
        nat.raise_for(rc, err)
        self.n = int(present.size)
        self._host_refs = (present, lon, lat)  # keep the source alive past the asynchronous copy

    def filtered_next_state(self, params_list, cfg: EngineConfig = EngineConfig(), *, lo: int = 0,
                            hi: int = 0, raise_on_collapse: bool = True) -> np.ndarray:
        """(B, K) distribution of the state one step past the history, per
        parameter set (reference simforecast._filtered_next_state_dist,
        simforecast.py:97-118), from the same device chain product."""
        pp = _PackedParams(params_list)
        out = np.empty((pp.pack.B, pp.pack.K), dtype=np.float64)
        status = np.empty(pp.pack.B, dtype=np.int32)
        c = _native_config(cfg, lo, hi)
        err = nat.errbuf()
        rc = nat.lib().thmm_filtered_state(self._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                           nat.as_ptr(out, nat.c_double), nat.as_ptr(status, nat.c_int32), err,
                                           len(err))
        if rc == nat.THMM_ECOLLAPSE and not raise_on_collapse:
            return out
        nat.raise_for(rc, err)
        return out

    def runs_info(self, k: int, precision: str = "float64") -> dict:
        """Whether evaluations at (K, precision) on this handle run the
        run-absorbing chain (thmm_runs_info), with the estimated steps per
        record and its launch plan."""
        return nat.runs_info(self._handle, k, precision)

    def emissions(self, params, lo: int = 0, hi: Optional[int] = None, *, chain: bool = False) -> np.ndarray:
        """(hi-lo, K) emission table of records [lo, hi) (reference
        _emission_columns, core.py:235-260).  ``chain=True``: computed with the
        chain kernels' emission arithmetic (thmm_emissions_chain) -- the
        values the likelihood multiplies by."""
        hi = self.n if hi is None else int(hi)
        pp = _PackedParams([params])
        out = np.empty((max(hi - lo, 0), pp.pack.K), dtype=np.float64)
        err = nat.errbuf()
        fn = nat.lib().thmm_emissions_chain if chain else nat.lib().thmm_emissions
        rc = fn(self._handle, nat.ctypes.byref(pp.struct), int(lo), int(hi),
                nat.as_ptr(out, nat.c_double), err, len(err))
        nat.raise_for(rc, err)
        return out


def fold_nodes(params_list, nodes_m_ptr: int, nodes_e_ptr: int, n_nodes: int, device: int,
               stream: int = 0, raise_on_collapse: bool = True, m_stride_g: Optional[int] = None,
               e_stride_g: Optional[int] = None) -> np.ndarray:
    """Ordered fold of ``n_nodes`` device nodes per proposal into
    log-likelihoods (device analogue of ``combine_segments``).  Default
    layout [G][B]; with strides, node g of proposal b sits at
    ``m + g*m_stride_g + b*KP*KP`` and its exponent at ``e[g*e_stride_g + b]``
    (doubles)."""
    pp = _PackedParams(params_list)
    out = np.empty(pp.pack.B, dtype=np.float64)
    status = np.empty(pp.pack.B, dtype=np.int32)
    err = nat.errbuf()
    if m_stride_g is None:
        rc = nat.lib().thmm_fold_nodes(nat.ctypes.byref(pp.struct), int(n_nodes), nat.c_void_p(nodes_m_ptr),
                                       nat.c_void_p(nodes_e_ptr), int(device), nat.c_void_p(stream or None),
                                       nat.as_ptr(out, nat.c_double), nat.as_ptr(status, nat.c_int32), err,
                                       len(err))
    else:
        rc = nat.lib().thmm_fold_nodes_strided(
            nat.ctypes.byref(pp.struct), int(n_nodes), nat.c_void_p(nodes_m_ptr), int(m_stride_g),
            nat.c_void_p(nodes_e_ptr), int(e_stride_g), int(device), nat.c_void_p(stream or None),
            nat.as_ptr(out, nat.c_double), nat.as_ptr(status, nat.c_int32), err, len(err))
    if rc == nat.THMM_ECOLLAPSE and not raise_on_collapse:
        return out
    nat.raise_for(rc, err)
    return out


def padded_states(k: int) -> int:
    return ((int(k) + 7) // 8) * 8


# Per-thread scratch stream per device for the host-array entry points, so
# repeated calls reuse one device allocation (thread-safe by construction).
_scratch = threading.local()


def _scratch_obs(present, lon, lat) -> DeviceObservations:
    dev = default_device()
    pool = getattr(_scratch, "pool", None)
    if pool is None:
        pool = _scratch.pool = {}
    handle = pool.get(dev)
    if handle is None:
        handle = pool[dev] = DeviceObservations(present, lon, lat, device=dev)
    else:
        handle.assign(present, lon, lat)
    return handle


def _host_loglik_batch(params_list, present, lon, lat, cfg: EngineConfig, raise_on_collapse: bool) -> np.ndarray:
    """Evaluate host arrays through the per-thread scratch handle: pinned
    arrays are read in place by the kernels (thmm_loglik_mapped, zero-copy),
    pageable ones go through the pipelined upload (copies overlap the chain)."""
    dev = default_device()
    pool = getattr(_scratch, "pool", None)
    if pool is None:
        pool = _scratch.pool = {}
    handle = pool.get(dev)
    if handle is None:  # first use: creating the handle uploads the stream once
        handle = pool[dev] = DeviceObservations(present, lon, lat, device=dev)
        return handle.loglik_batch(params_list, cfg, raise_on_collapse=raise_on_collapse)
    return handle.loglik_host_batch(params_list, present, lon, lat, cfg, raise_on_collapse=raise_on_collapse,
                                    mapped=True, _checked=True)


# ---------------------------------------------------------------------------
# reference API
# ---------------------------------------------------------------------------


def batch_emissions(params: HmmParams, obs: Sequence[Observation]) -> np.ndarray:
    """Stage 1 as an explicit (N, K) table (engine.py:234-243), on the GPU."""
    if len(obs) == 0:
        raise ValueError("observation sequence is empty")
    return _scratch_obs(*observation_arrays(obs)).emissions(params)


def scale_by_emission(gamma: np.ndarray, diag: np.ndarray) -> np.ndarray:
    """Stage 2 on one record: ``Gamma diag(e)`` (engine.py:246-256)."""
    gamma = np.asarray(gamma, dtype=np.float64)
    diag = np.asarray(diag, dtype=np.float64)
    if gamma.ndim != 2 or gamma.shape[0] != gamma.shape[1]:
        raise ValueError("gamma must be square")
    if diag.shape != (gamma.shape[0],):
        raise ValueError("diagonal length must match gamma")
    if not np.all(np.isfinite(diag)) or np.any(diag < 0.0):
        raise ValueError("emission diagonal must be finite and nonnegative")
    return gamma * diag


def segment_chain_product(factors, cfg: EngineConfig) -> List[SegmentProduct]:
    """Stage 3 over an explicit (n, K, K) factor stack (engine.py:259-289),
    reduced on the GPU."""
    arr = np.ascontiguousarray(factors, dtype=np.float64)
    if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
        raise ValueError("factors must be a stack of square matrices")
    n, k = arr.shape[0], arr.shape[1]
    if n < 1:
        raise ValueError("factor chain is empty")
    if k > MAX_PARALLEL_STATES:
        raise ValueError(f"parallel engine supports at most {MAX_PARALLEL_STATES} states, got {k}")
    if not np.all(np.isfinite(arr)) or np.any(arr < 0.0):
        raise ValueError("factors must be finite and nonnegative")
    segments = cfg.resolved_segments()
    if segments > n:
        raise ValueError(f"cannot cut a chain of {n} factors into {segments} segments")
    nat.require_device()
    out_m = np.empty((segments, k, k), dtype=np.float64)
    out_ls = np.empty(segments, dtype=np.float64)
    err = nat.errbuf()
    rc = nat.lib().thmm_factor_segments(nat.as_ptr(arr, nat.c_double), n, k, segments, cfg.renorm_period,
                                        default_device(), nat.as_ptr(out_m, nat.c_double),
                                        nat.as_ptr(out_ls, nat.c_double), err, len(err))
    nat.raise_for(rc, err)
    if cfg.dtype == np.float32:
        out_m = out_m.astype(np.float32)
    return [SegmentProduct(ScaledMatrix(out_m[i], float(out_ls[i])), lo, hi)
            for i, (lo, hi) in enumerate(segment_bounds(n, segments))]


def combine_segments(delta: np.ndarray, parts: Sequence[SegmentProduct]) -> float:
    """Ordered fold of segment products against delta (engine.py:292-318).

    Operates on host ``SegmentProduct`` objects exactly like the reference
    (an O(S K^2) host fold); the device path folds its own segments with
    ``fold_nodes`` instead."""
    if len(parts) == 0:
        raise ValueError("no segment products to combine")
    order = sorted(parts, key=lambda s: s.lo)
    for a, b in zip(order, order[1:]):
        if a.hi != b.lo:
            raise ValueError("segment products must tile the chain contiguously")
    v = np.asarray(delta, dtype=np.float64).copy()
    acc = 0.0
    for part in order:
        v = v @ part.product.m
        acc += part.product.log_scale
        top = v.max()
        if top <= 0.0:
            raise RuntimeError("running state vector collapsed to zero while combining segments")
        acc += math.log(float(top))
        v /= top
    return math.log(float(v.sum())) + acc


def _check_k(params) -> None:
    if int(params.K) > MAX_PARALLEL_STATES:
        raise ValueError(f"parallel engine supports at most {MAX_PARALLEL_STATES} states, got {params.K}")


def _parallel_loglik_arrays(params: HmmParams, present: np.ndarray, lon: np.ndarray,
                            lat: np.ndarray, cfg: EngineConfig) -> float:
    """Array-level entry (engine.py:321-345); the MCMC driver's hook."""
    if np.asarray(present).size == 0:
        raise ValueError("observation sequence is empty")
    _check_k(params)
    present, lon, lat = _host_arrays(present, lon, lat)
    return float(_host_loglik_batch([params], present.view(np.bool_), lon, lat, cfg, raise_on_collapse=True)[0])


def parallel_loglik(params: HmmParams, obs: Sequence[Observation], cfg: EngineConfig) -> float:
    """Log-likelihood through the segmented engine (engine.py:348-359)."""
    present, lon, lat = observation_arrays(obs)
    return _parallel_loglik_arrays(params, present, lon, lat, cfg)


def parallel_loglik_batch(params_list, obs, cfg: EngineConfig) -> np.ndarray:
    """Batched-proposal entry: log-likelihood of every parameter set in
    ``params_list`` (common K) over one observation stream, in one launch.

    ``obs`` is a ``DeviceObservations``, a sequence of ``Observation`` or a
    ``(present, lon, lat)`` tuple.  Collapsed proposals return -inf (the MCMC
    driver treats non-finite values as rejections, reference bayes.py:768).
    """
    if isinstance(params_list, ParamPack):  # pre-packed (proposals.params_from_vectors)
        if params_list.K > MAX_PARALLEL_STATES:
            raise ValueError(f"parallel engine supports at most {MAX_PARALLEL_STATES} states, got {params_list.K}")
    else:
        params_list = list(params_list)
        if not params_list:
            raise ValueError("no parameter sets given")
        _check_k(params_list[0])
    if isinstance(obs, DeviceObservations):
        handle = obs
    elif isinstance(obs, tuple) and len(obs) == 3:
        if np.asarray(obs[0]).size == 0:
            raise ValueError("observation sequence is empty")
        pr, lo, la = _host_arrays(*obs)
        return _host_loglik_batch(params_list, pr.view(np.bool_), lo, la, cfg, raise_on_collapse=False)
    else:
        if len(obs) == 0:
            raise ValueError("observation sequence is empty")
        handle = _scratch_obs(*observation_arrays(obs))
    return handle.loglik_batch(params_list, cfg)
