"""ctypes binding of the C-ABI in include/thmm.h (libthmm.so, built in-tree).

There is no fallback: if the shared library is missing or no CUDA device is
visible, every entry point raises.  The library is loaded lazily so that
importing the package (and the host-only helpers) works on machines without
a GPU.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint8, c_void_p

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libthmm.so")

THMM_OK, THMM_EINVAL, THMM_ECOLLAPSE, THMM_ECUDA = 0, 1, 2, 3
THMM_F64, THMM_F32, THMM_TF32, THMM_TF32X3, THMM_TF32X2 = 0, 1, 2, 3, 4
# EngineConfig.precision -> thmm_config.precision.  "tf32"/"tf32x2"/"tf32x3" are the
# precision-study extensions (tcgen05 tensor-core products, float32 semantics).
PRECISION_CODES = {"float64": THMM_F64, "float32": THMM_F32, "tf32": THMM_TF32, "tf32x3": THMM_TF32X3,
                   "tf32x2": THMM_TF32X2}
MAX_STATES = 80

# Every symbol include/thmm.h declares, with (restype, argtypes).
_obs = c_void_p
_dp = POINTER(c_double)
_u8p = POINTER(c_uint8)
_i32p = POINTER(c_int32)


class ThmmParams(ctypes.Structure):
    # pointers as c_void_p: built from ndarray.ctypes.data (an int) without the
    # ~3 us per-array cost of data_as(POINTER(...)) on the MCMC hot call
    _fields_ = [("K", c_int32), ("B", c_int32), ("gamma", c_void_p), ("delta", c_void_p), ("states", c_void_p)]


class ThmmConfig(ctypes.Structure):
    _fields_ = [("renorm_period", c_int32), ("precision", c_int32), ("segments", c_int64),
                ("lo", c_int64), ("hi", c_int64), ("stream", c_void_p)]


SIGNATURES = {
    "thmm_version": (c_int, []),
    "thmm_device_count": (c_int, []),
    "thmm_padded_states": (c_int, [c_int32]),
    "thmm_obs_create": (c_int, [_u8p, _dp, _dp, c_int64, c_int, POINTER(_obs), c_char_p, c_size_t]),
    "thmm_obs_assign": (c_int, [_obs, _u8p, _dp, _dp, c_int64, c_char_p, c_size_t]),
    "thmm_obs_assign_device": (c_int, [_obs, c_void_p, c_void_p, c_void_p, c_int64, c_char_p, c_size_t]),
    "thmm_obs_destroy": (c_int, [_obs]),
    "thmm_obs_length": (c_int64, [_obs]),
    "thmm_obs_device": (c_int, [_obs]),
    "thmm_loglik": (c_int, [_obs, POINTER(ThmmParams), POINTER(ThmmConfig), c_void_p, c_void_p, c_char_p, c_size_t]),
    "thmm_range_nodes": (c_int, [_obs, POINTER(ThmmParams), POINTER(ThmmConfig), c_void_p, c_void_p,
                                 c_char_p, c_size_t]),
    "thmm_range_nodes_async": (c_int, [_obs, POINTER(ThmmParams), POINTER(ThmmConfig), c_void_p, c_void_p,
                                       c_char_p, c_size_t]),
    "thmm_range_nodes_host": (c_int, [_obs, _u8p, _dp, _dp, c_int64, POINTER(ThmmParams), POINTER(ThmmConfig),
                                      c_void_p, c_void_p, c_char_p, c_size_t]),
    "thmm_fold_nodes": (c_int, [POINTER(ThmmParams), c_int32, c_void_p, c_void_p, c_int, c_void_p, _dp, _i32p,
                                c_char_p, c_size_t]),
    "thmm_fold_nodes_strided": (c_int, [POINTER(ThmmParams), c_int32, c_void_p, c_int64, c_void_p, c_int64, c_int,
                                        c_void_p, _dp, _i32p, c_char_p, c_size_t]),
    "thmm_peer_create": (c_int, [c_int, c_int, c_int, c_int64, POINTER(c_void_p), c_void_p, c_char_p, c_size_t]),
    "thmm_peer_open": (c_int, [c_void_p, c_void_p, c_char_p, c_size_t]),
    "thmm_peer_loglik": (c_int, [c_void_p, _obs, _u8p, _dp, _dp, c_int64, POINTER(ThmmParams), POINTER(ThmmConfig),
                                 _dp, _i32p, c_char_p, c_size_t]),
    "thmm_peer_destroy": (c_int, [c_void_p]),
    "thmm_host_register": (c_int, [c_void_p, c_size_t, c_char_p, c_size_t]),
    "thmm_host_unregister": (c_int, [c_void_p]),
    "thmm_emissions": (c_int, [_obs, POINTER(ThmmParams), c_int64, c_int64, _dp, c_char_p, c_size_t]),
    "thmm_emissions_chain": (c_int, [_obs, POINTER(ThmmParams), c_int64, c_int64, _dp, c_char_p, c_size_t]),
    "thmm_filtered_state": (c_int, [_obs, POINTER(ThmmParams), POINTER(ThmmConfig), _dp, _i32p, c_char_p,
                                    c_size_t]),
    "thmm_loglik_host": (c_int, [_obs, c_void_p, c_void_p, c_void_p, c_int64, POINTER(ThmmParams),
                                 POINTER(ThmmConfig), c_void_p, c_void_p, c_char_p, c_size_t]),
    "thmm_loglik_mapped": (c_int, [_obs, c_void_p, c_void_p, c_void_p, c_int64, POINTER(ThmmParams),
                                   POINTER(ThmmConfig), c_void_p, c_void_p, c_char_p, c_size_t]),
    "thmm_stationary": (c_int, [_dp, c_int32, c_int32, c_double, c_int32, c_int, _dp, _i32p, c_char_p,
                                c_size_t]),
    "thmm_csv_count": (c_int, [c_char_p, POINTER(c_int64), c_char_p, c_size_t]),
    "thmm_csv_read": (c_int, [c_char_p, c_int64, _u8p, _dp, _dp, POINTER(c_int64), c_char_p, c_size_t]),
    "thmm_factor_segments": (c_int, [_dp, c_int64, c_int32, c_int64, c_int32, c_int, _dp, _dp, c_char_p,
                                     c_size_t]),
    "thmm_last_launch_count": (c_int, []),
    "thmm_profile_enable": (c_int, [c_int]),
    "thmm_profile_last": (c_int, [_dp, _dp, POINTER(c_int64)]),
    "thmm_plan_info": (c_int, [c_int32, c_int32, c_int, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p]),
    "thmm_runs_info": (c_int, [c_void_p, c_int32, c_int32, _i32p, _dp, _i32p, _i32p, _i32p, _i32p, _i32p]),
    "thmm_profile_runs": (c_int, []),
    "thmm_set_runs_mode": (c_int, [c_int]),
    "thmm_set_collapse_mode": (c_int, [c_int]),
    "thmm_profile_phases": (c_int, [_dp, _dp]),
    "thmm_set_stitch_mode": (c_int, [c_int]),
    "thmm_stitch_shard": (c_int, [_obs, POINTER(ThmmParams), POINTER(ThmmConfig), c_int32, c_void_p, c_char_p,
                                  c_size_t]),
    "thmm_stitch_link": (c_int, [_obs, POINTER(ThmmParams), POINTER(ThmmConfig), c_void_p, c_int64, c_void_p,
                                 c_char_p, c_size_t]),
    "thmm_stitch_shard_host": (c_int, [_obs, c_void_p, c_void_p, c_void_p, c_int64, POINTER(ThmmParams),
                                       POINTER(ThmmConfig), c_int32, c_void_p, c_char_p, c_size_t]),
    "thmm_stitch_segments": (c_int64, [_obs, c_int32, c_int32]),
    "thmm_profile_collect": (c_int, []),
    "thmm_stitch_reruns": (ctypes.c_longlong, []),
    "thmm_set_collapse_params": (c_int, [c_double, c_int64, c_double]),
    "thmm_collapse_stats": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64), _dp]),
}

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """The CUDA library could not be loaded or no device is visible."""


def load_library(path: str = LIB_PATH):
    """Load libthmm.so and bind every C-ABI symbol (raises if missing)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def raise_for(rc: int, err: ctypes.Array) -> None:
    if rc == THMM_OK:
        return
    msg = err.value.decode(errors="replace") or f"thmm error {rc}"
    if rc == THMM_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def errbuf():
    return ctypes.create_string_buffer(512)


def as_ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(POINTER(ctype))


def require_device() -> None:
    n = lib().thmm_device_count()
    if n < 1:
        raise NativeUnavailable("no CUDA device is visible; the B200 likelihood has no CPU fallback")


def last_launch_count() -> int:
    return int(lib().thmm_last_launch_count())


def profile_enable(on: bool = True) -> None:
    lib().thmm_profile_enable(1 if on else 0)


def profile_last():
    """(chain_ms, fold_ms, segments) of the calling thread's last call."""
    a, b, s = c_double(), c_double(), c_int64()
    lib().thmm_profile_last(ctypes.byref(a), ctypes.byref(b), ctypes.byref(s))
    return a.value, b.value, s.value


def runs_info(handle, k: int, precision: str = "float64") -> dict:
    """Whether the handle's evaluations at (K, precision) use the run-absorbing
    chain, its estimated steps per record and launch plan (thmm_runs_info)."""
    act, g, w, r, c, big_r = (c_int32() for _ in range(6))
    spr = c_double()
    rc = lib().thmm_runs_info(handle, int(k), PRECISION_CODES[precision], ctypes.byref(act), ctypes.byref(spr),
                              ctypes.byref(g), ctypes.byref(w), ctypes.byref(r), ctypes.byref(c),
                              ctypes.byref(big_r))
    if rc != THMM_OK:
        raise RuntimeError(f"thmm_runs_info failed ({rc})")
    return dict(active=bool(act.value), steps_per_record=spr.value, G=g.value, W=w.value, regs=r.value,
                ctas_per_sm=c.value, R=big_r.value)


def set_runs_mode(mode: int) -> None:
    """Run-absorbing chain: -1 automatic (cost model), 0 never, 1 always when eligible."""
    if lib().thmm_set_runs_mode(int(mode)) != THMM_OK:
        raise ValueError(f"runs mode must be -1, 0 or 1, got {mode}")


def set_collapse_mode(mode: int) -> None:
    """1: rank-one collapse of converged segments (default), 0: off."""
    if lib().thmm_set_collapse_mode(int(mode)) != THMM_OK:
        raise ValueError("collapse mode must be 0 or 1")


def profile_phases():
    """(mode, phase-1 ms, phase-2 ms) of the last profiled evaluation: mode 0
    matrix path, 1 rank-one collapse (burn-in, vector continuation), 2
    stitched chain (main pass, links)."""
    a, b = ctypes.c_double(), ctypes.c_double()
    mode = lib().thmm_profile_phases(ctypes.byref(a), ctypes.byref(b))
    return int(mode), a.value, b.value


def set_stitch_mode(mode: int) -> None:
    """1: stitched chain for whole-chain evaluations in collapse mode (default), 0: off."""
    if lib().thmm_set_stitch_mode(int(mode)) != THMM_OK:
        raise ValueError("stitch mode must be 0 or 1")


def stitch_reruns() -> int:
    """Stitched evaluations repeated on the collapse path (a link did not converge)."""
    return int(lib().thmm_stitch_reruns())


def set_collapse_params(tol: float = 0.0, min_len: int = 0, min_fill: float = 0.0) -> None:
    """Rank-one test tolerance, shortest collapse-mode segment, and the gate
    (B n >= min_fill x 1024 x one wave of vector rows; negative: no gate);
    0 keeps the current value."""
    if lib().thmm_set_collapse_params(float(tol), int(min_len), float(min_fill)) != THMM_OK:
        raise ValueError("tolerance and minimum length must be >= 0")


def collapse_stats(handle) -> dict:
    """Segments of the handle's last collapse-mode evaluation: total,
    collapsed, and records spent in the matrix burn-in."""
    nodes, col, burned = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    rc = lib().thmm_collapse_stats(handle, ctypes.byref(nodes), ctypes.byref(col), ctypes.byref(burned))
    if rc != THMM_OK:
        return {"nodes": int(nodes.value), "collapsed": 0, "burn_records": 0.0}
    return {"nodes": int(nodes.value), "collapsed": int(col.value), "burn_records": float(burned.value)}


def profile_runs() -> bool:
    """True if the calling thread's last likelihood call ran the run-absorbing chain."""
    return bool(lib().thmm_profile_runs())


def plan_info(k: int, precision: str = "float64", device: int = 0) -> dict:
    """Launch plan for K states (diagnostic; see thmm_plan_info)."""
    vals = [c_int32() for _ in range(6)]
    rc = lib().thmm_plan_info(int(k), PRECISION_CODES[precision], int(device),
                              *[ctypes.byref(v) for v in vals])
    if rc != THMM_OK:
        raise RuntimeError(f"thmm_plan_info failed ({rc})")
    return dict(zip(("nt", "tail", "G", "W", "regs", "ctas_per_sm"), (v.value for v in vals)))
