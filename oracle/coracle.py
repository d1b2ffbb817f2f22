"""ctypes binding of oracle/thmm_oracle.c -- TEST INFRASTRUCTURE ONLY.

Same duck-typed parameters as oracle/thmm_oracle.py; see thmm_oracle.c for
the reference file:line each function restates.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_uint8

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "liboracle.so")
FIELDS = ("_p", "_q", "_mu0", "_mu1", "_l00", "_l10", "_l11", "_log_det")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            from paper_2003_03508_b200.build import build_oracle
            build_oracle()
        lib = ctypes.CDLL(LIB)
        dp, u8p, ip = POINTER(c_double), POINTER(c_uint8), POINTER(c_int)
        lib.thmo_forward.restype = c_double
        lib.thmo_forward.argtypes = [c_int, dp, dp, dp, u8p, dp, dp, c_int64, c_int, ip]
        lib.thmo_parallel.restype = c_double
        lib.thmo_parallel.argtypes = [c_int, dp, dp, dp, u8p, dp, dp, c_int64, c_int64, c_int, c_int, ip]
        lib.thmo_segments.restype = c_int
        lib.thmo_segments.argtypes = [c_int, dp, dp, u8p, dp, dp, c_int64, c_int64, c_int, c_int, dp, dp]
        lib.thmo_emissions.restype = None
        lib.thmo_emissions.argtypes = [c_int, dp, u8p, dp, dp, c_int64, dp]
        _lib = lib
    return _lib


def _p(a, t=c_double):
    return a.ctypes.data_as(POINTER(t))


def _prep(params, present, lon, lat):
    k = len(params._p)
    g = np.ascontiguousarray(params.gamma, dtype=np.float64)
    d = np.ascontiguousarray(params.delta, dtype=np.float64)
    st = np.ascontiguousarray(np.stack([np.asarray(getattr(params, f), dtype=np.float64) for f in FIELDS]))
    pr = np.ascontiguousarray(present, dtype=np.bool_).view(np.uint8)
    lo = np.ascontiguousarray(lon, dtype=np.float64)
    la = np.ascontiguousarray(lat, dtype=np.float64)
    return k, g, d, st, pr, lo, la


def forward_loglik(params, present, lon, lat, renorm_period=1):
    """Serial Algorithm 1 (reference core.py:270-302); -inf on collapse."""
    if np.asarray(present).size == 0:
        raise ValueError("observation sequence is empty")
    k, g, d, st, pr, lo, la = _prep(params, present, lon, lat)
    status = c_int(0)
    return _load().thmo_forward(k, _p(g), _p(d), _p(st), _p(pr, c_uint8), _p(lo), _p(la), pr.size,
                                int(renorm_period), ctypes.byref(status))


def parallel_loglik(params, present, lon, lat, segments, renorm_period=8, threads=None):
    """Segmented engine (reference engine.py:321-345); RuntimeError on collapse."""
    if np.asarray(present).size == 0:
        raise ValueError("observation sequence is empty")
    k, g, d, st, pr, lo, la = _prep(params, present, lon, lat)
    threads = os.cpu_count() if threads is None else threads
    status = c_int(0)
    v = _load().thmo_parallel(k, _p(g), _p(d), _p(st), _p(pr, c_uint8), _p(lo), _p(la), pr.size,
                              int(segments), int(renorm_period), int(threads), ctypes.byref(status))
    if status.value == 2:
        raise RuntimeError("running state vector collapsed to zero while combining segments")
    if status.value:
        raise ValueError("invalid arguments")
    return v


def segment_products(params, present, lon, lat, segments, renorm_period=8, threads=None):
    k, g, d, st, pr, lo, la = _prep(params, present, lon, lat)
    ms = np.empty((segments, k, k))
    ls = np.empty(segments)
    threads = os.cpu_count() if threads is None else threads
    rc = _load().thmo_segments(k, _p(g), _p(st), _p(pr, c_uint8), _p(lo), _p(la), pr.size, int(segments),
                               int(renorm_period), int(threads), _p(ms), _p(ls))
    if rc:
        raise ValueError("invalid arguments")
    return ms, ls


def emissions(params, present, lon, lat):
    k, g, d, st, pr, lo, la = _prep(params, present, lon, lat)
    out = np.empty((pr.size, k))
    _load().thmo_emissions(k, _p(st), _p(pr, c_uint8), _p(lo), _p(la), pr.size, _p(out))
    return out
