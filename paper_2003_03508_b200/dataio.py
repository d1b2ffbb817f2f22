"""Observation CSV straight to arrays / a device stream.

The reference reads its dataset CSV (header ``timestamp,lon,lat``) with a
Python ``csv`` loop that builds one ``Observation`` per hour
(reference dataio.py:46-87), then ``observation_arrays`` splits them again
(core.py:209-222).  Here the native parser in libthmm (thmm_io.cu) fills
``present/lon/lat`` in one pass with the same validation and the same
``line N: ...`` errors, and ``load_device_observations`` uploads the result
once for the likelihood engine.
"""

from __future__ import annotations

import ctypes
import os
from typing import Tuple

import numpy as np

from . import _native as nat


def load_arrays(path, with_timestamps: bool = False):
    """``(present, lon, lat)`` (and ``t_us`` int64 microseconds since the
    epoch if requested) from an observation CSV; ValueError on bad input."""
    path_b = os.fsencode(os.fspath(path))
    lib = nat.lib()
    err = nat.errbuf()
    n = ctypes.c_int64()
    nat.raise_for(lib.thmm_csv_count(path_b, ctypes.byref(n), err, len(err)), err)
    present = np.zeros(n.value, dtype=np.uint8)
    lon = np.zeros(n.value, dtype=np.float64)
    lat = np.zeros(n.value, dtype=np.float64)
    t_us = np.zeros(n.value, dtype=np.int64) if with_timestamps else None
    tp = t_us.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if with_timestamps else None
    rc = lib.thmm_csv_read(path_b, n.value, nat.as_ptr(present, ctypes.c_uint8), nat.as_ptr(lon, ctypes.c_double),
                           nat.as_ptr(lat, ctypes.c_double), tp, err, len(err))
    nat.raise_for(rc, err)
    out: Tuple = (present.view(np.bool_), lon, lat)
    return out + (t_us,) if with_timestamps else out


def load_device_observations(path, device=None):
    """Parse an observation CSV and upload it as a ``DeviceObservations``."""
    from .engine import DeviceObservations

    present, lon, lat = load_arrays(path)
    if present.size == 0:
        raise ValueError("observation sequence is empty")
    return DeviceObservations(present, lon, lat, device=device)
