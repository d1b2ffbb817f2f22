"""Phase times of the rank-one collapse path per workload (burn-in on the
run-absorbing chain, vector continuation, tree), against the matrix path.

    python tools/collapse_probe.py [--minlen 256,1024,4096] [--workloads k80_n1e8,...]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="k5_n1e4,k25_n1e6,k50_n1e7,k80_n1e8,k25_n1e6_b256")
ap.add_argument("--minlen", default="1024")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
_native.require_device()
for wl in a.workloads.split(","):
    plist, pr, lo, la = synth.make_workload(wl)
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    rows = []
    for mode, ml in [(0, 0), (2, 0)] + [(1, int(m)) for m in a.minlen.split(",")]:
        _native.set_collapse_mode(1 if mode else 0)
        _native.set_stitch_mode(1 if mode == 2 else 0)
        if ml:
            _native.set_collapse_params(0.0, ml)
        _native.profile_enable(True)
        for _ in range(2):
            v = dev.loglik_batch(plist, cfg)
        ch, fo, ph = [], [], []
        t0 = time.perf_counter()
        for _ in range(a.reps):
            v = dev.loglik_batch(plist, cfg)
            c, f, nseg = _native.profile_last()
            ch.append(c)
            fo.append(f)
            ph.append(_native.profile_phases())
        wall = (time.perf_counter() - t0) / a.reps * 1e3
        _native.profile_enable(False)
        st = _native.collapse_stats(dev._handle) if mode == 1 else {}
        burn = statistics.median(p[1] for p in ph) if mode else None
        vec = statistics.median(p[2] for p in ph) if mode else None
        print(f"{wl:14s} mode={ph[-1][0]} minlen={ml:5d} segs={nseg:6d} chain={statistics.median(ch):9.3f} ms "
              f"(burn {burn if burn is None else round(burn, 3)}, vec {vec if vec is None else round(vec, 3)}) "
              f"tree={statistics.median(fo):7.3f} wall={wall:9.3f} ms  stats={st}  ll0={v[0]:.10f}", flush=True)
    dev.close()
_native.set_collapse_mode(1)
_native.set_stitch_mode(1)
_native.set_collapse_params(0.0, 1024)
