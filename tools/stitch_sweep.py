"""Stitched-chain time vs segment length for chains below the default gate
(where the matrix paths run): K=25 N=1e6 (configs[1]) and Shikoku-sized
chains.  Prints links that failed (evaluations repeated on the collapse path).

    python tools/stitch_sweep.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

_native.require_device()
for wl, n in (("k25_n1e6", None), ("k25_n1e6", 105_000), ("k5_n1e4", None), ("k50_n1e7", 1_000_000)):
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    _native.profile_enable(True)
    for ml, fill in ((0, 0.25), (96, -1.0), (128, -1.0), (192, -1.0), (256, -1.0), (384, -1.0), (512, -1.0)):
        _native.set_collapse_params(0.0, ml or 1024, fill)
        r0 = _native.stitch_reruns()
        for _ in range(3):
            v = dev.loglik_batch(plist, cfg)
        ts = []
        for _ in range(10):
            v = dev.loglik_batch(plist, cfg)
            c, f, s = _native.profile_last()
            ts.append(c + f)
        mode = _native.profile_phases()[0]
        print(f"{wl} n={pr.size} minlen={ml or 1024} gate={fill}: mode {mode} segs {s} device {statistics.median(ts):.3f} ms "
              f"reruns {_native.stitch_reruns() - r0} ll {v[0]:.10f}", flush=True)
    dev.close()
_native.set_collapse_params(0.0, 1024, 0.25)
