"""Stitched chain in the under-filled regime: main-pass / link time per
record step for chains too short to fill a wave of rows (the paper's
catalogue sizes, configs[1], an 8-GPU shard of configs[2]/[3]), against the
path the default gate picks.

    python tools/stitch_latency.py [minlen ...]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

_native.require_device()
minlens = [int(a) for a in sys.argv[1:]] or [192]
cases = (("k5_n1e4", None), ("k25_n1e6", 20_000), ("k25_n1e6", 105_000), ("k25_n1e6", None),
         ("k50_n1e7", 105_000), ("k50_n1e7", 1_250_000), ("k80_n1e8", 105_000), ("k80_n1e8", 1_250_000))


def timed(dev, plist, cfg, reps=10):
    for _ in range(3):
        v = dev.loglik_batch(plist, cfg)
    ts, ph = [], []
    for _ in range(reps):
        v = dev.loglik_batch(plist, cfg)
        c, f, s = _native.profile_last()
        ts.append(c + f)
        ph.append(_native.profile_phases())
    return v[0], statistics.median(ts), s, ph[len(ph) // 2]


for wl, n in cases:
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    plist = plist[:1]
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    _native.profile_enable(True)
    _native.set_collapse_params(0.0, 1024, 0.25)
    ll0, t0, s0, ph0 = timed(dev, plist, cfg)
    print(f"{wl} n={pr.size}: default mode {ph0[0]} segs {s0} device {t0 * 1e3:.1f} us", flush=True)
    for ml in minlens:
        _native.set_collapse_params(0.0, ml, -1.0)
        r0 = _native.stitch_reruns()
        ll, t, s, (mode, a, b) = timed(dev, plist, cfg)
        steps = pr.size / max(s, 1)
        print(f"    stitched minlen {ml}: mode {mode} segs {s} device {t * 1e3:.1f} us  main {a * 1e3:.1f} us "
              f"({a * 1e3 / steps:.3f} us/step over {steps:.0f})  links {b * 1e3:.1f} us  reruns "
              f"{_native.stitch_reruns() - r0}  rel {abs(ll - ll0) / abs(ll0):.1e}", flush=True)
    dev.close()
_native.set_collapse_params(0.0, 1024, 0.25)
