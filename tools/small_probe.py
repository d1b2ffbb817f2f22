"""Device time of small chains (MCMC-sized) vs the segment count: chain +
tree phases of the matrix path for explicit segment counts.

    python tools/small_probe.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

_native.require_device()
_native.profile_enable(True)
for wl, n in (("k5_n1e4", None), ("k25_n1e6", 20_000), ("k25_n1e6", 105_000)):
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    dev = eng.DeviceObservations(pr, lo, la)
    for segs in (None, 37, 74, 148, 296, 592, 1184, 2368):
        cfg = eng.EngineConfig(segments=segs)
        for _ in range(5):
            v = dev.loglik(plist[0], cfg)
        ts = []
        for _ in range(20):
            v = dev.loglik(plist[0], cfg)
            c, f, s = _native.profile_last()
            ts.append((c + f, c, f))
        ts.sort()
        t, c, f = ts[len(ts) // 2]
        print(f"{wl} n={pr.size} segments={segs}: used {s}  device {t * 1e3:.1f} us (chain {c * 1e3:.1f} tree {f * 1e3:.1f})",
              flush=True)
    dev.close()
