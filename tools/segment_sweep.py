"""Wall time of one device-resident evaluation vs the segment count, for
short chains where the chain/tree balance decides latency.

    python tools/segment_sweep.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import fixtures as fx  # noqa: E402
import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native  # noqa: E402

for k, n in ((5, 10_000), (5, 105_000), (10, 105_000), (25, 105_000), (25, 1_000_000)):
    rng = np.random.default_rng(k)
    p = fx.random_params(rng, k)
    pr, lo, la = fx.random_obs_arrays(rng, n)
    dev = eng.DeviceObservations(pr, lo, la)
    res = []
    for segs in (None, 148, 296, 592, 1184, 2368, 4736, 9472):
        if segs is not None and segs > n // 4:
            continue
        cfg = eng.EngineConfig(segments=segs)
        for _ in range(3):
            dev.loglik(p, cfg)
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            dev.loglik(p, cfg)
            ts.append(time.perf_counter() - t0)
        res.append(f"{'auto' if segs is None else segs}:{1e6 * np.median(ts):.0f}")
    print(f"K={k} N={n}: " + " ".join(res) + " (us)", flush=True)
