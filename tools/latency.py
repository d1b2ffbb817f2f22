"""Per-call wall latency of a device-resident likelihood evaluation (the MCMC
inner loop: new parameters every call, observations resident).

    python tools/latency.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

for name, n in (("k5_n1e4", 10_000), ("k25_n1e6", 100_000), ("k25_n1e6", 1_000_000), ("k50_n1e7", 100_000)):
    plist, pr, lo, la = synth.make_workload(name, n=n)
    p = plist[0]
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    _native.profile_enable(True)
    for _ in range(5):
        dev.loglik(p, cfg)
    reps = 200 if n <= 100_000 else 50
    t0 = time.perf_counter()
    for _ in range(reps):
        v = dev.loglik(p, cfg)
    dt = (time.perf_counter() - t0) / reps
    c, f, s = _native.profile_last()
    t1 = time.perf_counter()
    for _ in range(reps):
        eng.pack_params([p])
    pk = (time.perf_counter() - t1) / reps
    print(f"{name} N={n}: {1e6*dt:8.1f} us/call  chain {1e3*c:8.1f} us  fold {1e3*f:6.1f} us  "
          f"pack {1e6*pk:5.1f} us  segments {s}  launches {_native.last_launch_count()}  loglik {v:.6f}", flush=True)
