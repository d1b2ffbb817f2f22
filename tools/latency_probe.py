"""Chain / tree split and per-call wall time of device-resident evaluations
for short chains (config 0 and Shikoku-sized N ~ 1e5, the MCMC use case).

    python tools/latency_probe.py
"""
import sys, time, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2003_03508_b200 as eng
from paper_2003_03508_b200 import _native, synth
import fixtures as fx
_native.profile_enable(True)
for wl in ("k5_n1e4",):
    plist, pr, lo, la = synth.make_workload(wl)
    dev = eng.DeviceObservations(pr, lo, la)
    for _ in range(3): v = dev.loglik_batch(plist, eng.EngineConfig())
    ts=[]
    for _ in range(50):
        t0=time.perf_counter(); v = dev.loglik_batch(plist, eng.EngineConfig()); ts.append(time.perf_counter()-t0)
    c,f,s = _native.profile_last()
    print(wl, "wall %.1f us" % (1e6*np.median(ts)), "chain %.1f fold %.1f segs %d" % (1e3*c, 1e3*f, s), v[0])
for k, n in ((25, 20000), (50, 20000), (80, 5000), (5, 105000), (8, 105000), (10, 105000), (16, 105000), (25, 105000), (30, 105000)):
    rng = np.random.default_rng(k); p = fx.random_params(rng, k); pr, lo, la = fx.random_obs_arrays(rng, n)
    dev = eng.DeviceObservations(pr, lo, la)
    for _ in range(3): v = dev.loglik(p, eng.EngineConfig())
    ts=[]
    for _ in range(30):
        t0=time.perf_counter(); v = dev.loglik(p, eng.EngineConfig()); ts.append(time.perf_counter()-t0)
    c,f,s = _native.profile_last()
    print(k, n, "wall %.1f us" % (1e6*np.median(ts)), "chain %.1f fold %.1f segs %d" % (1e3*c, 1e3*f, s))
