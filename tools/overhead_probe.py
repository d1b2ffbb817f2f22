"""Per-call host overhead of the device-resident likelihood (small problems,
where the MCMC inner loop is latency-bound): Python packing vs the C call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native as nat, synth  # noqa: E402
from paper_2003_03508_b200.engine import _PackedParams, _native_config  # noqa: E402


def med(fn, reps=200):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts))


plist, pr, lo, la = synth.make_workload("k5_n1e4")
p = plist[0]
dev = eng.DeviceObservations(pr, lo, la)
cfg = eng.EngineConfig()
print(f"dev.loglik (full python path):   {med(lambda: dev.loglik(p, cfg)):7.1f} us")
print(f"  _PackedParams([p]):            {med(lambda: _PackedParams([p])):7.1f} us")
print(f"  _native_config:                {med(lambda: _native_config(cfg)):7.1f} us")
pp = _PackedParams([p])
c = _native_config(cfg)
out = np.empty(1)
st = np.empty(1, dtype=np.int32)
err = nat.errbuf()


def raw():
    nat.lib().thmm_loglik(dev._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c), nat.as_ptr(out, nat.c_double),
                          nat.as_ptr(st, nat.c_int32), err, len(err))


print(f"  raw thmm_loglik ctypes call:   {med(raw):7.1f} us")
nat.profile_enable(True)
raw()
ch, fo, _ = nat.profile_last()
print(f"  GPU chain + tree (events):     {1e3 * (ch + fo):7.1f} us")
