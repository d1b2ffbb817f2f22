"""Where the time of one small likelihood call goes (MCMC-sized chains):
Python packing, config, the C call (graph replay + wait), device phases, and
the reference API from pageable arrays.

    python tools/latency_breakdown.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native as nat, synth  # noqa: E402
from paper_2003_03508_b200.engine import _PackedParams, _native_config  # noqa: E402


def med(fn, reps=200):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts))


cases = [("k5_n1e4", None), ("k25_n1e6", 105_000), ("k25_n1e6", 20_000), ("k50_n1e7", 105_000)]
for wl, n in cases:
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    p = plist[0]
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    t_pack = med(lambda: _PackedParams([p]))
    t_cfg = med(lambda: _native_config(cfg, 0, 0, 0))
    pp = _PackedParams([p])
    c = _native_config(cfg, 0, 0, 0)
    out = np.empty(1)
    st = np.empty(1, dtype=np.int32)
    err = nat.errbuf()
    t_c = med(lambda: nat.lib().thmm_loglik(dev._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                            nat.as_ptr(out, nat.c_double), nat.as_ptr(st, nat.c_int32), err, len(err)))
    t_dev = med(lambda: dev.loglik(p, cfg))
    nat.profile_enable(True)
    dev.loglik(p, cfg)
    ch, fo, segs = nat.profile_last()
    mode = nat.profile_phases()[0]
    nat.profile_enable(False)
    t_api = med(lambda: eng._parallel_loglik_arrays(p, pr, lo, la, cfg), reps=100)
    from paper_2003_03508_b200 import engine as _e
    t_ha = med(lambda: _e._host_arrays(pr, lo, la))
    hpr, hlo, hla = _e._host_arrays(pr, lo, la)
    t_pin = med(lambda: _e._auto_pin(hpr, hlo, hla))
    scratch = _e._scratch.pool[_e.default_device()]
    t_map = med(lambda: nat.lib().thmm_loglik_mapped(scratch._handle, hpr.ctypes.data, hlo.ctypes.data, hla.ctypes.data,
                                                     hpr.size, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                                     out.ctypes.data, st.ctypes.data, err, len(err)))
    t_hb = med(lambda: scratch.loglik_host_batch([p], hpr.view(np.bool_), hlo, hla, cfg, raise_on_collapse=True,
                                                 mapped=True))
    print(f"{wl:9s} n={pr.size:8d}  pack {t_pack:6.1f} us  cfg {t_cfg:5.1f} us  C call {t_c:7.1f} us  "
          f"dev.loglik {t_dev:7.1f} us  reference API (pageable) {t_api:7.1f} us  |  device chain {1e3 * ch:6.1f} "
          f"tree {1e3 * fo:5.1f} us  segs {segs}  mode {mode}", flush=True)
    print(f"{'':9s} host-array call: _host_arrays {t_ha:5.1f} us  _auto_pin {t_pin:5.1f} us  "
          f"thmm_loglik_mapped (C) {t_map:6.1f} us  loglik_host_batch {t_hb:6.1f} us", flush=True)
    dev.close()
