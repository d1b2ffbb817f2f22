"""Precision study probe: every engine precision vs the FP64 path, plus chain
timings on the bench workloads (device-resident stream).

    python tools/tc_probe.py [--perf] [--ks 5,25,50,80]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import fixtures as fx  # noqa: E402
import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ks", default="1,2,5,8,9,16,17,25,31,33,48,50,64,65,72,79,80")
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--perf", action="store_true")
ap.add_argument("--perf-n80", type=int, default=10_000_000)
a = ap.parse_args()

PRECS = ("float32", "tf32", "tf32x2", "tf32x3")
for k in [int(x) for x in a.ks.split(",")]:
    rng = np.random.default_rng(1000 + k)
    p = fx.random_params(rng, k)
    pr, lo, la = fx.random_obs_arrays(rng, a.n)
    ref = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())
    out = [f"K={k:2d} f64={ref:.10f}"]
    for prec in PRECS:
        v = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(precision=prec))
        out.append(f"{prec}={abs(v - ref) / abs(ref):.2e}")
    for prec in ("tf32", "tf32x2", "tf32x3"):
        plan = _native.plan_info(k, prec)
        out.append(f"[{prec} W={plan['W']} G={plan['G']} regs={plan['regs']}]")
    print(" ".join(out), flush=True)

if a.perf:
    _native.profile_enable(True)
    for wl, n in (("k25_n1e6", None), ("k50_n1e7", None), ("k80_n1e8", a.perf_n80), ("k25_n1e6_b256", None)):
        plist, pr, lo, la = synth.make_workload(wl, n=n)
        dev = eng.DeviceObservations(pr, lo, la)
        K, N, B = plist[0].K, pr.size, len(plist)
        base = None
        for prec in ("float64", "float32", "tf32", "tf32x2", "tf32x3"):
            if B > 1 and prec == "float32":
                continue
            cfg = eng.EngineConfig(precision=prec)
            dev.loglik_batch(plist, cfg)
            best = None
            for _ in range(3):
                t0 = time.perf_counter()
                v = dev.loglik_batch(plist, cfg)
                wall = time.perf_counter() - t0
                c, f, s = _native.profile_last()
                best = (c, f, s, wall) if best is None or c < best[0] else best
            if prec == "float64":
                base = v
            c, f, s, wall = best
            err = float(np.max(np.abs(v - base) / np.abs(base)))
            print(f"{wl} N={N} B={B} {prec:8s} chain={c:.3f} ms fold={f:.3f} ms wall={1e3 * wall:.2f} ms "
                  f"segs={s} alg TFLOP/s={2 * K ** 3 * N * B / c / 1e9:.1f} obs/s={N * B / (c + f) * 1e3:.3e} "
                  f"max rel vs f64={err:.2e}", flush=True)
