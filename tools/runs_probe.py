"""Run-absorbing chain vs record-by-record kernel: device chain/tree times
(CUDA events) and the automatic decision, over BASELINE workloads and a
presence sweep at K=25.

    python tools/runs_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import fixtures as fx  # noqa: E402
import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

_native.profile_enable(True)


def timed(dev, plist, reps=20):
    cfg = eng.EngineConfig()
    v = dev.loglik_batch(plist, cfg)
    best = None
    for _ in range(reps):
        v = dev.loglik_batch(plist, cfg)
        c, f, s = _native.profile_last()
        if best is None or c + f < best[0] + best[1]:
            best = (c, f, s)
    return v, best


def compare(tag, plist, pr, lo, la):
    dev = eng.DeviceObservations(pr, lo, la)
    k = plist[0].K
    info = dev.runs_info(k)
    out = {}
    for mode in (0, 1):
        _native.set_runs_mode(mode)
        v, (c, f, s) = timed(dev, plist)
        out[mode] = (np.array(v, copy=True), c, f, s, _native.profile_runs())
    _native.set_runs_mode(-1)
    (v0, c0, f0, s0, r0), (v1, c1, f1, s1, r1) = out[0], out[1]
    n = pr.size * len(plist)
    d = float(np.max(np.abs(v1 - v0) / np.abs(v0)))
    print(f"{tag:28s} K={k:2d} B={len(plist):3d} steps/rec~{info['steps_per_record']:.3f} auto={'runs' if info['active'] else 'rec '}"
          f" | record: chain {c0:8.3f} fold {f0:6.3f} ms ({n / (c0 + f0) / 1e6:6.3f} Gobs/s, {s0} segs)"
          f" | runs: chain {c1:8.3f} fold {f1:6.3f} ms ({n / (c1 + f1) / 1e6:6.3f} Gobs/s, {s1} segs)"
          f" | speedup {(c0 + f0) / (c1 + f1):5.2f}x  rel diff {d:.1e}", flush=True)
    dev.close()


for wl in ("k25_n1e6", "k5_n1e4"):
    plist, pr, lo, la = synth.make_workload(wl)
    compare(wl, plist, pr, lo, la)
for wl, n in (("k50_n1e7", 2_000_000), ("k80_n1e8", 500_000)):
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    compare(f"{wl} (N={n})", plist, pr, lo, la)
plist, pr, lo, la = synth.make_workload("k25_n1e6_b256")
compare("k25_n1e6_b256 (B=256)", plist, pr, lo, la)
rng = np.random.default_rng(9)
for k in (8, 16, 25, 32):
    p = fx.random_params(rng, k)
    for prob in (0.02, 0.13, 0.3, 0.5):
        pr = rng.random(1_000_000) < prob
        lo = np.where(pr, rng.uniform(-1.5, 1.5, pr.size), 0.0)
        la = np.where(pr, rng.uniform(-1.5, 1.5, pr.size), 0.0)
        compare(f"random present={prob}", [p], pr, lo, la)
