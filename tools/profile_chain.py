"""Run one workload through the device-resident path a few times (for ncu).

    python tools/profile_chain.py --workload k25_n1e6 --reps 3
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="k25_n1e6")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--segments", type=int, default=None)
ap.add_argument("--precision", default="float64")
a = ap.parse_args()
plist, pr, lo, la = synth.make_workload(a.workload, n=a.n)
dev = eng.DeviceObservations(pr, lo, la)
cfg = eng.EngineConfig(segments=a.segments, precision=a.precision)
_native.profile_enable(True)
for i in range(a.reps):
    t0 = time.perf_counter()
    v = dev.loglik_batch(plist, cfg)
    c, f, s = _native.profile_last()
    K = plist[0].K
    print(f"rep {i}: loglik[0]={v[0]:.10f} wall={1e3*(time.perf_counter()-t0):.3f} ms chain={c:.3f} ms "
          f"fold={f:.3f} ms segments={s} chain TFLOP/s={2*K**3*pr.size*len(plist)/c/1e9:.2f} {a.precision}", flush=True)
