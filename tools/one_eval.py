"""One (or a few) likelihood evaluations of a named workload -- for ncu / sanitizer runs.

    python tools/one_eval.py k80_n1e8 [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

wl = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
plist, pr, lo, la = synth.make_workload(wl)
dev = eng.DeviceObservations(pr, lo, la)
for _ in range(reps):
    v = dev.loglik_batch(plist, eng.EngineConfig())
print(wl, v[:4], _native.collapse_stats(dev._handle))
