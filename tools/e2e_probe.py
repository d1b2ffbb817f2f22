"""Break down the host-array (e2e) evaluation: upload vs likelihood, graphs on/off."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import synth  # noqa: E402

plist, pr, lo, la = synth.make_workload("k25_n1e6")
p = plist[0]
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (pr.view(np.uint8), lo, la)]
pin[0] = pin[0].view(np.bool_)
cfg = eng.EngineConfig()
dev = eng.DeviceObservations(*pin)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print(f"assign (pinned 17 MB H2D + sync): {t(lambda: dev.assign(*pin)):.3f} ms")
print(f"loglik device-resident:          {t(lambda: dev.loglik(p, cfg)):.3f} ms")
print(f"assign + loglik:                 {t(lambda: (dev.assign(*pin), dev.loglik(p, cfg))):.3f} ms")
print(f"_parallel_loglik_arrays:         {t(lambda: eng._parallel_loglik_arrays(p, *pin, cfg)):.3f} ms")
from paper_2003_03508_b200 import _native  # noqa: E402
_native.profile_enable(True)
print(f"  ... with profiling events on:   {t(lambda: eng._parallel_loglik_arrays(p, *pin, cfg)):.3f} ms")
_native.profile_enable(False)
if hasattr(eng, "loglik_host_pipelined"):
    print(f"pipelined host entry:            {t(lambda: eng.loglik_host_pipelined(p, *pin, cfg)):.3f} ms")
