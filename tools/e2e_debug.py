"""Why is the e2e leg slow inside bench.py?  Replays bench.py's sequence
(device-resident timed loop with profiling, L2 flush buffer, then the
zero-copy host-array calls) step by step and times the host-array call after
each stage.

    python tools/e2e_debug.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

plist, pr, lo, la = synth.make_workload("k25_n1e6")
cfg = eng.EngineConfig()
pin_pr = torch.from_numpy(pr.view(np.uint8)).pin_memory().numpy().view(np.bool_)
pin_lo = torch.from_numpy(lo).pin_memory().numpy()
pin_la = torch.from_numpy(la).pin_memory().numpy()


def e2e(tag, reps=100):
    for _ in range(20):
        eng._parallel_loglik_arrays(plist[0], pin_pr, pin_lo, pin_la, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        eng._parallel_loglik_arrays(plist[0], pin_pr, pin_lo, pin_la, cfg)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    print(f"{tag:50s} {ms:.3f} ms/call  launches={_native.last_launch_count()} runs={_native.profile_runs()}",
          flush=True)


e2e("fresh")
dev = eng.DeviceObservations(pr, lo, la)
e2e("after a device-resident handle")
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
flush.zero_()
e2e("after a 256 MiB flush buffer")
_native.profile_enable(True)
for _ in range(50):
    flush.zero_()
    dev.loglik_batch(plist, cfg, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
e2e("profiling on, after device loop")
_native.profile_enable(False)
e2e("profiling off again")
