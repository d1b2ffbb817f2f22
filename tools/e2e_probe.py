"""End-to-end reference-API calls (pageable host arrays, zero-copy reads)
against the device-resident evaluation, per path (stitched chain on / off).

    python tools/e2e_probe.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

_native.require_device()


def med(fn, reps):
    for _ in range(max(5, reps // 4)):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


CASES = (("k25_n1e6", None, 60), ("k80_n1e8", 10_000_000, 20), ("k50_n1e7", None, 30))
if len(sys.argv) > 1:  # e.g. k80_n1e8:0:8  (workload, n (0 = full), reps)
    CASES = tuple((w, int(n) or None, int(r)) for w, n, r in (a.split(":") for a in sys.argv[1:]))
for wl, n, reps in CASES:
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    p = plist[0]
    cfg = eng.EngineConfig()
    dev = eng.DeviceObservations(pr, lo, la)
    for st in ((1, 0) if os.environ.get("PROBE_NOSTITCH", "1") == "1" else (1,)):
        _native.set_stitch_mode(st)
        t_dev = med(lambda: dev.loglik(p, cfg), reps)
        t_api = med(lambda: eng._parallel_loglik_arrays(p, pr, lo, la, cfg), reps)
        _native.profile_enable(True)
        dev.loglik(p, cfg)
        ph_dev = _native.profile_phases()
        eng._parallel_loglik_arrays(p, pr, lo, la, cfg)
        eng._parallel_loglik_arrays(p, pr, lo, la, cfg)
        ph_api = _native.profile_phases()
        _native.profile_enable(False)
        print(f"{wl} n={pr.size} stitch={st}: device-resident {t_dev:.3f} ms  reference API (pageable host arrays) "
              f"{t_api:.3f} ms  | phases (mode, main/burn-in ms, links/vector ms): device {ph_dev}  api {ph_api}",
              flush=True)
    _native.set_stitch_mode(1)
    dev.close()

# host->device bandwidth of this box: DMA from pinned memory
import torch  # noqa: E402

if os.environ.get("PROBE_DMA", "1") != "1":
    sys.exit(0)

for mb in (17, 170):
    h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"H2D DMA {mb} MiB pinned: {ms:.3f} ms = {mb * 1.048576 / ms:.1f} GB/s", flush=True)
