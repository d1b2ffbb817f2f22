"""Stability of the e2e leg: the host-array evaluation timed in blocks of 100
calls over ~3 s, in a fresh process (as bench.py's e2e leg runs).

    python tools/e2e_blocks.py [--blocks 20]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=20)
ap.add_argument("--per", type=int, default=100)
a = ap.parse_args()

plist, pr, lo, la = synth.make_workload("k25_n1e6")
p = plist[0]
cfg = eng.EngineConfig()
pin_pr = torch.from_numpy(pr.view(np.uint8)).pin_memory().numpy().view(np.bool_)
pin_lo = torch.from_numpy(lo).pin_memory().numpy()
pin_la = torch.from_numpy(la).pin_memory().numpy()
for _ in range(3):
    eng._parallel_loglik_arrays(p, pin_pr, pin_lo, pin_la, cfg)
torch.cuda.synchronize()
ms = []
for _ in range(a.blocks):
    t0 = time.perf_counter()
    for _ in range(a.per):
        eng._parallel_loglik_arrays(p, pin_pr, pin_lo, pin_la, cfg)
    torch.cuda.synchronize()
    ms.append((time.perf_counter() - t0) / a.per * 1e3)
print("block ms/step:", " ".join(f"{x:.3f}" for x in ms))
print(f"mean {np.mean(ms):.3f} median {np.median(ms):.3f} min {min(ms):.3f} max {max(ms):.3f}")
