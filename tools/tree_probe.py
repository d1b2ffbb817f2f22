"""Latency of the one-launch segment tree vs node count S and K: wall time of
thmm_fold_nodes (finish mode) on device-resident nodes, median of many calls.
The slope over log4(S) is the per-level latency.

    python tools/tree_probe.py
"""
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures as fx  # noqa: E402
import paper_2003_03508_b200 as eng  # noqa: E402

rng = np.random.default_rng(5)
for k in (5, 25, 50, 80):
    p = fx.random_params(rng, k)
    kp = eng.padded_states(k)
    row = []
    for s in (1, 4, 16, 64, 256, 1024, 4096):
        m = torch.rand((s, 1, kp, kp), dtype=torch.float64, device="cuda") * 0.5 + 0.25
        m[:, :, k:, :] = 0
        m[:, :, :, k:] = 0
        e = torch.zeros((s, 1), dtype=torch.float64, device="cuda")
        for _ in range(5):
            eng.fold_nodes([p], m.data_ptr(), e.data_ptr(), s, device=0)
        ts = []
        for _ in range(50):
            t0 = time.perf_counter()
            eng.fold_nodes([p], m.data_ptr(), e.data_ptr(), s, device=0)
            ts.append(time.perf_counter() - t0)
        row.append((s, 1e6 * float(np.median(ts))))
    base = row[0][1]
    print(f"K={k:2d} " + "  ".join(f"S={s}:{t:6.1f}us" for s, t in row) +
          f"   per level ~{(row[-1][1] - row[1][1]) / (math.log(4096, 4) - 1):.1f} us", flush=True)
