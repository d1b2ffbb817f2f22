"""BASELINE.json configs[3]: FP64 vs FP32 / TF32 tensor-core tolerance study
on the full K=80, N=10^8 synthetic chain (1 GPU; the 8-GPU shard of the same
chain folds the same per-range nodes, see tests/test_gpu_tensorcore.py).

Every precision is timed on the device-resident stream (chain + segment tree,
CUDA events) and compared against the reference's own logL for this chain
(tests/golden/bench_configs.json, computed by the reference's kernels).

    python tools/precision_study.py [--workload k80_n1e8] [--reps 3] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native, synth  # noqa: E402

BOUNDS = {"float64": 1e-9, "float32": 1e-4, "tf32x3": 1e-6, "tf32x2": 1e-4, "tf32": 2e-3}

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="k80_n1e8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()

t0 = time.perf_counter()
plist, pr, lo, la = synth.make_workload(a.workload)
gen_s = time.perf_counter() - t0
with open(os.path.join(ROOT, "tests", "golden", "bench_configs.json")) as fh:
    gold = json.load(fh)["workloads"][a.workload]
want = np.array(gold["loglik"][: len(plist)])
dev = eng.DeviceObservations(pr, lo, la)
K, N, B = plist[0].K, pr.size, len(plist)
_native.profile_enable(True)
rows = []
print(f"{a.workload}: K={K} N={N} B={B} (synthetic data {gen_s:.1f} s); golden logL[0]={want[0]:.10f} "
      f"({gold.get('reference_method', 'reference engine')})", flush=True)
PATHS = {"stitched": (1, 1), "collapse": (1, 0), "matrix": (0, 0)}  # (collapse mode, stitch mode)
for prec, path in (("float64", "stitched"), ("float64", "collapse"), ("float64", "matrix"), ("float32", None),
                   ("tf32x3", None), ("tf32x2", None), ("tf32", None)):
    cm, sm = PATHS.get(path, (1, 1))
    _native.set_collapse_mode(cm)
    _native.set_stitch_mode(sm)
    cfg = eng.EngineConfig(precision=prec)
    v = dev.loglik_batch(plist, cfg)
    best = None
    for _ in range(a.reps):
        v = dev.loglik_batch(plist, cfg)
        c, f, s = _native.profile_last()
        if best is None or c + f < best[0] + best[1]:
            best = (c, f, s)
    c, f, s = best
    err = float(np.max(np.abs(v - want) / np.abs(want)))
    plan = _native.plan_info(K, prec)
    mode = _native.profile_phases()[0]
    row = dict(precision=prec, path={2: "stitched chain", 1: "rank-one collapse"}.get(
                   mode, "run-absorbing" if _native.profile_runs() else "record by record / tensor-core matrix"),
               loglik=float(v[0]), rel_err_vs_reference=err, bound=BOUNDS[prec],
               within_bound=err <= BOUNDS[prec], chain_ms=c, fold_ms=f, segments=s,
               obs_per_s=N * B / ((c + f) / 1e3),
               reference_equivalent_tflops=2 * K ** 3 * N * B / ((c + f) / 1e3) / 1e12, plan=plan)
    rows.append(row)
    print(f"{prec:8s} {row['path']:22s} logL={v[0]:.10f} rel_err={err:.3e} (bound {BOUNDS[prec]:.0e}: "
          f"{'ok' if row['within_bound'] else 'EXCEEDED'}) chain={c:.2f} ms fold={f:.3f} ms "
          f"-> {row['obs_per_s']:.3e} obs/s ({row['reference_equivalent_tflops']:.1f} TFLOP/s at 2K^3/obs)", flush=True)
_native.set_collapse_mode(1)
_native.set_stitch_mode(1)
if a.json:
    with open(a.json, "w") as fh:
        json.dump({"workload": a.workload, "K": K, "N": N, "B": B, "golden": float(want[0]), "rows": rows}, fh, indent=1)
