"""Small evaluations touching every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py --quick
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py --quick
    compute-sanitizer --tool initcheck python tools/sanitize_cases.py --quick

Families: chain_f64 (plain / skip / tailed / lean plans), the stitched chain
(chain_fwd / chain_link / stitch_finish) and the rank-one collapse
(chain_runs burn-in test / chain_vec), chain_runs (with
THMM_RUNS=1: every K), the zero-copy host entry, chain_f32,
chain_tc (tf32, tf32x2, tf32x3; H=1 and H=2), the one-launch tree, the
host-array chunk pipeline, range nodes + strided fold, the filtered
next-state pass, the emission table, stationary distributions.  Results are
checked against the C oracle so a sanitizer-perturbed run still has to be
right.  Graphs are disabled (THMM_GRAPHS=0) unless --graphs: the sanitizer
tracks graph launches too, but eager launches give clearer reports.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true", help="fewer K values (racecheck is ~100x slower)")
ap.add_argument("--graphs", action="store_true")
a = ap.parse_args()
if not a.graphs:
    os.environ["THMM_GRAPHS"] = "0"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures as fx  # noqa: E402
import paper_2003_03508_b200 as eng  # noqa: E402
from oracle import coracle  # noqa: E402
from paper_2003_03508_b200 import proposals  # noqa: E402

BOUND = {"float64": 1e-9, "float32": 1e-4, "tf32x3": 1e-6, "tf32x2": 1e-4, "tf32": 2e-3}
ks = (1, 5, 9, 25, 32, 50, 80) if a.quick else (1, 2, 5, 8, 9, 10, 11, 12, 17, 18, 19, 25, 26, 27, 28, 32, 33, 34, 35, 42, 50, 57, 64, 73, 80)
precs = ("float64", "float32", "tf32x3", "tf32x2", "tf32")
rng = np.random.default_rng(2024)
n = 600
worst = {p: 0.0 for p in precs}
for k in ks:
    p = fx.random_params(rng, k)
    pr, lo, la = fx.random_obs_arrays(rng, n)
    want = coracle.forward_loglik(p, pr, lo, la)
    dev = eng.DeviceObservations(pr, lo, la)
    for prec in precs:
        for segs in (None, 7):
            got = dev.loglik(p, eng.EngineConfig(segments=segs, precision=prec))
            worst[prec] = max(worst[prec], abs(got - want) / abs(want))
    # host-array pipeline (chunked H2D) on a pinned copy
    pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (pr.view(np.uint8), lo, la)]
    got = dev.loglik_host_batch([p], pin[0].view(np.bool_), pin[1], pin[2], eng.EngineConfig())[0]
    worst["float64"] = max(worst["float64"], abs(got - want) / abs(want))
    # zero-copy: the kernels read the pinned arrays in place
    got = dev.loglik_host_batch([p], pin[0].view(np.bool_), pin[1], pin[2], eng.EngineConfig(), mapped=True)[0]
    worst["float64"] = max(worst["float64"], abs(got - want) / abs(want))
    dev.close()
    print(f"K={k} ok", flush=True)
print("worst rel error:", {q: f"{v:.1e}" for q, v in worst.items()})
for q, v in worst.items():
    assert v <= BOUND[q], (q, v)

# batch + range nodes + strided fold
k = 25
plist = [fx.random_params(rng, k) for _ in range(3)]
pr, lo, la = fx.random_obs_arrays(rng, 3000)
dev = eng.DeviceObservations(pr, lo, la)
whole = dev.loglik_batch(plist, eng.EngineConfig())
kp = eng.padded_states(k)
G = 3
m = torch.empty((G, len(plist), kp, kp), dtype=torch.float64, device="cuda")
e = torch.empty((G, len(plist)), dtype=torch.float64, device="cuda")
for g, (x, y) in enumerate(eng.segment_bounds(pr.size, G)):
    dev.range_nodes(plist, eng.EngineConfig(), x, y, m[g].data_ptr(), e[g].data_ptr())
folded = eng.fold_nodes(plist, m.data_ptr(), e.data_ptr(), G, device=0)
assert np.max(np.abs(np.asarray(folded) - whole) / np.abs(whole)) <= 1e-9
# filtered next-state pass, emission table, stationary distributions
nxt = dev.filtered_next_state(plist, eng.EngineConfig())
assert np.allclose(np.asarray(nxt).sum(axis=-1), 1.0)
em = dev.emissions(plist[0], 0, 100)
assert em.shape == (100, k) and np.all(np.isfinite(em))
gam = np.stack([np.asarray(q.gamma) for q in plist])
st = proposals.stationary_distribution_batch(gam)
assert np.allclose(np.einsum("bi,bij->bj", st, gam), st, atol=1e-9)
dev.close()

# forgetting-based paths (thmm_vec.cuh): stitched chain (main pass, links,
# finish), its fallback, and the rank-one collapse (burn-in test + vector
# continuation), all forced onto short chains; a stitched shard + link
from paper_2003_03508_b200 import _native  # noqa: E402

_native.set_collapse_params(0.0, 256, -1.0)
for k in ((5, 25, 50) if a.quick else (3, 9, 17, 25, 33, 50, 57, 80)):
    plist = [fx.random_params(rng, k) for _ in range(2)]
    pr, lo, la = fx.random_obs_arrays(rng, 4099, present_prob=0.3)
    dev = eng.DeviceObservations(pr, lo, la)
    for stitch in (1, 0):
        _native.set_stitch_mode(stitch)
        got = dev.loglik_batch(plist, eng.EngineConfig())
        for p_, g_ in zip(plist, got):
            w_ = coracle.forward_loglik(p_, pr, lo, la)
            assert abs(g_ - w_) <= 1e-9 * abs(w_), (k, stitch, g_, w_)
    _native.set_stitch_mode(1)
    kp = eng.padded_states(k)
    blk = torch.empty(2 * (kp + 2), dtype=torch.float64, device="cuda")
    lnk = torch.empty(4, dtype=torch.float64, device="cuda")
    from paper_2003_03508_b200.engine import _native_config, _PackedParams  # noqa: E402

    pp = _PackedParams(plist)
    c = _native_config(eng.EngineConfig(), 0, 0, 0)
    err = _native.errbuf()
    assert _native.lib().thmm_stitch_shard(dev._handle, _native.ctypes.byref(pp.struct), _native.ctypes.byref(c), 1,
                                            blk.data_ptr(), err, len(err)) == 0, err.value
    assert _native.lib().thmm_stitch_link(dev._handle, _native.ctypes.byref(pp.struct), _native.ctypes.byref(c),
                                           _native.c_void_p(blk.data_ptr()), kp + 2, lnk.data_ptr(), err,
                                           len(err)) == 0, err.value
    torch.cuda.synchronize()
    dev.close()
    print(f"stitch/collapse K={k} ok", flush=True)
_native.set_collapse_params(0.0, 1024, 0.25)
print("SANITIZE CASES PASSED")

# host arrays on the stitched chain staged by DMA in time chunks: one launch
# that waits per record window for stream-memory-operation signals (or one
# launch per chunk), and a rank's host shard (thmm_stitch_shard_host)
_native.set_collapse_params(0.0, 256, -1.0)  # the stitched chain regardless of the cost model
for k in (9, 33):
    p = fx.random_params(rng, k)
    pr, lo, la = fx.random_obs_arrays(rng, 300_007, present_prob=0.3)
    want = coracle.forward_loglik(p, pr, lo, la)
    pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (pr.view(np.uint8), lo, la)]
    scratch = eng.DeviceObservations(pr[:10], lo[:10], la[:10])
    got = scratch.loglik_host_batch([p], pin[0].view(np.bool_), pin[1], pin[2], eng.EngineConfig(), mapped=True)[0]
    assert abs(got - want) <= 1e-9 * abs(want), (k, got, want)
    kp = eng.padded_states(k)
    blk = torch.empty(kp + 2, dtype=torch.float64, device="cuda")
    pp = _PackedParams([p])
    c = _native_config(eng.EngineConfig(), 0, 0, 0)
    err = _native.errbuf()
    assert _native.lib().thmm_stitch_shard_host(scratch._handle, pin[0].ctypes.data, pin[1].ctypes.data,
                                                pin[2].ctypes.data, pr.size, _native.ctypes.byref(pp.struct),
                                                _native.ctypes.byref(c), 1, blk.data_ptr(), err, len(err)) == 0, err.value
    torch.cuda.synchronize()
    scratch.close()
    print(f"staged host stitched K={k} ok", flush=True)
_native.set_collapse_params(0.0, 1024, 0.25)
print("SANITIZE CASES PASSED (staged)")
