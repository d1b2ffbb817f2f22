"""Zero-copy host-array entry (thmm_loglik_mapped) -- needs a B200.

Pinned host arrays are read in place by the chain kernels over PCIe
(uncached loads, coordinates only for present records).  Same kernels, same
arithmetic as the device-resident path, so results must be bitwise equal to
it; against the C oracle at the FP64 bar (1e-9, stated in the north star).
"""

import numpy as np
import pytest

import fixtures as fx
from golden_io import load, rel
from oracle import coracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


def _pinned(pr, lo, la):
    import torch

    out = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (pr.view(np.uint8), lo, la)]
    return out, (out[0].numpy().view(np.bool_), out[1].numpy(), out[2].numpy())


@pytest.mark.parametrize("runs_mode", [0, 1])
@pytest.mark.parametrize("precision", ["float64", "float32", "tf32x3"])
def test_mapped_equals_device_resident(eng, precision, runs_mode):
    from paper_2003_03508_b200 import _native

    _native.set_runs_mode(runs_mode)
    try:
        rng = np.random.default_rng(41)
        for k in (5, 25, 50):
            plist = [fx.random_params(rng, k) for _ in range(3)]
            pr, lo, la = fx.random_obs_arrays(rng, 30011, present_prob=0.2)
            keep, (ppr, plo, pla) = _pinned(pr, lo, la)
            dev = eng.DeviceObservations(pr, lo, la)
            cfg = eng.EngineConfig(precision=precision)
            want = dev.loglik_batch(plist, cfg)
            scratch = eng.DeviceObservations(pr[:10], lo[:10], la[:10])
            for _ in range(3):  # eager, capture, graph replay
                got = scratch.loglik_host_batch(plist, ppr, plo, pla, cfg, mapped=True)
                assert np.array_equal(got, want), (k, precision, runs_mode, got, want)
            assert len(scratch) == 10  # the handle's own records are untouched
            if precision == "float64":
                o = np.array([coracle.forward_loglik(p, pr, lo, la) for p in plist])
                assert np.max(np.abs(got - o) / np.abs(o)) <= 1e-9
            dev.close()
            scratch.close()
            del keep
    finally:
        _native.set_runs_mode(-1)


def test_mapped_subrange_and_segments(eng):
    rng = np.random.default_rng(8)
    p = fx.random_params(rng, 25)
    pr, lo, la = fx.random_obs_arrays(rng, 5000, present_prob=0.15)
    keep, (ppr, plo, pla) = _pinned(pr, lo, la)
    scratch = eng.DeviceObservations(pr[:5], lo[:5], la[:5])
    for segs in (None, 1, 13):
        got = scratch.loglik_host_batch([p], ppr, plo, pla, eng.EngineConfig(segments=segs), mapped=True)[0]
        want = coracle.forward_loglik(p, pr, lo, la)
        assert rel(got, want) <= 1e-9, segs
    scratch.close()
    del keep


def test_pageable_arrays_fall_back_to_the_copy_pipeline(eng):
    rng = np.random.default_rng(9)
    p = fx.random_params(rng, 12)
    pr, lo, la = fx.random_obs_arrays(rng, 3000)
    scratch = eng.DeviceObservations(pr[:5], lo[:5], la[:5])
    got = scratch.loglik_host_batch([p], pr, lo, la, eng.EngineConfig(), mapped=True)[0]
    assert rel(got, coracle.forward_loglik(p, pr, lo, la)) <= 1e-9
    assert len(scratch) == 3000  # the copy pipeline replaced the handle's records
    scratch.close()


def test_reference_api_with_pinned_arrays_k25_workload(eng):
    """_parallel_loglik_arrays (the reference's own entry point) on the K=25
    N=10^6 workload in pinned memory: the zero-copy route, against the golden."""
    from paper_2003_03508_b200 import synth

    gold = load("bench_configs.json")["workloads"]["k25_n1e6"]
    plist, pr, lo, la = synth.make_workload("k25_n1e6")
    keep, (ppr, plo, pla) = _pinned(pr, lo, la)
    for _ in range(3):
        got = eng._parallel_loglik_arrays(plist[0], ppr, plo, pla, eng.EngineConfig())
        assert rel(got, gold["loglik"][0]) <= 1e-12
    del keep


def test_pageable_arrays_pinned_on_first_use(eng):
    """The reference API with pageable arrays: the second call page-locks them
    in place (thmm_host_register) and reads them zero-copy -- bitwise equal to
    the device-resident value; releasing the arrays unregisters the range."""
    import gc

    from paper_2003_03508_b200 import engine as e

    rng = np.random.default_rng(77)
    p = fx.random_params(rng, 25)
    pr, lo, la = fx.random_obs_arrays(rng, 200_003, present_prob=0.15)
    dev = eng.DeviceObservations(pr, lo, la)
    want = dev.loglik(p, eng.EngineConfig())
    dev.close()
    lo2, la2 = lo.copy(), la.copy()  # fresh pageable buffers (1.6 MB each)
    keys = [(int(a.ctypes.data), int(a.nbytes)) for a in (lo2, la2)]
    vals = [eng._parallel_loglik_arrays(p, pr, lo2, la2, eng.EngineConfig()) for _ in range(4)]
    assert all(v == want for v in vals), (vals, want)
    assert all(e._pinned_ranges.get(k, (False,))[0] for k in keys)
    del lo2, la2
    gc.collect()
    assert not any(k in e._pinned_ranges for k in keys)
    o = coracle.forward_loglik(p, pr, lo, la)
    assert abs(want - o) <= 1e-9 * abs(o)


@pytest.mark.parametrize("k", [9, 25, 50, 80])
def test_staged_stitched_equals_device_resident(eng, k):
    """Host-array evaluations on the stitched chain stage the records into HBM
    by DMA in time chunks (each chunk of the main pass continues the rows the
    previous one left): bitwise equal to the one-launch device-resident pass,
    eager and as a replayed graph, and within 1e-9 of the C oracle."""
    from paper_2003_03508_b200 import _native

    rng = np.random.default_rng(500 + k)
    plist = [fx.random_params(rng, k)]
    n = 600_007 if k <= 25 else 300_007
    pr, lo, la = fx.random_obs_arrays(rng, n, present_prob=0.3)
    keep, (ppr, plo, pla) = _pinned(pr, lo, la)
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    _native.set_collapse_params(0.0, 192, -1.0)  # stitched chain regardless of the cost model
    try:
        want = dev.loglik_batch(plist, cfg)
        scratch = eng.DeviceObservations(pr[:10], lo[:10], la[:10])
        for _ in range(3):  # eager, capture, graph replay
            got = scratch.loglik_host_batch(plist, ppr, plo, pla, cfg, mapped=True)
            assert np.array_equal(got, want), (k, got, want)
        o = coracle.forward_loglik(plist[0], pr, lo, la)
        assert abs(got[0] - o) <= 1e-9 * abs(o)
        scratch.close()
    finally:
        _native.set_collapse_params(0.0, 1024, 0.25)
        dev.close()
        del keep


def test_staged_multi_launch_fallback_matches():
    """THMM_STAGE_SINGLE=0 (no stream-memory-operation signals: one main-pass
    launch per time chunk) gives the same bits as the single launch and the
    device-resident pass (subprocess: the switch is read once per process)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import fixtures as fx, paper_2003_03508_b200 as eng\n"
        "from paper_2003_03508_b200 import _native\n"
        "rng = np.random.default_rng(77); p = fx.random_params(rng, 41)\n"
        "pr, lo, la = fx.random_obs_arrays(rng, 400_003, present_prob=0.3)\n"
        "_native.set_collapse_params(0.0, 192, -1.0)\n"
        "pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (pr.view(np.uint8), lo, la)]\n"
        "want = eng.DeviceObservations(pr, lo, la).loglik(p, eng.EngineConfig())\n"
        "s = eng.DeviceObservations(pr[:10], lo[:10], la[:10])\n"
        "got = [s.loglik_host_batch([p], pin[0].view(np.bool_), pin[1], pin[2], eng.EngineConfig(), mapped=True)[0]"
        " for _ in range(3)]\n"
        "print(repr(float(want)), repr(float(got[0])), repr(float(got[2])))\n"
    ) % (root, os.path.join(root, "tests"))
    vals = []
    for single in ("1", "0"):
        env = dict(os.environ, THMM_STAGE_SINGLE=single, THMM_STITCH_HOST="1")
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        want, g0, g2 = (float(x) for x in out.stdout.split())
        assert g0 == want and g2 == want, (single, want, g0, g2)
        vals.append(want)
    assert vals[0] == vals[1]
