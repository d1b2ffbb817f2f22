"""Precision-study modes on the tcgen05 tensor cores -- needs a B200.

BASELINE.json configs[3] asks for an FP64 vs FP32/TF32 tensor-core tolerance
study.  The FP64 DMMA path is the parity path (1e-9); the study modes keep
the reference's float32 semantics (engine.py:331-333) with the chain products
on tcgen05.mma kind::tf32:

    precision="tf32x3"  hi+lo split operands, 3 MMAs per product
                        stated bound: 1e-6 relative to FP64 (observed <= 4e-7)
    precision="tf32x2"  Gamma split hi+lo, rows rounded to tf32 (2 MMAs)
                        stated bound: 1e-4 relative
    precision="tf32"    plain TF32 operands (10-bit mantissa)
                        stated bound: 2e-3 relative (observed <= 6e-4)

tf32x3 also meets the reference's own 32-bit tolerance (1e-4, SPEC.md:193,
test_engine.py:188-195); plain tf32 does not at small K, which is why it is a
study mode and never the default.
"""

import numpy as np
import pytest

import fixtures as fx
from golden_io import load, regen_cases, rel
from oracle import coracle

pytestmark = pytest.mark.gpu

BOUND = {"tf32x3": 1e-6, "tf32x2": 1e-4, "tf32": 2e-3}


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


@pytest.mark.parametrize("prec", ["tf32x3", "tf32x2", "tf32"])
def test_all_k_against_serial(eng, prec):
    worst = 0.0
    for c, p, pr, lo, la in regen_cases("matches_serial"):
        for segs in (None, 4):
            got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=segs, precision=prec))
            worst = max(worst, rel(got, c["serial"]))
    assert worst <= BOUND[prec], worst
    if prec == "tf32x3":
        assert worst <= 1e-4  # the reference's float32 tolerance


@pytest.mark.parametrize("k", [1, 2, 5, 8, 9, 16, 17, 24, 25, 31, 32, 33, 40, 47, 48, 49, 56, 57, 63, 64, 65, 72, 79, 80])
def test_every_tile_shape(eng, k):
    """Every (UMMA N, contraction) instantiation, against the C oracle."""
    rng = np.random.default_rng(500 + k)
    p = fx.random_params(rng, k)
    pr, lo, la = fx.random_obs_arrays(rng, 3001)
    want = coracle.forward_loglik(p, pr, lo, la)
    for prec in ("tf32x3", "tf32x2", "tf32"):
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(precision=prec))
        assert rel(got, want) <= BOUND[prec], (k, prec, got, want)


def test_ragged_segments(eng):
    """Segment lengths differing by one inside a CTA (end-aligned idle step),
    one-record segments, and a single segment."""
    rng = np.random.default_rng(77)
    for k in (5, 25, 50, 80):
        p = fx.random_params(rng, k)
        n = 997
        pr, lo, la = fx.random_obs_arrays(rng, n)
        want = coracle.forward_loglik(p, pr, lo, la)
        for segs in (1, 2, 3, 7, 100, 333, n - 1, n):
            got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=segs, precision="tf32x3"))
            assert rel(got, want) <= BOUND["tf32x3"], (k, segs)


def test_single_record_and_tiny_chains(eng):
    rng = np.random.default_rng(3)
    for k in (1, 7, 25, 80):
        p = fx.random_params(rng, k)
        for n in (1, 2, 3, 17):
            pr, lo, la = fx.random_obs_arrays(rng, n)
            want = coracle.forward_loglik(p, pr, lo, la)
            got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(precision="tf32x3"))
            assert rel(got, want) <= BOUND["tf32x3"], (k, n)


def test_batch_and_determinism(eng):
    rng = np.random.default_rng(8)
    plist = [fx.random_params(rng, 33) for _ in range(6)]
    pr, lo, la = fx.random_obs_arrays(rng, 20000)
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig(precision="tf32x3")
    a = dev.loglik_batch(plist, cfg)
    b = dev.loglik_batch(plist, cfg)
    assert np.array_equal(a, b)  # run-to-run bitwise
    f64 = dev.loglik_batch(plist, eng.EngineConfig())
    assert np.max(np.abs(a - f64) / np.abs(f64)) <= BOUND["tf32x3"]


def test_range_nodes_fold(eng):
    """Shard math (multi-GPU combine) in the study mode: ranges -> nodes -> fold."""
    import torch

    rng = np.random.default_rng(21)
    plist = [fx.random_params(rng, 50) for _ in range(2)]
    pr, lo, la = fx.random_obs_arrays(rng, 6000)
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig(precision="tf32x3")
    whole = dev.loglik_batch(plist, eng.EngineConfig())
    kp = eng.padded_states(50)
    G = 3
    m = torch.empty((G, len(plist), kp, kp), dtype=torch.float64, device="cuda")
    e = torch.empty((G, len(plist)), dtype=torch.float64, device="cuda")
    for g, (a, b) in enumerate(eng.segment_bounds(pr.size, G)):
        dev.range_nodes(plist, cfg, a, b, m[g].data_ptr(), e[g].data_ptr())
    got = eng.fold_nodes(plist, m.data_ptr(), e.data_ptr(), G, device=0)
    for x, y in zip(got, whole):
        assert rel(x, y) <= BOUND["tf32x3"]


def test_collapse_raises(eng):
    st = eng.StateEmission(0.5, np.array([0.0, 0.0]), np.eye(2) * 1e-6)
    p = eng.HmmParams(gamma=np.array([[1.0]]), delta=np.array([1.0]), states=(st,))
    pr = np.array([True] * 4)
    lo = np.array([1e3] * 4)
    la = np.zeros(4)
    with pytest.raises(RuntimeError):
        eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(precision="tf32x3"))


def test_full_size_workload_k25(eng):
    """BASELINE.json configs[1] at full size against the reference golden."""
    from paper_2003_03508_b200 import synth

    gold = load("bench_configs.json")["workloads"]["k25_n1e6"]
    plist, pr, lo, la = synth.make_workload("k25_n1e6")
    dev = eng.DeviceObservations(pr, lo, la)
    for prec in ("tf32x3", "tf32"):
        got = dev.loglik_batch(plist, eng.EngineConfig(precision=prec))
        assert rel(got[0], gold["loglik"][0]) <= BOUND[prec], prec
