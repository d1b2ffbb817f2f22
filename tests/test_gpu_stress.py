"""Randomised parity sweep over the engine's code paths -- needs a B200.

Random K (1..80), chain length (1..30000), batch size, explicit or automatic
segment count, renormalisation period, and entry point (device-resident
batch with graph replay, host-array pipeline, host-array batch, range nodes
+ strided fold with a random range split, and the 32-bit / tensor-core
modes), each against the C oracle at the mode's bound (FP64: 1e-9).
Every case runs with the engine's own kernel choice and again with the
run-absorbing chain forced.  Seeded: failures reproduce.
"""

import numpy as np
import pytest

import fixtures as fx
from oracle import coracle

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


@pytest.mark.parametrize("runs_mode", [-1, 1])
@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("THMM_STRESS_SEEDS", "12"))))
def test_random_paths(eng, seed, runs_mode):
    """runs_mode -1: the engine's own choice of chain kernel; 1: the
    run-absorbing chain forced for every FP64 evaluation.  Host-array cases
    use pinned arrays half of the time (the zero-copy entry)."""
    from paper_2003_03508_b200 import _native

    _native.set_runs_mode(runs_mode)
    try:
        _random_paths(eng, seed + (0 if runs_mode < 0 else 5000))
    finally:
        _native.set_runs_mode(-1)


def _random_paths(eng, seed):
    import torch

    from paper_2003_03508_b200 import _native

    rng = np.random.default_rng(9000 + seed)
    for case in range(12):
        k = int(rng.integers(1, 81))
        n = int(np.exp(rng.uniform(0, np.log(30000))))
        b = int(rng.integers(1, 5))
        plist = [fx.random_params(rng, k) for _ in range(b)]
        pr, lo, la = fx.random_obs_arrays(rng, n, present_prob=float(rng.uniform(0.1, 0.9)))
        segs = None if rng.random() < 0.5 else int(rng.integers(1, min(n, 5000) + 1))
        period = int(rng.choice([1, 3, 8, 17]))
        path = case % 5
        prec = "float64" if path < 4 else str(rng.choice(["float32", "tf32x2", "tf32x3"]))
        cfg = eng.EngineConfig(segments=segs, renorm_period=period, precision=prec)
        want = np.array([coracle.forward_loglik(p, pr, lo, la) for p in plist])
        if path == 0:
            dev = eng.DeviceObservations(pr, lo, la)
            got = dev.loglik_batch(plist, cfg)
            got2 = dev.loglik_batch(plist, cfg)  # graph replay
            assert np.array_equal(got, got2)
        elif path == 1:
            arrs = (pr, lo, la)
            if rng.random() < 0.5:  # pinned: the zero-copy entry
                pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (pr.view(np.uint8), lo, la)]
                arrs = (pin[0].numpy().view(np.bool_), pin[1].numpy(), pin[2].numpy())
            got = np.array([eng._parallel_loglik_arrays(p, *arrs, cfg) for p in plist])
        elif path == 2:
            got = eng.parallel_loglik_batch(plist, (pr, lo, la), cfg)
        elif path == 4:
            got = eng.DeviceObservations(pr, lo, la).loglik_batch(plist, cfg)
        else:
            dev = eng.DeviceObservations(pr, lo, la)
            g = int(rng.integers(1, min(n, 9) + 1))
            kp = eng.padded_states(k)
            blk = b * kp * kp + b + ((b * kp * kp + b) & 1)
            buf = torch.zeros(g * blk, dtype=torch.float64, device="cuda")
            for i, (a, e) in enumerate(eng.segment_bounds(n, g)):
                base = buf.data_ptr() + 8 * i * blk
                dev.range_nodes(plist, cfg, a, e, base, base + 8 * b * kp * kp)
            got = eng.fold_nodes(plist, buf.data_ptr(), buf.data_ptr() + 8 * b * kp * kp, g, device=0,
                                 m_stride_g=blk, e_stride_g=blk)
        rel = np.abs(got - want) / np.abs(want)
        bound = {"float64": TOL, "float32": 1e-4, "tf32x2": 1e-4, "tf32x3": 1e-6}[prec]
        if prec == "tf32x2" and n < 1000:
            # tf32x2 rounds the rows to tf32 every step (relative error up to
            # 2^-11, random): on chains this short the log-likelihood error
            # does not average out (seed 137: K=1, N=34 gives 1.1e-4)
            bound = 5e-4
        assert rel.max() <= bound, (seed, case, path, prec, k, n, b, segs, period, rel.max(), _native.profile_runs())
