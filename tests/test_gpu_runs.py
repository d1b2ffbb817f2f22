"""Run-absorbing FP64 chain (csrc/thmm_runs.cuh) -- needs a B200.

A run of r absent records multiplies the chain by (Gamma diag(1-p))^r; the
kernel applies precomputed powers instead of r record steps.  Same product,
different association over absent runs, so the parity bar is the FP64 one
(1e-9 relative, stated in the north star; observed ~1e-14).  Every test
forces the mode on (thmm_set_runs_mode(1)) except the automatic-decision
test, and compares with the C oracle or the reference golden.
"""

import numpy as np
import pytest

import fixtures as fx
from golden_io import load, rel
from oracle import coracle

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    _native.set_runs_mode(1)
    yield eng
    _native.set_runs_mode(-1)


def _obs(rng, n, present_prob):
    pr = rng.random(n) < present_prob
    lo = np.where(pr, rng.uniform(-1.5, 1.5, n), 0.0)
    la = np.where(pr, rng.uniform(-1.5, 1.5, n), 0.0)
    return pr, lo, la


# every tail width (K % 8 = 1..4 above 8: tail = 1..4 SIMT states) at every
# head width, incl. K = 26/27 (one-CTA shape, R = 16) and 34/35 (R = 16 with
# two groups), plus the padded residues 5..7
@pytest.mark.parametrize("k", [1, 2, 3, 5, 7, 8, 9, 10, 11, 12, 16, 17, 18, 19, 20, 24, 25, 26, 27, 28, 29, 31, 32,
                               33, 34, 35, 36, 40, 41, 44, 48, 49, 50, 56, 57, 60, 64, 65, 72, 73, 76, 80])
def test_every_variant_against_oracle(eng, k):
    """All (head tiles, skip, tail) instantiations and every chunk limit
    (R = 16, 8, 4, 3 by K), over presence fractions from all-absent to
    all-present."""
    from paper_2003_03508_b200 import _native

    rng = np.random.default_rng(700 + k)
    p = fx.random_params(rng, k)
    for prob in (0.0, 0.05, 0.13, 0.5, 1.0):
        pr, lo, la = _obs(rng, 2003, prob)
        want = coracle.forward_loglik(p, pr, lo, la)
        dev = eng.DeviceObservations(pr, lo, la)
        for segs in (None, 1, 7):
            got = dev.loglik(p, eng.EngineConfig(segments=segs))
            assert _native.profile_runs()
            assert rel(got, want) <= TOL, (k, prob, segs, got, want)
        dev.close()


def test_window_edges_and_tiny_chains(eng):
    """Chains of 1..70 records (window edges at 32, 64), runs crossing windows
    and segment boundaries, one-record segments."""
    rng = np.random.default_rng(11)
    for k in (4, 25):
        p = fx.random_params(rng, k)
        for n in (1, 2, 3, 15, 16, 17, 31, 32, 33, 47, 63, 64, 65, 70):
            for prob in (0.0, 0.1, 0.9):
                pr, lo, la = _obs(rng, n, prob)
                want = coracle.forward_loglik(p, pr, lo, la)
                for segs in (None, 1, n):
                    got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=segs))
                    assert rel(got, want) <= TOL, (k, n, prob, segs)


def test_long_runs_and_renormalisation(eng):
    """Long absent stretches (hundreds of chunks of R) with extreme p: the
    table powers carry their own exponents, nothing underflows."""
    rng = np.random.default_rng(5)
    for k in (6, 25):
        p = fx.random_params(rng, k, p_range=(0.9, 0.999))  # q down to 1e-3: (Gamma Q)^16 ~ 1e-48
        n = 20000
        pr = np.zeros(n, dtype=bool)
        pr[rng.choice(n, 40, replace=False)] = True
        lo = np.where(pr, rng.uniform(-1, 1, n), 0.0)
        la = np.where(pr, rng.uniform(-1, 1, n), 0.0)
        want = coracle.forward_loglik(p, pr, lo, la)
        for period in (1, 8, 64):
            got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(renorm_period=period))
            assert rel(got, want) <= TOL, (k, period, got, want)


def test_batch_range_fold_and_host_pipeline(eng):
    """Batched proposals, range nodes + strided fold (the multi-GPU combine)
    and the chunked host-array pipeline all on the run-absorbing chain."""
    import torch

    rng = np.random.default_rng(23)
    k = 25
    plist = [fx.random_params(rng, k) for _ in range(5)]
    pr, lo, la = _obs(rng, 150_000, 0.13)
    want = np.array([coracle.forward_loglik(p, pr, lo, la) for p in plist])
    dev = eng.DeviceObservations(pr, lo, la)
    got = dev.loglik_batch(plist, eng.EngineConfig())
    assert np.max(np.abs(got - want) / np.abs(want)) <= TOL
    kp = eng.padded_states(k)
    G = 3
    m = torch.empty((G, len(plist), kp, kp), dtype=torch.float64, device="cuda")
    e = torch.empty((G, len(plist)), dtype=torch.float64, device="cuda")
    for g, (a, b) in enumerate(eng.segment_bounds(pr.size, G)):
        dev.range_nodes(plist, eng.EngineConfig(), a, b, m[g].data_ptr(), e[g].data_ptr())
    folded = np.asarray(eng.fold_nodes(plist, m.data_ptr(), e.data_ptr(), G, device=0))
    assert np.max(np.abs(folded - want) / np.abs(want)) <= TOL
    pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (pr.view(np.uint8), lo, la)]
    for _ in range(3):  # eager, capture, graph replay
        h = dev.loglik_host_batch(plist, pin[0].view(np.bool_), pin[1], pin[2], eng.EngineConfig())
        assert np.max(np.abs(h - want) / np.abs(want)) <= TOL
    dev.close()


def test_collapse_raises(eng):
    st = eng.StateEmission(0.5, np.array([0.0, 0.0]), np.eye(2) * 1e-6)
    p = eng.HmmParams(gamma=np.array([[1.0]]), delta=np.array([1.0]), states=(st,))
    pr = np.array([True] * 4)
    lo = np.array([1e3] * 4)
    la = np.zeros(4)
    with pytest.raises(RuntimeError):
        eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())


def test_full_size_k25_workload_against_golden(eng):
    """BASELINE configs[1] (K=25, N=10^6, 13% present) against the reference's logL."""
    from paper_2003_03508_b200 import synth

    gold = load("bench_configs.json")["workloads"]["k25_n1e6"]
    plist, pr, lo, la = synth.make_workload("k25_n1e6")
    dev = eng.DeviceObservations(pr, lo, la)
    got = dev.loglik_batch(plist, eng.EngineConfig())
    assert rel(got[0], gold["loglik"][0]) <= TOL
    assert rel(got[0], gold["loglik"][0]) <= 1e-12  # observed ~1e-15


def test_automatic_decision(eng):
    """The cost model picks the run-absorbing chain for sparse event streams
    and the record-by-record kernel for dense ones; results agree either way."""
    from paper_2003_03508_b200 import _native, synth

    _native.set_runs_mode(-1)
    try:
        plist, pr, lo, la = synth.make_workload("k25_n1e6", n=200_000)  # ~13% present
        dev = eng.DeviceObservations(pr, lo, la)
        info = dev.runs_info(25)
        assert info["active"] and 0.2 < info["steps_per_record"] < 0.45, info
        a = dev.loglik(plist[0], eng.EngineConfig())
        assert _native.profile_runs()
        _native.set_runs_mode(0)
        b = dev.loglik(plist[0], eng.EngineConfig())
        assert not _native.profile_runs()
        assert rel(a, b) <= 1e-12
        _native.set_runs_mode(-1)
        rng = np.random.default_rng(3)
        pr2, lo2, la2 = _obs(rng, 100_000, 0.6)
        dev2 = eng.DeviceObservations(pr2, lo2, la2)
        assert not dev2.runs_info(25)["active"]
        info80 = dev.runs_info(80)  # R = 3; 2e5 records are below the wide-row minimum (2.6e5)
        assert info80["R"] == 3 and not info80["active"], info80
        assert not dev.runs_info(25, "float32")["active"]  # FP64 only
    finally:
        _native.set_runs_mode(1)
