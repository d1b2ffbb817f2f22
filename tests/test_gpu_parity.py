"""CUDA path vs the reference goldens and the oracle -- needs a B200.

Every call goes through the C-ABI (libthmm.so) via the drop-in engine API.
Tolerance: the north-star bound of 1e-9 relative in FP64 is asserted
everywhere; the tighter figure each test also checks is what FP64 tensor-core
arithmetic actually delivers (rounding-level, ~1e-13).
"""

import math

import numpy as np
import pytest

import fixtures as fx
from golden_io import load, regen_cases, rel
from oracle import coracle

pytestmark = pytest.mark.gpu

TOL = 1e-9      # north_star tolerance (BASELINE.json)
TIGHT = 1e-11   # observed FP64 DMMA agreement, kept as a regression guard


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


def test_native_library_is_loaded(eng):
    from paper_2003_03508_b200 import _native

    assert _native.lib().thmm_device_count() >= 1
    assert _native.lib().thmm_version() >= 100


def test_matches_serial_all_k(eng):
    worst = 0.0
    for c, p, pr, lo, la in regen_cases("matches_serial"):
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=4))
        r = rel(got, c["serial"])
        assert r <= TOL, (c["k"], got, c["serial"])
        worst = max(worst, r, rel(got, c["parallel_s4"]))
        auto = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())
        worst = max(worst, rel(auto, c["serial"]))
    assert worst < TIGHT, worst


def test_segment_count_invariance(eng):
    (c, p, pr, lo, la), = regen_cases("segment_invariance")
    vals = [eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=int(s)))
            for s in (1, 2, 3, 7, 16, 100, 300)]
    for v in vals:
        assert rel(v, c["parallel"]["1"]) < 1e-12


def test_single_segment_tracks_serial_schedule(eng):
    (c, p, pr, lo, la), = regen_cases("schedule")
    for r, want in c["serial"].items():
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=1, renorm_period=int(r)))
        assert rel(got, want) <= 1e-11


def test_worker_count_does_not_change_value(eng):
    (c, p, pr, lo, la), = regen_cases("workers")
    one = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(workers=1, segments=4))
    four = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(workers=4, segments=4))
    assert one == four
    assert rel(one, c["value"]) < TIGHT


def test_deterministic_run_to_run(eng):
    (c, p, pr, lo, la), = regen_cases("long_k25")
    cfg = eng.EngineConfig()
    vals = {eng._parallel_loglik_arrays(p, pr, lo, la, cfg) for _ in range(5)}
    assert len(vals) == 1
    assert rel(vals.pop(), c["serial"]) < TIGHT


def test_single_observation_and_brute_force(eng):
    for c, p, pr, lo, la in regen_cases("brute") + regen_cases("single_obs"):
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())
        want = c.get("brute", c["serial"])
        assert rel(got, want) < 1e-12


def test_object_api_and_reference_types(eng):
    (c, p, pr, lo, la), = regen_cases("renorm_k5")
    obs = [eng.Observation((x, y)) if f else eng.Observation(None) for f, x, y in zip(pr, lo, la)]
    got = eng.parallel_loglik(p, obs, eng.EngineConfig(segments=3))
    assert rel(got, c["serial"]["1"]) < TIGHT


def test_emission_table(eng):
    (c, p, pr, lo, la), = regen_cases("emissions")
    obs = [eng.Observation((x, y)) if f else eng.Observation(None) for f, x, y in zip(pr, lo, la)]
    got = eng.batch_emissions(p, obs)
    want = np.array(c["table"])
    assert got.shape == want.shape
    # only exp() may differ (CUDA vs numpy), by an ulp or two
    np.testing.assert_allclose(got, want, rtol=5e-16 * 4, atol=0)
    assert np.array_equal(got[~pr], want[~pr])


def test_factor_segment_products(eng):
    (c, p, pr, lo, la), = regen_cases("factor_segments")
    ed = np.array([np.asarray(p.gamma) * row for row in coracle.emissions(p, pr, lo, la)])
    parts = eng.segment_chain_product(ed, eng.EngineConfig(segments=3))
    assert [(q.lo, q.hi) for q in parts] == [(g["lo"], g["hi"]) for g in c["parts"]]
    for q, g in zip(parts, c["parts"]):
        assert q.product.m.max() == 1.0
        np.testing.assert_allclose(q.product.m * math.exp(q.product.log_scale),
                                   np.array(g["m"]) * math.exp(g["log_scale"]), rtol=1e-12)
    assert rel(eng.combine_segments(p.delta, parts), c["combined"]) < 1e-12


def test_criterion1_oracle_equivalence(eng):
    gold = load("criterion1.json")["instances"]
    worst = 0.0
    for g, (k, n, segs, p, pr, lo, la) in zip(gold, fx.criterion1_instances()):
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=segs))
        worst = max(worst, rel(got, g["serial"]))
        if g["brute"] is not None:
            worst = max(worst, rel(got, g["brute"]))
    assert worst < 1e-10, worst


def test_criterion2_segment_invariance(eng):
    from paper_2003_03508_b200 import synth

    g = load("criterion2.json")
    rng = np.random.default_rng(2)
    p = synth.sample_prior_params(25, rng)
    _, pr, lo, la = synth.simulate_arrays(p, 100_000, rng)
    vals = [eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=s))
            for s in (1, 2, 7, 28, None)]
    ref = g["parallel"]["1"]
    assert (max(vals) - min(vals)) / abs(ref) < 1e-10
    assert max(rel(v, ref) for v in vals) < 1e-10


def test_rejects_bad_input(eng):
    (c, p, pr, lo, la), = regen_cases("brute")[:1]
    with pytest.raises(ValueError):
        eng._parallel_loglik_arrays(p, pr[:0], lo[:0], la[:0], eng.EngineConfig())
    with pytest.raises(ValueError):
        eng.parallel_loglik(p, [], eng.EngineConfig())
    big = fx.random_params(np.random.default_rng(45), 81, sigma_scale=1.0)
    with pytest.raises(ValueError):
        eng._parallel_loglik_arrays(big, pr, lo, la, eng.EngineConfig())


def test_collapse_raises(eng):
    # A state-0-only chain whose emissions underflow to exactly zero.
    st = eng.StateEmission(0.5, np.array([0.0, 0.0]), np.eye(2) * 1e-6)
    p = eng.HmmParams(gamma=np.array([[1.0]]), delta=np.array([1.0]), states=(st,))
    pr = np.array([True] * 4)
    lo = np.array([1e3] * 4)
    la = np.zeros(4)
    with pytest.raises(RuntimeError):
        eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())
    out = eng.parallel_loglik_batch([p, p], (pr, lo, la), eng.EngineConfig())
    assert np.all(np.isneginf(out))


def test_batch_matches_single(eng):
    rng = np.random.default_rng(7)
    plist = [fx.random_params(rng, 17) for _ in range(9)]
    pr, lo, la = fx.random_obs_arrays(rng, 3000)
    dev = eng.DeviceObservations(pr, lo, la)
    batch = dev.loglik_batch(plist, eng.EngineConfig())
    for p, b in zip(plist, batch):
        s = coracle.forward_loglik(p, pr, lo, la)
        assert rel(b, s) < TIGHT
        assert rel(dev.loglik(p, eng.EngineConfig()), s) < TIGHT


def test_range_nodes_fold_equals_whole(eng):
    """Sharding property: split the chain in G ranges, reduce each to a node,
    fold in order -- same value as the whole chain (multi-GPU math on 1 GPU)."""
    import torch

    rng = np.random.default_rng(11)
    plist = [fx.random_params(rng, 25) for _ in range(3)]
    pr, lo, la = fx.random_obs_arrays(rng, 5000)
    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    whole = dev.loglik_batch(plist, cfg)
    kp = eng.padded_states(25)
    for G in (1, 2, 3, 8):
        m = torch.empty((G, len(plist), kp, kp), dtype=torch.float64, device="cuda")
        e = torch.empty((G, len(plist)), dtype=torch.float64, device="cuda")
        for g, (a, b) in enumerate(eng.segment_bounds(pr.size, G)):
            dev.range_nodes(plist, cfg, a, b, m[g].data_ptr(), e[g].data_ptr())
        got = eng.fold_nodes(plist, m.data_ptr(), e.data_ptr(), G, device=0)
        for x, y in zip(got, whole):
            assert rel(x, y) < 1e-12


@pytest.mark.slow
@pytest.mark.parametrize("name", ["k5_n1e4", "k25_n1e6", "k25_n1e6_b256", "k50_n1e7", "k80_n1e8"])
def test_bench_workloads_vs_reference(eng, name):
    from paper_2003_03508_b200 import synth

    gold = load("bench_configs.json")["workloads"].get(name)
    if gold is None:
        pytest.skip(f"golden for {name} not generated")
    plist, pr, lo, la = synth.make_workload(name)
    assert fx.digest(pr, lo, la) == gold["obs_digest"]
    dev = eng.DeviceObservations(pr, lo, la)
    got = dev.loglik_batch(plist, eng.EngineConfig())
    want = np.array(gold["loglik"])
    r = np.abs(got - want) / np.abs(want)
    assert r.max() <= TOL, r.max()
    # size-independent property at full size: an explicit different segment count agrees
    alt = dev.loglik_batch(plist[:2], eng.EngineConfig(segments=97))
    assert np.max(np.abs(alt - got[:2]) / np.abs(got[:2])) < 1e-11


def test_float32_close_to_float64(eng):
    """Reference test_engine.py:188-195: float32 within 1e-4 of float64 (the
    SPEC's 32-bit tolerance)."""
    (c, p, pr, lo, la), = regen_cases("float32")
    f64 = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=2))
    f32 = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(segments=2, precision="float32"))
    assert rel(f64, c["f64"]) < TIGHT
    assert abs(f32 - f64) <= 1e-4 * abs(f64)
    assert abs(f32 - c["f32"]) <= 1e-4 * abs(c["f32"])


def test_float32_all_k(eng):
    worst = 0.0
    for c, p, pr, lo, la in regen_cases("matches_serial"):
        got = eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig(precision="float32"))
        worst = max(worst, rel(got, c["serial"]))
    assert worst <= 1e-4, worst


def test_sharded_nccl_single_rank(eng):
    """ShardedLoglik over a real NCCL process group (world 1 on one B200):
    range nodes -> NCCL all-gather -> device fold, same value as one GPU."""
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2003_03508_b200.distributed import ShardedLoglik

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(12)
        plist = [fx.random_params(rng, 25) for _ in range(2)]
        pr, lo, la = fx.random_obs_arrays(rng, 4000)
        sh = ShardedLoglik(pr, lo, la, device=0)
        got = sh.loglik_batch(plist, eng.EngineConfig())
        want = eng.DeviceObservations(pr, lo, la).loglik_batch(plist, eng.EngineConfig())
        for x, y in zip(got, want):
            assert rel(x, y) < 1e-12
        assert rel(sh.loglik(plist[0]), coracle.forward_loglik(plist[0], pr, lo, la)) < TIGHT
        sh.close()
    finally:
        dist.destroy_process_group()


def test_filtered_next_state(eng):
    """Forecast conditioning (reference simforecast.py:97-118), batched."""
    for c, p, pr, lo, la in regen_cases("filtered"):
        dev = eng.DeviceObservations(pr, lo, la)
        got = dev.filtered_next_state([p, p], eng.EngineConfig())
        want = np.array(c["dist"])
        for row in got:
            np.testing.assert_allclose(row, want, rtol=1e-10, atol=1e-14)
            assert abs(row.sum() - 1.0) < 1e-12


def test_host_array_pipeline_matches_golden(eng):
    """_parallel_loglik_arrays with host arrays: pipelined chunked upload
    (several chain launches feeding one tree) gives the reference value."""
    from paper_2003_03508_b200 import synth

    gold = load("bench_configs.json")["workloads"]["k25_n1e6"]["loglik"][0]
    plist, pr, lo, la = synth.make_workload("k25_n1e6")
    vals = [eng._parallel_loglik_arrays(plist[0], pr, lo, la, eng.EngineConfig()) for _ in range(3)]
    assert vals[1] == vals[2]                       # deterministic through the pipelined path
    for v in vals:
        assert rel(v, gold) <= TOL
        assert rel(v, gold) < 1e-12
    # a different stream through the same scratch handle, then back
    small = eng._parallel_loglik_arrays(plist[0], pr[:1000], lo[:1000], la[:1000], eng.EngineConfig())
    assert rel(small, coracle.forward_loglik(plist[0], pr[:1000], lo[:1000], la[:1000])) < TIGHT
    assert eng._parallel_loglik_arrays(plist[0], pr, lo, la, eng.EngineConfig()) == vals[2]


def test_stationary_batch_and_vector_pack(eng):
    """One-launch stationary distributions + vectorised proposal packing
    feeding the batched likelihood."""
    from paper_2003_03508_b200 import proposals

    cases = regen_cases("stationary")
    for c, p, pr, lo, la in cases:
        got = proposals.stationary_distribution_batch(np.stack([p.gamma, p.gamma]))
        for row in got:
            np.testing.assert_allclose(row, np.array(c["pi"]), rtol=1e-9, atol=1e-13)
    # stationary-delta proposals packed from vectors == object path
    rng = np.random.default_rng(21)
    plist = [fx.random_params(rng, 9) for _ in range(6)]
    vecs = proposals.params_to_vectors(plist)
    pack, ok = proposals.params_from_vectors(9, vecs, delta_mode="stationary")
    assert ok.all()
    pr, lo, la = fx.random_obs_arrays(rng, 800)
    dev = eng.DeviceObservations(pr, lo, la)
    got = dev.loglik_batch(pack, eng.EngineConfig())
    from oracle import thmm_oracle as npo
    for v, p in zip(got, plist):
        tied = eng.HmmParams(gamma=p.gamma, delta=npo.stationary_distribution(p.gamma), states=p.states)
        assert rel(v, coracle.forward_loglik(tied, pr, lo, la)) < 1e-10


def test_many_chain_sampler_runs_and_matches_single_eval(eng):
    """Batched MCMC: C chains, one likelihood launch per
    block move; the tracked log-likelihood of every chain equals a fresh
    single evaluation of its final state."""
    from paper_2003_03508_b200 import mcmc, proposals, synth

    k = 5
    plist, pr, lo, la = synth.make_workload("k5_n1e4", n=3000)
    base = plist[0]
    base = eng.HmmParams(gamma=0.99 * base.gamma + 0.01 / k, delta=base.delta, states=base.states)
    init = np.repeat(proposals.params_to_vectors([base]), 8, axis=0)
    dev = eng.DeviceObservations(pr, lo, la)
    res = mcmc.run_chains(k, dev, init, 10, steps=(0.1, 0.1, 0.005, 0.02), rng=np.random.default_rng(1))
    assert res.vectors.shape == (10, 8, proposals.vector_length(k))
    assert res.evaluations <= 1 + 9 * 4 + 2  # 9 sweeps of 4 blocks + 2 rejuvenation moves (it = 4, 8)
    assert res.proposed["rejuvenate"] == 2
    assert all(0.0 <= a.mean() <= 1.0 for a in res.acceptance.values())
    final = res.vectors[-1]
    pack, ok = proposals.params_from_vectors(k, final, "uniform")
    assert ok.all()
    again = dev.loglik_batch(pack, eng.EngineConfig())
    np.testing.assert_allclose(again, res.log_likelihood[-1], rtol=1e-12)


def test_batch_beyond_one_launch(eng, monkeypatch):
    """Batches larger than one launch's proposal limit run as consecutive
    launches (limit lowered here so the test stays small)."""
    monkeypatch.setattr(eng.engine, "MAX_BATCH", 3)
    rng = np.random.default_rng(77)
    plist = [fx.random_params(rng, 9) for _ in range(8)]
    pr, lo, la = fx.random_obs_arrays(rng, 2000)
    dev = eng.DeviceObservations(pr, lo, la)
    got = dev.loglik_batch(plist, eng.EngineConfig())
    assert got.shape == (8,)
    for p, v in zip(plist, got):
        assert rel(v, coracle.forward_loglik(p, pr, lo, la)) < TIGHT
