"""The CPU oracle (numpy + C restatements) against the reference goldens.

Pins oracle/thmm_oracle.py and oracle/thmm_oracle.c to the values the
reference itself produced (tests/golden/, made by oracle/gen_golden.py)
before either is trusted as the checker of the CUDA path.
"""

import math

import numpy as np
import pytest

import fixtures as fx
from conftest import needs_reference
from golden_io import load, regen_cases, rel
from oracle import coracle
from oracle import thmm_oracle as npo


def test_regenerated_inputs_match_digests():
    assert len(regen_cases()) == len(load("engine_cases.json")["cases"])


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_matches_serial_cases(impl):
    for c, p, pr, lo, la in regen_cases("matches_serial"):
        if impl == "numpy":
            s = npo.forward_loglik_arrays(p, pr, lo, la, 1)
            par = npo.parallel_loglik_arrays(p, pr, lo, la, segments=4)
        else:
            s = coracle.forward_loglik(p, pr, lo, la, 1)
            par = coracle.parallel_loglik(p, pr, lo, la, segments=4, threads=2)
        assert rel(s, c["serial"]) < 1e-12, c["k"]
        assert rel(par, c["parallel_s4"]) < 1e-12, c["k"]


def test_schedule_and_segments():
    (c, p, pr, lo, la), = regen_cases("schedule")
    for r, want in c["serial"].items():
        assert rel(npo.forward_loglik_arrays(p, pr, lo, la, int(r)), want) < 1e-13
        assert rel(coracle.forward_loglik(p, pr, lo, la, int(r)), want) < 1e-13
    for r, want in c["parallel"].items():
        assert rel(npo.parallel_loglik_arrays(p, pr, lo, la, 1, int(r)), want) < 1e-13
    (c, p, pr, lo, la), = regen_cases("segment_invariance")
    for s, want in c["parallel"].items():
        assert rel(coracle.parallel_loglik(p, pr, lo, la, int(s), threads=3), want) < 1e-13


def test_brute_force_and_single_observation():
    for c, p, pr, lo, la in regen_cases("brute"):
        assert rel(npo.brute_force_loglik(p, pr, lo, la), c["brute"]) < 1e-12
        assert rel(coracle.forward_loglik(p, pr, lo, la), c["serial"]) < 1e-12
    (c, p, pr, lo, la), = regen_cases("single_obs")
    e = npo.emission_columns(p, pr, lo, la)[0]
    assert rel(math.log(float(p.delta @ p.gamma @ e)), c["serial"]) < 1e-12


def test_emission_table():
    (c, p, pr, lo, la), = regen_cases("emissions")
    want = np.array(c["table"])
    assert np.array_equal(npo.emission_columns(p, pr, lo, la), want)
    np.testing.assert_allclose(coracle.emissions(p, pr, lo, la), want, rtol=1e-14, atol=0)


def test_factor_segments_and_combine():
    (c, p, pr, lo, la), = regen_cases("factor_segments")
    ed = npo.emission_columns(p, pr, lo, la)
    parts = []
    for part in c["parts"]:
        m, ls = npo.chain_segment(np.asarray(p.gamma), ed[part["lo"]:part["hi"]], 8)
        np.testing.assert_allclose(m * math.exp(ls), np.array(part["m"]) * math.exp(part["log_scale"]),
                                   rtol=1e-12)
        parts.append((part["lo"], part["hi"], m, ls))
    assert rel(npo.combine_segments(p.delta, parts), c["combined"]) < 1e-12
    with pytest.raises(ValueError):
        npo.combine_segments(p.delta, [parts[0], parts[2]])
    with pytest.raises(RuntimeError):
        npo.combine_segments(np.array([0.5, 0.5]), [(0, 3, np.zeros((2, 2)), 0.0)])


def test_filtered_next_state():
    for c, p, pr, lo, la in regen_cases("filtered"):
        np.testing.assert_allclose(npo.filtered_next_state(p, pr, lo, la), np.array(c["dist"]), rtol=1e-12,
                                   atol=1e-300)


def test_criterion1_instances_c_oracle():
    gold = load("criterion1.json")["instances"]
    worst = 0.0
    for g, (k, n, segs, p, pr, lo, la) in zip(gold, fx.criterion1_instances()):
        assert (k, n, segs) == (g["k"], g["n"], g["segments"])
        assert fx.digest(pr, lo, la) == g["obs_digest"]
        s = coracle.forward_loglik(p, pr, lo, la)
        par = coracle.parallel_loglik(p, pr, lo, la, segs, threads=2)
        worst = max(worst, rel(s, g["serial"]), rel(par, g["parallel"]))
        if g["brute"] is not None:
            worst = max(worst, rel(s, g["brute"]))
    assert worst < 1e-11, worst


def test_criterion2_c_oracle():
    from paper_2003_03508_b200 import synth

    g = load("criterion2.json")
    rng = np.random.default_rng(2)
    p = synth.sample_prior_params(25, rng)
    _, pr, lo, la = synth.simulate_arrays(p, 100_000, rng)
    assert fx.digest(pr, lo, la) == g["obs_digest"]
    for s, want in g["parallel"].items():
        assert rel(coracle.parallel_loglik(p, pr, lo, la, int(s)), want) < 1e-12


@needs_reference
def test_fixtures_match_reference_generators():
    import sys

    sys.path.insert(0, "/root/reference/pkg/tests")
    sys.path.insert(0, "/root/reference/pkg/src")
    import test_core as tc
    from tremorhmm import observation_arrays

    for seed, k, n in ((3, 4, 40), (9, 30, 100)):
        r1, r2 = np.random.default_rng(seed), np.random.default_rng(seed)
        a, b = tc.random_params(r1, k), fx.random_params(r2, k)
        for f in ("gamma", "delta", "_p", "_mu0", "_mu1", "_l00", "_l10", "_l11", "_log_det"):
            assert np.array_equal(getattr(a, f), getattr(b, f))
        for x, y in zip(observation_arrays(tc.random_obs(r1, n)), fx.random_obs_arrays(r2, n)):
            assert np.array_equal(x, y)


def test_stationary_distribution():
    for c, p, pr, lo, la in regen_cases("stationary"):
        np.testing.assert_allclose(npo.stationary_distribution(p.gamma), np.array(c["pi"]), rtol=1e-12, atol=1e-15)
