"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

TEST INFRASTRUCTURE ONLY.  Run in the build container (the reference is not
on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py [small|bench|all]

It imports the reference package from /root/reference/pkg/src (read-only) and
its test fixtures from /root/reference/pkg/tests, evaluates the reference's own
public functions (``forward_loglik``, ``parallel_loglik``,
``brute_force_loglik``, ``batch_emissions`` and, for chains too long for the
reference's N x K emission table, its own kernels ``_emission_columns`` +
``_chain_fused_*`` + ``combine_segments`` streamed per segment -- bit-identical
to ``parallel_loglik(segments=S)``) and writes:

  tests/golden/engine_cases.json  unit cases of test_core / test_engine
  tests/golden/criterion1.json    the 200 instances of acceptance criterion 1
  tests/golden/bench_configs.json the BASELINE.json workloads (logL + input digests)

Inputs are not stored: tests regenerate them from the seeds with
tests/fixtures.py / paper_2003_03508_b200.synth and check the digests.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import tremorhmm as ref  # noqa: E402
from tremorhmm import core as ref_core, engine as ref_engine  # noqa: E402

import fixtures as fx  # noqa: E402
from paper_2003_03508_b200 import synth  # noqa: E402


def to_obs(present, lon, lat):
    return [ref.Observation((float(x), float(y))) if p else ref.Observation(None)
            for p, x, y in zip(present, lon, lat)]


def ref_params(p):
    """Rebuild a parameter set as the reference's own HmmParams."""
    states = tuple(ref.StateEmission(s.p, s.mu, s.sigma) for s in p.states)
    return ref.HmmParams(gamma=p.gamma, delta=p.delta, states=states)


def dump(name, obj):
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, name), "w") as fh:
        json.dump(obj, fh, indent=1, sort_keys=True)
    print("wrote", name)


def small_cases():
    cases = []

    def add(kind, seed, k, n, params, present, lon, lat, **vals):
        cases.append(dict(kind=kind, seed=seed, k=k, n=n, params_digest=fx.params_digest(params),
                          obs_digest=fx.digest(present, lon, lat), **vals))

    # test_engine.py:159-166 matches serial, K in {2,5,16,25,40} plus padding coverage
    for k in (1, 2, 3, 5, 7, 8, 9, 16, 17, 25, 33, 40, 49, 50, 57, 63, 64, 65, 72, 79, 80):
        seed = 40 + k
        rng = np.random.default_rng(seed)
        p = fx.random_params(rng, k)
        pr, lo, la = fx.random_obs_arrays(rng, 500)
        rp, obs = ref_params(p), to_obs(pr, lo, la)
        add("matches_serial", seed, k, 500, p, pr, lo, la,
            serial=ref.forward_loglik(rp, obs),
            parallel_s4=ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=4)))
    # test_engine.py:168-176 segment-count invariance
    rng = np.random.default_rng(41)
    p = fx.random_params(rng, 8)
    pr, lo, la = fx.random_obs_arrays(rng, 300)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("segment_invariance", 41, 8, 300, p, pr, lo, la,
        parallel={str(s): ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=s)) for s in (1, 2, 3, 7, 16)})
    # test_engine.py:178-186 single segment tracks the serial schedule
    rng = np.random.default_rng(42)
    p = fx.random_params(rng, 6)
    pr, lo, la = fx.random_obs_arrays(rng, 128)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("schedule", 42, 6, 128, p, pr, lo, la,
        serial={str(r): ref.forward_loglik(rp, obs, renorm_period=r) for r in (1, 4, 8, 64)},
        parallel={str(r): ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=1, renorm_period=r))
                  for r in (1, 4, 8, 64)})
    # test_engine.py:188-195 float32 vs float64
    rng = np.random.default_rng(43)
    p = fx.random_params(rng, 10)
    pr, lo, la = fx.random_obs_arrays(rng, 2000)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("float32", 43, 10, 2000, p, pr, lo, la,
        f64=ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=2)),
        f32=ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=2, precision="float32")))
    # test_engine.py:197-203 worker invariance
    rng = np.random.default_rng(44)
    p = fx.random_params(rng, 12)
    pr, lo, la = fx.random_obs_arrays(rng, 1000)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("workers", 44, 12, 1000, p, pr, lo, la,
        value=ref.parallel_loglik(rp, obs, ref.EngineConfig(workers=1, segments=4)))
    # test_core.py:196-202 brute force (one generator across the loop)
    rng = np.random.default_rng(16)
    for k, n in ((2, 8), (3, 6), (4, 5), (5, 4)):
        p = fx.random_params(rng, k)
        pr, lo, la = fx.random_obs_arrays(rng, n)
        rp, obs = ref_params(p), to_obs(pr, lo, la)
        add("brute", 16, k, n, p, pr, lo, la, serial=ref.forward_loglik(rp, obs),
            brute=ref.brute_force_loglik(rp, obs))
    # test_core.py:188-194 single observation
    rng = np.random.default_rng(15)
    p = fx.random_params(rng, 3)
    pr, lo, la = np.array([True]), np.array([0.3]), np.array([-0.4])
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("single_obs", 15, 3, 1, p, pr, lo, la, serial=ref.forward_loglik(rp, obs),
        parallel=ref.parallel_loglik(rp, obs, ref.EngineConfig()))
    # test_core.py:205-212 renorm schedule, K=5 N=400
    rng = np.random.default_rng(17)
    p = fx.random_params(rng, 5)
    pr, lo, la = fx.random_obs_arrays(rng, 400)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("renorm_k5", 17, 5, 400, p, pr, lo, la,
        serial={str(r): ref.forward_loglik(rp, obs, renorm_period=r) for r in (1, 2, 3, 8, 50)})
    # test_core.py:214-219 long sequence K=25 N=10^4
    rng = np.random.default_rng(18)
    p = fx.random_params(rng, 25)
    pr, lo, la = fx.random_obs_arrays(rng, 10_000)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("long_k25", 18, 25, 10_000, p, pr, lo, la, serial=ref.forward_loglik(rp, obs),
        parallel_s8=ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=8)))
    # test_engine.py:52-61 emission table, K=6 N=200
    rng = np.random.default_rng(30)
    p = fx.random_params(rng, 6)
    pr, lo, la = fx.random_obs_arrays(rng, 200)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    add("emissions", 30, 6, 200, p, pr, lo, la, table=ref.batch_emissions(rp, obs).tolist())
    # test_engine.py:96-109 / 124-133 segment products over an explicit factor stack
    rng = np.random.default_rng(35)
    p = fx.random_params(rng, 4)
    pr, lo, la = fx.random_obs_arrays(rng, 30)
    rp, obs = ref_params(p), to_obs(pr, lo, la)
    factors = np.stack([ref.scale_by_emission(rp.gamma, d) for d in ref.batch_emissions(rp, obs)])
    parts = ref.segment_chain_product(factors, ref.EngineConfig(segments=3))
    add("factor_segments", 35, 4, 30, p, pr, lo, la,
        parts=[dict(lo=q.lo, hi=q.hi, m=q.product.m.tolist(), log_scale=q.product.log_scale) for q in parts],
        combined=ref.combine_segments(rp.delta, parts))
    # simforecast.py:97-118 filtered next-state distribution (forecast conditioning)
    from tremorhmm import simforecast as ref_sf
    for seed, k, n in ((60, 3, 50), (61, 25, 2000), (62, 9, 1), (63, 50, 700)):
        rng = np.random.default_rng(seed)
        p = fx.random_params(rng, k)
        pr, lo, la = fx.random_obs_arrays(rng, n)
        rp, obs = ref_params(p), to_obs(pr, lo, la)
        add("filtered", seed, k, n, p, pr, lo, la, dist=ref_sf._filtered_next_state_dist(rp, obs).tolist())
    # core.py:350-388 stationary distribution (delta tied to Gamma in the MCMC driver)
    for seed, k in ((70, 3), (71, 25), (72, 80)):
        rng = np.random.default_rng(seed)
        p = fx.random_params(rng, k)
        pr, lo, la = fx.random_obs_arrays(rng, 1)
        add("stationary", seed, k, 1, p, pr, lo, la, pi=ref_core.stationary_distribution(p.gamma).tolist())
    dump("engine_cases.json", dict(generator="oracle/gen_golden.py", reference="tremorhmm 0.1.0",
                                   cases=cases))


def criterion1():
    out = []
    t0 = time.time()
    for k, n, segs, p, pr, lo, la in fx.criterion1_instances():
        rp, obs = ref_params(p), to_obs(pr, lo, la)
        serial = ref.forward_loglik(rp, obs)
        par = ref.parallel_loglik(rp, obs, ref.EngineConfig(segments=segs))
        brute = ref.brute_force_loglik(rp, obs) if k ** (n + 1) <= 1_000_000 else None
        out.append(dict(k=k, n=n, segments=segs, params_digest=fx.params_digest(p),
                        obs_digest=fx.digest(pr, lo, la), serial=serial, parallel=par, brute=brute))
    print(f"criterion1: {time.time() - t0:.1f} s")
    dump("criterion1.json", dict(generator="oracle/gen_golden.py", seed=20260814, instances=out))


def ref_chunked(params, present, lon, lat, segments, threads=8, period=8):
    """Reference kernels streamed per segment == parallel_loglik(segments=S)."""
    gamma = np.ascontiguousarray(params.gamma)
    k = params.K
    kern = ref_engine._chain_fused_small if k < 16 else ref_engine._chain_fused_blas
    bounds = ref_engine.segment_bounds(present.size, segments)

    def task(b):
        lo_, hi_ = b
        ed = ref_core._emission_columns(params, present[lo_:hi_], lon[lo_:hi_], lat[lo_:hi_])
        m, ls = kern(gamma, ed, 0, hi_ - lo_, period)
        return ref_engine.SegmentProduct(ref_core.ScaledMatrix(m, ls), lo_, hi_)

    with ThreadPoolExecutor(threads) as pool:
        parts = list(pool.map(task, bounds))
    return ref_engine.combine_segments(params.delta, parts)


def bench_configs(names):
    path = os.path.join(GOLD, "bench_configs.json")
    doc = json.load(open(path)) if os.path.exists(path) else dict(generator="oracle/gen_golden.py",
                                                                   workloads={})
    for name in names:
        t0 = time.time()
        plist, pr, lo, la = synth.make_workload(name)
        w = synth.WORKLOADS[name]
        entry = dict(k=w["k"], n=w["n"], seed=w["seed"], batch=w["batch"],
                     obs_digest=fx.digest(pr, lo, la),
                     params_digests=[fx.params_digest(p) for p in plist],
                     present_fraction=float(pr.mean()))
        rps = [ref_params(p) for p in plist]
        if name == "k5_n1e4":
            obs = to_obs(pr, lo, la)
            entry["serial"] = ref.forward_loglik(rps[0], obs)
            entry["parallel_s8"] = ref.parallel_loglik(rps[0], obs, ref.EngineConfig(workers=8, segments=8))
            entry["loglik"] = [entry["parallel_s8"]]
        elif name == "k25_n1e6":
            entry["serial"] = ref_core._forward_loglik_arrays(rps[0], pr, lo, la, 1)
            entry["parallel_s8"] = ref_engine._parallel_loglik_arrays(
                rps[0], pr, lo, la, ref.EngineConfig(workers=8, segments=8))
            entry["loglik"] = [entry["parallel_s8"]]
        elif name == "k25_n1e6_b256":
            entry["loglik"] = [ref_engine._parallel_loglik_arrays(rp, pr, lo, la,
                                                                  ref.EngineConfig(workers=8, segments=8))
                               for rp in rps]
            entry["serial_first"] = ref_core._forward_loglik_arrays(rps[0], pr, lo, la, 1)
        else:
            entry["loglik"] = [ref_chunked(rps[0], pr, lo, la, segments=64)]
            entry["reference_method"] = "reference _emission_columns + _chain_fused_blas per segment " \
                                        "+ combine_segments, 64 segments (== parallel_loglik(segments=64))"
        entry["seconds"] = time.time() - t0
        doc["workloads"][name] = entry
        print(name, entry["loglik"][:2], f"{entry['seconds']:.1f}s", flush=True)
        dump("bench_configs.json", doc)


def criterion2():
    rng = np.random.default_rng(2)
    p = synth.sample_prior_params(25, rng)
    _, pr, lo, la = synth.simulate_arrays(p, 100_000, rng)
    rp = ref_params(p)
    vals = {str(s): ref_engine._parallel_loglik_arrays(rp, pr, lo, la, ref.EngineConfig(segments=s))
            for s in (1, 2, 7, 28)}
    dump("criterion2.json", dict(generator="oracle/gen_golden.py", seed=2, k=25, n=100_000,
                                 params_digest=fx.params_digest(p), obs_digest=fx.digest(pr, lo, la),
                                 parallel=vals, serial=ref_core._forward_loglik_arrays(rp, pr, lo, la, 1)))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "cases":
        small_cases()
    if what in ("small", "all"):
        small_cases()
        criterion1()
        criterion2()
    if what in ("bench", "all"):
        bench_configs(["k5_n1e4", "k25_n1e6"])
    if what in ("bigbench", "all"):
        bench_configs(["k25_n1e6_b256", "k50_n1e7", "k80_n1e8"])
