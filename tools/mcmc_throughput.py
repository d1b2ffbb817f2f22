"""The consumer of the likelihood: MCMC iterations per second on a
Shikoku-sized synthetic catalogue (N ~ 105,000 hourly records).

1. the reference sampler ``tremorhmm.run_chain`` with its own CPU engine
   (baseline/_ref, one worker per physical core);
2. the SAME reference sampler with the B200 likelihood swapped in through its
   ``loglik_fn`` hook (bayes.py:693) -- the drop-in, unchanged driver;
3. the many-chain lockstep sampler (mcmc.run_chains): C chains per batched
   likelihood launch.

    python tools/mcmc_throughput.py [--k 25] [--n 105000] [--iters 20] [--chains 256]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numpy as np  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import mcmc, proposals, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=25)
ap.add_argument("--n", type=int, default=105_000)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--ref-iters", type=int, default=3)
ap.add_argument("--chains", type=int, default=256)
a = ap.parse_args()

rng = np.random.default_rng(7)
truth = synth.sample_prior_params(a.k, rng)
_, pr, lo, la = synth.simulate_arrays(truth, a.n, rng)
print(f"K={a.k} N={a.n} (synthetic, reference bench recipe)", flush=True)

ref_path = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(ref_path, "tremorhmm")):
    sys.path.insert(0, ref_path)
    import tremorhmm as th

    obs = [th.Observation((x, y)) if f else th.Observation(None) for f, x, y in zip(pr, lo, la)]
    spec = th.PriorSpec.default_for(a.k)
    cores = os.cpu_count() or 1
    mc = th.McmcConfig(iterations=a.ref_iters, thin=1, seed=3)
    ecfg = th.EngineConfig(workers=cores, segments=cores)
    try:
        th.run_chain(a.k, obs, spec, th.McmcConfig(iterations=1, thin=1, seed=3), ecfg,
                     delta_mode="uniform")  # numba warm-up
        t0 = time.perf_counter()
        th.run_chain(a.k, obs, spec, mc, ecfg, delta_mode="uniform")
        t_ref = (time.perf_counter() - t0) / a.ref_iters
        print(f"1. reference run_chain, reference CPU engine ({cores} workers): {t_ref * 1e3:9.1f} ms/iteration "
              f"({1 / t_ref:8.2f} it/s)", flush=True)
    except RuntimeError as exc:  # the reference initialises from prior draws only
        print(f"1. reference run_chain could not initialise on this catalogue: {exc}", flush=True)

    dev = eng.DeviceObservations(pr, lo, la)
    cfg = eng.EngineConfig()
    calls = [0]

    def loglik_fn(p):
        calls[0] += 1
        return dev.loglik(p, cfg)

    try:
        th.run_chain(a.k, None, spec, th.McmcConfig(iterations=2, thin=1, seed=3), ecfg,
                     delta_mode="uniform", loglik_fn=loglik_fn)
        calls[0] = 0
        mc2 = th.McmcConfig(iterations=a.iters, thin=1, seed=3)
        t0 = time.perf_counter()
        th.run_chain(a.k, None, spec, mc2, ecfg, delta_mode="uniform", loglik_fn=loglik_fn)
        t_drop = (time.perf_counter() - t0) / a.iters
        print(f"2. reference run_chain, B200 likelihood via loglik_fn:         {t_drop * 1e3:9.1f} ms/iteration "
              f"({1 / t_drop:8.2f} it/s, {calls[0] / a.iters:.2f} likelihood calls/iteration)", flush=True)
    except RuntimeError as exc:
        print(f"2. reference run_chain could not initialise on this catalogue: {exc}", flush=True)
else:
    print("reference package not installed (tools/install_reference.sh): skipping 1-2")

dev = eng.DeviceObservations(pr, lo, la)
start = eng.HmmParams(gamma=0.999 * np.asarray(truth.gamma) + 0.001 / a.k, delta=truth.delta, states=truth.states)
init = np.repeat(proposals.params_to_vectors([start]), a.chains, axis=0)
mcmc.run_chains(a.k, dev, init, 2, rng=np.random.default_rng(1))
t0 = time.perf_counter()
res = mcmc.run_chains(a.k, dev, init, a.iters + 1, rng=np.random.default_rng(1), points=(pr, lo, la))
t_many = (time.perf_counter() - t0) / a.iters
print(f"3. many-chain sampler, {a.chains} chains per launch:                {t_many * 1e3:9.1f} ms/iteration "
      f"({a.chains / t_many:8.1f} chain-it/s, {res.evaluations} batched launches)", flush=True)
