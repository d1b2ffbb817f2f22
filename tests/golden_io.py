"""Load the golden fixtures (generated from the reference by oracle/gen_golden.py)."""

import json
import os

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def cases(kind=None):
    doc = load("engine_cases.json")["cases"]
    return [c for c in doc if kind is None or c["kind"] == kind]


def rel(a, b):
    return abs(a - b) / abs(b)


def regen_cases(kind=None):
    """Rebuild the inputs of every engine case from its seed (same recipe as
    oracle/gen_golden.py) and check them against the stored digests."""
    import numpy as np

    import fixtures as fx

    out = []
    brute_rng = None
    for c in cases():
        if c["kind"] == "brute":
            brute_rng = brute_rng or np.random.default_rng(16)
            rng = brute_rng
        else:
            rng = np.random.default_rng(c["seed"])
        p = fx.random_params(rng, c["k"])
        if c["kind"] == "single_obs":
            pr, lo, la = np.array([True]), np.array([0.3]), np.array([-0.4])
        else:
            pr, lo, la = fx.random_obs_arrays(rng, c["n"])
        assert fx.params_digest(p) == c["params_digest"], c["kind"]
        assert fx.digest(pr, lo, la) == c["obs_digest"], c["kind"]
        if kind is None or c["kind"] == kind:
            out.append((c, p, pr, lo, la))
    return out


def emission_case_inputs(name):
    """(params, present, lon, lat) of a golden emission case (recipe shared
    with oracle/gen_golden_emissions.py)."""
    import numpy as np

    import fixtures as fx

    if name in ("near", "far_tail", "absent"):
        rng = np.random.default_rng(36)
        p = fx.random_params(rng, 6)
        if name == "near":
            pr, lo, la = fx.random_obs_arrays(rng, 400)
        elif name == "far_tail":
            pr, lo, la = fx.random_obs_arrays(rng, 400, present_prob=0.9, spread=40.0)
        else:
            pr, lo, la = fx.random_obs_arrays(rng, 400, present_prob=0.0)
        return p, pr, lo, la
    from paper_2003_03508_b200 import synth

    wl, n = {"k80_bench": ("k80_n1e8", 300), "k25_bench": ("k25_n1e6", 600)}[name]
    plist, pr, lo, la = synth.make_workload(wl, n=n)
    return plist[0], pr, lo, la
