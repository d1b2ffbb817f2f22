"""Golden emission tables from the REFERENCE's ``batch_emissions`` for the
hot-path emission test (tests/test_gpu_emissions.py).

TEST INFRASTRUCTURE ONLY.  Run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_emissions.py

Cases (inputs regenerated from seeds on the GPU box, pinned by digest):
  * ``near``     -- reference test fixture recipe (test_core.py:25-47), K=6;
  * ``far_tail`` -- the same parameters with records spread far from every
    mean (spread 40): emissions from O(1) down through 1e-200, subnormals
    and exact zeros -- where a reciprocal-based quotient could drift;
  * ``absent``   -- all records absent (the diagonal is q = 1-p exactly);
  * ``k80_bench``/``k25_bench`` -- 300/600-record prefixes of the BASELINE
    workloads (prior draw, simulated Shikoku-like path).
Writes tests/golden/emission_cases.json (digests) and emission_cases.npz
(the float64 tables, bit-exact).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import tremorhmm as ref  # noqa: E402

import fixtures as fx  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "oracle"))
from gen_golden import ref_params, to_obs  # noqa: E402
from golden_io import emission_case_inputs as case_inputs  # noqa: E402


CASES = ("near", "far_tail", "absent", "k25_bench", "k80_bench")


def main():
    out, tables = [], {}
    for name in CASES:
        p, pr, lo, la = case_inputs(name)
        table = ref.batch_emissions(ref_params(p), to_obs(pr, lo, la))
        out.append(dict(name=name, k=int(p.K), n=int(pr.size), params_digest=fx.params_digest(p),
                        obs_digest=fx.digest(pr, lo, la),
                        min_present=float(table[pr].min()) if pr.any() else None))
        tables[name] = np.asarray(table, dtype=np.float64)
        print(name, p.K, pr.size, "min present emission", out[-1]["min_present"])
    with open(os.path.join(ROOT, "tests", "golden", "emission_cases.json"), "w") as fh:
        json.dump(dict(generator="oracle/gen_golden_emissions.py", reference="tremorhmm 0.1.0 batch_emissions",
                       tables="emission_cases.npz", cases=out), fh)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "emission_cases.npz"), **tables)


if __name__ == "__main__":
    main()
