"""The hot path's emission values, held directly against the reference.

The chain kernels never write the emission diagonal to HBM; they evaluate it
with ``emission_rc`` (csrc/thmm_kernels.cuh): the reference's operation order
(core.py:255-258) with the two Cholesky divisions refined from correctly
rounded reciprocals.  ``thmm_emissions_chain`` runs that same device function
into a table, so the values the likelihood multiplies by are compared with
the reference's ``batch_emissions`` (tests/golden/emission_cases.*, generated
by oracle/gen_golden_emissions.py from the reference itself), element by
element in units in the last place: near-mean records, far-tail records
(emissions down to subnormals and exact zeros), an all-absent stream and
prefixes of the K=25 / K=80 BASELINE workloads.

Bound (stated): <= 4 ulp for every entry (only exp() and the reciprocal
refinement may differ from numpy); absent entries bit-identical (q = 1-p).
"""

import os

import numpy as np
import pytest

import fixtures as fx
from golden_io import GOLD, emission_case_inputs, load

ULP_BOUND = 4


def ulp_diff(a, b):
    """|a - b| in units in the last place for nonnegative doubles (ordered
    bit patterns: 0, subnormals and normals are consecutive integers)."""
    ia = np.asarray(a, dtype=np.float64).view(np.int64)
    ib = np.asarray(b, dtype=np.float64).view(np.int64)
    return np.abs(ia - ib)


def golden():
    meta = load("emission_cases.json")
    tables = np.load(os.path.join(GOLD, meta["tables"]))
    for c in meta["cases"]:
        p, pr, lo, la = emission_case_inputs(c["name"])
        assert fx.params_digest(p) == c["params_digest"] and fx.digest(pr, lo, la) == c["obs_digest"]
        yield c["name"], p, pr, lo, la, tables[c["name"]]


def test_oracle_emissions_match_reference_goldens():
    """Both oracle restatements (numpy, C) against the same goldens (CPU):
    the numpy one is the reference's arithmetic verbatim (bit-identical)."""
    from oracle import coracle
    from oracle import thmm_oracle as npo

    for name, p, pr, lo, la, want in golden():
        got = npo.emission_columns(p, pr, lo, la)
        assert np.array_equal(got, want), name
        assert ulp_diff(coracle.emissions(p, pr, lo, la), want).max() <= ULP_BOUND, name


@pytest.mark.gpu
@pytest.mark.parametrize("chain", [True, False])
def test_device_emissions_match_reference(chain):
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    worst = {}
    for name, p, pr, lo, la, want in golden():
        dev = eng.DeviceObservations(pr, lo, la)
        got = dev.emissions(p, chain=chain)
        dev.close()
        assert got.shape == want.shape
        d = ulp_diff(got, want)
        worst[name] = int(d.max())
        assert d.max() <= ULP_BOUND, (name, chain, int(d.max()))
        assert np.array_equal(got[~pr], want[~pr]), name  # absent rows: q exactly
        if name == "far_tail":  # the case exercises the far tail: tiny, subnormal and zero entries
            assert (want[pr] == 0).any() and ((want[pr] > 0) & (want[pr] < 1e-200)).any()
    print("max ulp per case", worst)
