"""Batched proposal packing (host, CPU) against the reference constructors."""

import numpy as np
import pytest

import fixtures as fx
from conftest import needs_reference
from paper_2003_03508_b200 import proposals
from paper_2003_03508_b200.model import HmmParams, StateEmission, pack_params


def _obj_from_vec(k, v, delta):
    g = v[:k * k].reshape(k, k)
    ps = v[k * k:k * k + k]
    mus = v[k * k + k:k * k + 3 * k].reshape(k, 2)
    sg = v[k * k + 3 * k:].reshape(k, 3)
    states = tuple(StateEmission(ps[j], mus[j], np.array([[sg[j, 0], sg[j, 1]], [sg[j, 1], sg[j, 2]]]))
                   for j in range(k))
    return HmmParams(gamma=g, delta=delta, states=states)


def test_vectors_roundtrip_and_uniform_pack():
    rng = np.random.default_rng(8)
    plist = [fx.random_params(rng, 7) for _ in range(5)]
    vecs = proposals.params_to_vectors(plist)
    assert vecs.shape == (5, proposals.vector_length(7))
    pack, ok = proposals.params_from_vectors(7, vecs, delta_mode="uniform")
    assert ok.all()
    ref = pack_params([_obj_from_vec(7, v, np.full(7, 1 / 7)) for v in vecs])
    np.testing.assert_array_equal(pack.gamma, ref.gamma)
    np.testing.assert_array_equal(pack.delta, ref.delta)
    np.testing.assert_allclose(pack.states, ref.states, rtol=1e-15, atol=0)


def test_invalid_rows_are_flagged():
    rng = np.random.default_rng(9)
    vecs = proposals.params_to_vectors([fx.random_params(rng, 3) for _ in range(6)])
    k = 3
    vecs[1, 0] += 1e-6                          # gamma row no longer stochastic
    vecs[2, k * k] = 1.0                        # p == 1
    vecs[3, k * k + 3 * k] = -1.0               # s00 < 0
    vecs[4, k * k + 3 * k + 1] = 10.0           # |s01| too large -> not PD
    vecs[5, k * k + k] = np.nan                 # mu not finite
    pack, ok = proposals.params_from_vectors(k, vecs, delta_mode="uniform")
    assert ok.tolist() == [True, False, False, False, False, False]
    assert pack.B == 1
    for i in range(1, 6):
        with pytest.raises(ValueError):
            _obj_from_vec(k, vecs[i], np.full(k, 1 / k))


@needs_reference
def test_layout_matches_reference_params_to_vector():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from tremorhmm import bayes

    rng = np.random.default_rng(10)
    p = fx.random_params(rng, 4)
    rp = bayes.params_from_vector(4, proposals.params_to_vectors([p])[0], delta_mode="uniform")
    np.testing.assert_array_equal(bayes.params_to_vector(rp), proposals.params_to_vectors([p])[0])
