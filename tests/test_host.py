"""Host-side logic: reference-mirroring types/config, the C-ABI library
surface, and loud failure without a GPU.  No kernel launches (CPU suite)."""

import math
import re
import os

import numpy as np
import pytest

import fixtures as fx
from golden_io import regen_cases, rel
import paper_2003_03508_b200 as eng
from paper_2003_03508_b200 import _native
from oracle import thmm_oracle as npo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestEngineConfig:
    def test_defaults_and_dtype(self):
        cfg = eng.EngineConfig()
        assert (cfg.workers, cfg.segments, cfg.renorm_period, cfg.precision) == (1, None, 8, "float64")
        assert cfg.dtype == np.float64
        assert eng.EngineConfig(precision="float32").dtype == np.float32
        # precision-study modes (tensor-core products, float32 semantics)
        for prec in ("tf32", "tf32x2", "tf32x3"):
            assert eng.EngineConfig(precision=prec).dtype == np.float32
        from paper_2003_03508_b200 import _native
        assert _native.PRECISION_CODES == {"float64": 0, "float32": 1, "tf32": 2, "tf32x3": 3, "tf32x2": 4}

    def test_segments_default_to_workers(self):
        assert eng.EngineConfig(workers=3).resolved_segments() == 3
        assert eng.EngineConfig(workers=3, segments=5).resolved_segments() == 5

    @pytest.mark.parametrize("kw", [dict(workers=0), dict(workers=1.5), dict(segments=0),
                                    dict(renorm_period=0), dict(precision="float16"),
                                    dict(precision="bf16")])
    def test_rejects(self, kw):
        with pytest.raises(ValueError):
            eng.EngineConfig(**kw)


class TestSegmentBounds:
    def test_partition_properties(self):
        for n in (1, 2, 7, 100, 1001):
            for s in (1, 2, 3, 8):
                if s > n:
                    continue
                b = eng.segment_bounds(n, s)
                assert b[0][0] == 0 and b[-1][1] == n
                sizes = [hi - lo for lo, hi in b]
                assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
                assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
                assert b == npo.segment_bounds(n, s)

    def test_explicit_split_and_rejects(self):
        assert eng.segment_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
        with pytest.raises(ValueError):
            eng.segment_bounds(5, 0)
        with pytest.raises(ValueError):
            eng.segment_bounds(5, 6)


def test_scale_by_emission_exact():
    rng = np.random.default_rng(32)
    p = fx.random_params(rng, 5)
    d = rng.uniform(0.1, 2.0, size=5)
    assert np.array_equal(eng.scale_by_emission(p.gamma, d), p.gamma @ np.diag(d))
    with pytest.raises(ValueError):
        eng.scale_by_emission(p.gamma, -d)


class TestCombineSegments:
    def _parts(self):
        (c, p, pr, lo, la), = regen_cases("factor_segments")
        parts = [eng.SegmentProduct(eng.ScaledMatrix(m, ls), a, b)
                 for a, b, m, ls in npo.segment_products(p, pr, lo, la, 3)]
        return c, p, parts

    def test_matches_golden_and_order_independent(self):
        c, p, parts = self._parts()
        a = eng.combine_segments(p.delta, parts)
        assert a == eng.combine_segments(p.delta, list(reversed(parts)))
        assert rel(a, c["combined"]) < 1e-12

    def test_gap_and_collapse(self):
        c, p, parts = self._parts()
        with pytest.raises(ValueError):
            eng.combine_segments(p.delta, [parts[0], parts[2]])
        zero = eng.SegmentProduct(eng.ScaledMatrix(np.zeros((2, 2))), 0, 3)
        with pytest.raises(RuntimeError):
            eng.combine_segments(np.array([0.5, 0.5]), [zero])
        with pytest.raises(ValueError):
            eng.combine_segments(p.delta, [])
        with pytest.raises(ValueError):
            eng.SegmentProduct(eng.ScaledMatrix(np.ones((2, 2))), 3, 3)


class TestModelTypes:
    def test_cholesky_matches_numpy(self):
        rng = np.random.default_rng(10)
        for _ in range(50):
            sigma = fx.random_spd(rng)
            st = eng.StateEmission(0.5, np.zeros(2), sigma)
            assert np.allclose(st.chol, np.linalg.cholesky(sigma), rtol=0, atol=1e-12)
            assert math.isclose(st.log_det, np.linalg.slogdet(sigma)[1], rel_tol=1e-12, abs_tol=1e-12)

    def test_rejects(self):
        for bad in (0.0, 1.0, -0.2, 1.2, float("nan")):
            with pytest.raises(ValueError):
                eng.StateEmission(bad, np.zeros(2), np.eye(2))
        for sig in ([[1.0, 2.0], [2.0, 1.0]], [[1.0, 0.5], [0.1, 1.0]], [[-1.0, 0.0], [0.0, 1.0]]):
            with pytest.raises(ValueError):
                eng.StateEmission(0.5, np.zeros(2), np.array(sig))
        states = (eng.StateEmission(0.5, np.zeros(2), np.eye(2)),) * 2
        with pytest.raises(ValueError):
            eng.HmmParams(gamma=np.array([[0.6, 0.5], [0.5, 0.5]]), delta=np.array([0.5, 0.5]), states=states)
        with pytest.raises(ValueError):
            eng.HmmParams(gamma=np.full((2, 2), 0.5), delta=np.array([0.7, 0.7]), states=states)
        with pytest.raises(ValueError):
            eng.Observation((float("nan"), 1.0))

    def test_frozen_and_arrays(self):
        p = fx.random_params(np.random.default_rng(0), 3)
        assert p.K == 3
        with pytest.raises(ValueError):
            p.gamma[0, 0] = 0.9
        obs = [eng.Observation((1.0, 2.0)), eng.Observation(None), eng.Observation((-3.0, 4.5))]
        pr, lo, la = eng.observation_arrays(obs)
        assert pr.tolist() == [True, False, True] and lo.tolist() == [1.0, 0.0, -3.0]
        assert la.tolist() == [2.0, 0.0, 4.5]

    def test_pack_params_layout(self):
        rng = np.random.default_rng(3)
        plist = [fx.random_params(rng, 4) for _ in range(3)]
        pk = eng.pack_params(plist)
        assert pk.gamma.shape == (3, 4, 4) and pk.states.shape == (8, 3, 4)
        assert np.array_equal(pk.states[0, 1], plist[1]._p)
        assert np.array_equal(pk.states[1, 2], plist[2]._q)
        assert np.array_equal(pk.states[7, 0], plist[0]._log_det)
        with pytest.raises(ValueError):
            eng.pack_params([plist[0], fx.random_params(rng, 5)])


def header_symbols():
    text = open(os.path.join(ROOT, "include", "thmm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+(thmm_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, s
    assert lib.thmm_version() >= 100
    assert lib.thmm_padded_states(25) == 32 and lib.thmm_padded_states(80) == 80


def test_library_built_for_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(_native.load_library().thmm_device_count() > 0, reason="GPU present")
def test_fails_loudly_without_gpu():
    (c, p, pr, lo, la), = regen_cases("brute")[:1]
    with pytest.raises(_native.NativeUnavailable):
        eng._parallel_loglik_arrays(p, pr, lo, la, eng.EngineConfig())
    with pytest.raises(_native.NativeUnavailable):
        eng.DeviceObservations(pr, lo, la)
    with pytest.raises(ValueError):   # argument errors still come first, like the reference
        eng._parallel_loglik_arrays(p, pr[:0], lo[:0], la[:0], eng.EngineConfig())
