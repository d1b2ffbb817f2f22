"""pytest plugin: run the REFERENCE's own test suite against the B200 engine.

Loaded with ``-p ref_shim`` when pytest runs the reference's tests
(baseline/_ref/ref_tests, installed by tools/install_reference.sh).  It
replaces exactly the hot path the drop-in covers -- ``parallel_loglik`` and
``_parallel_loglik_arrays`` (reference engine.py:321-359, re-exported by
__init__.py:50-59) -- with the B200 engine, converting the reference's own
``EngineConfig`` field by field; everything else (the serial oracle, brute
force, priors, simulation) stays the reference's.  This is how a tremorhmm
maintainer would swap the backend in.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import tremorhmm  # noqa: E402  (the reference package, baseline/_ref)
import tremorhmm.engine as ref_engine  # noqa: E402

import paper_2003_03508_b200 as b200  # noqa: E402
from paper_2003_03508_b200 import _native  # noqa: E402

_native.require_device()  # the CUDA path, or fail loudly


def _cfg(cfg):
    return b200.EngineConfig(workers=cfg.workers, segments=cfg.segments, renorm_period=cfg.renorm_period,
                             precision=cfg.precision)


def parallel_loglik(params, obs, cfg):
    return b200.parallel_loglik(params, obs, _cfg(cfg))


def _parallel_loglik_arrays(params, present, lon, lat, cfg):
    return b200._parallel_loglik_arrays(params, present, lon, lat, _cfg(cfg))


CALLS = {"n": 0}


def _counted(fn):
    def wrapper(*a, **kw):
        CALLS["n"] += 1
        return fn(*a, **kw)
    return wrapper


tremorhmm.parallel_loglik = ref_engine.parallel_loglik = _counted(parallel_loglik)
ref_engine._parallel_loglik_arrays = _counted(_parallel_loglik_arrays)


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"ref_shim: {CALLS['n']} likelihood calls served by the B200 engine "
                                f"({_native.LIB_PATH})")
