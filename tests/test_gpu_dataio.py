"""Observation CSV -> device stream -> likelihood, on the B200.

A BASELINE workload is written as the reference's dataset CSV (header
``timestamp,lon,lat``, hourly ISO timestamps, empty fields for quiet hours,
plus blank lines and padded fields the reference loader tolerates), loaded
with ``dataio.load_device_observations`` (native parser in libthmm, then one
upload) and evaluated.  Checked against:
  * the reference engine's golden logL of the same workload (tests/golden/
    bench_configs.json, K=5 N=10^4) at the FP64 bar 1e-9;
  * the reference's own loader (``tremorhmm.dataio.load_dataset`` ->
    ``observation_arrays``, from baseline/_ref when installed) bit for bit,
    and the C oracle's likelihood over those arrays;
  * malformed files raise the reference's ``line N: ...`` ValueError before
    anything reaches the device.
"""

import json
import os
import sys
from datetime import datetime, timedelta

import numpy as np
import pytest

from golden_io import GOLD

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write_csv(path, pr, lo, la):
    t0 = datetime(2013, 4, 1)
    lines = ["timestamp,lon,lat"]
    for i, (f, x, y) in enumerate(zip(pr, lo, la)):
        ts = (t0 + timedelta(hours=i)).isoformat()
        if f:
            x, y = float(x), float(y)  # repr of a Python float round-trips exactly
            lines.append(f"{ts},{x!r},{y!r}" if i % 7 else f"{ts}, {x!r} , {y!r}")  # padded fields too
        else:
            lines.append(f"{ts},,")
        if i % 1000 == 999:
            lines.append("")  # blank lines are skipped by the reference loader
    path.write_text("\n".join(lines) + "\n")


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


def test_csv_to_device_matches_golden(eng, tmp_path):
    from oracle import coracle
    from paper_2003_03508_b200 import dataio, synth

    plist, pr, lo, la = synth.make_workload("k5_n1e4")
    path = tmp_path / "k5.csv"
    _write_csv(path, pr, lo, la)
    dev = dataio.load_device_observations(path)
    assert len(dev) == pr.size
    got = dev.loglik(plist[0], eng.EngineConfig())
    gold = json.load(open(os.path.join(GOLD, "bench_configs.json")))["workloads"]["k5_n1e4"]["loglik"][0]
    assert abs(got - gold) <= 1e-9 * abs(gold), (got, gold)
    # bitwise the device-resident value of the in-memory arrays (the parse is exact)
    ref_dev = eng.DeviceObservations(pr, lo, la)
    assert got == ref_dev.loglik(plist[0], eng.EngineConfig())
    want = coracle.forward_loglik(plist[0], pr, lo, la)
    assert abs(got - want) <= 1e-9 * abs(want)
    dev.close()
    ref_dev.close()


def test_csv_matches_reference_loader(eng, tmp_path):
    from oracle import coracle
    from paper_2003_03508_b200 import dataio, synth

    ref = None
    for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "tremorhmm")):
            sys.path.insert(0, p)
            from tremorhmm import core as ref_core, dataio as ref_io
            ref = (ref_core, ref_io)
            break
    if ref is None:
        pytest.skip("reference package not installed")
    plist, pr, lo, la = synth.make_workload("k25_n1e6", n=20_000)
    path = tmp_path / "k25.csv"
    _write_csv(path, pr, lo, la)
    want = ref[0].observation_arrays(ref[1].load_dataset(path).observations)
    got = dataio.load_arrays(path)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    dev = dataio.load_device_observations(path)
    val = dev.loglik(plist[0], eng.EngineConfig())
    o = coracle.forward_loglik(plist[0], *want)
    assert abs(val - o) <= 1e-9 * abs(o)
    dev.close()


@pytest.mark.parametrize("text,msg", [
    ("timestamp,lon,lat\n2024-01-01T00:00:00,1\n", "line 2: expected 3 fields, got 2"),
    ("timestamp,lon,lat\n2024-01-01T01:00:00,1,2\n2024-01-01T01:00:00,1,2\n", "line 3: timestamps must be strictly"),
    ("timestamp,lon,lat\n2024-01-01T00:00:00,1,\n", "line 2: lon and lat must be both present or both empty"),
    ("timestamp,lon,lat\n", "observation sequence is empty"),
])
def test_malformed_csv_rejected_before_upload(eng, tmp_path, text, msg):
    from paper_2003_03508_b200 import dataio

    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        dataio.load_device_observations(p)
