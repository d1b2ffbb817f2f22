"""Native observation-CSV ingestion vs the reference loader (CPU only)."""

import numpy as np
import pytest

from conftest import needs_reference
from paper_2003_03508_b200 import dataio


def write(tmp_path, text, name="d.csv"):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_roundtrip_and_quiet_hours(tmp_path):
    p = write(tmp_path, "timestamp,lon,lat\n2024-01-01T00:00:00,133.25,33.5\n2024-01-01T01:00:00,,\n"
                        "2024-01-01T02:00:00, -1.5e2 ,0.125\n\n2024-01-01T03:00:00.5+00:00,1,2\n")
    pr, lo, la, ts = dataio.load_arrays(p, with_timestamps=True)
    assert pr.tolist() == [True, False, True, True]
    assert lo.tolist() == [133.25, 0.0, -150.0, 1.0]
    assert la.tolist() == [33.5, 0.0, 0.125, 2.0]
    assert np.all(np.diff(ts) > 0)
    assert ts[1] - ts[0] == 3_600_000_000


@pytest.mark.parametrize("text,msg", [
    ("", "line 1: missing header"),
    ("time,lon,lat\n", "line 1: header must be"),
    ("timestamp,lon,lat\n2024-01-01T00:00:00,1\n", "line 2: expected 3 fields, got 2"),
    ("timestamp,lon,lat\nyesterday,1,2\n", "line 2: bad timestamp"),
    ("timestamp,lon,lat\n2024-01-01T01:00:00,1,2\n2024-01-01T01:00:00,1,2\n", "line 3: timestamps must be strictly"),
    ("timestamp,lon,lat\n2024-01-01T00:00:00,1,\n", "line 2: lon and lat must be both present or both empty"),
    ("timestamp,lon,lat\n2024-01-01T00:00:00,abc,2\n", "line 2: bad coordinate"),
    ("timestamp,lon,lat\n2024-01-01T00:00:00,inf,2\n", "line 2: coordinates must be finite"),
])
def test_errors_match_reference_messages(tmp_path, text, msg):
    p = write(tmp_path, text)
    with pytest.raises(ValueError, match=msg):
        dataio.load_arrays(p)


@needs_reference
def test_matches_reference_loader(tmp_path):
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from tremorhmm import dataio as ref_io
    from tremorhmm import core as ref_core

    rng = np.random.default_rng(3)
    lines = ["timestamp,lon,lat"]
    for h in range(500):
        ts = f"2019-{1 + h // 400:02d}-{1 + (h // 24) % 16:02d}T{h % 24:02d}:{(h * 7) % 60:02d}:00"
        if rng.random() < 0.4:
            lines.append(f"{ts},{rng.uniform(132, 135):.9f},{rng.uniform(32, 35):.9f}")
        else:
            lines.append(f"{ts},,")
    # keep timestamps strictly increasing for the reference too
    rows = [lines[0]] + [f"2019-01-01T00:00:00+00:00".replace("00:00:00", f"{i // 3600 % 24:02d}:{i // 60 % 60:02d}:{i % 60:02d}").replace("01-01", f"01-{1 + i // 86400:02d}") + "," + r.split(",", 1)[1] for i, r in enumerate(lines[1:])]
    p = write(tmp_path, "\n".join(rows) + "\n")
    ds = ref_io.load_dataset(p)
    want = ref_core.observation_arrays(ds.observations)
    got = dataio.load_arrays(p)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
