"""Per-rank device time of the strong-scaling shards on one GPU: the stitched
shard reduction (thmm_stitch_shard: main pass + links + shard summary) of
N/g records for g = 1, 2, 4, 8, plus the external link a rank >= 1 adds --
the compute a rank does at g GPUs (the exchange adds two small all-gathers).

    python tools/shard_scaling_probe.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2003_03508_b200 as eng  # noqa: E402
from paper_2003_03508_b200 import _native as nat, synth  # noqa: E402
from paper_2003_03508_b200.engine import _native_config, _PackedParams  # noqa: E402

nat.require_device()
for wl in ("k80_n1e8", "k50_n1e7"):
    plist, pr, lo, la = synth.make_workload(wl)
    p = plist[0]
    n = pr.size
    base = None
    for g in (1, 2, 4, 8):
        m = n // g
        dev = eng.DeviceObservations(pr[n - m:], lo[n - m:], la[n - m:])  # the last rank's shard
        kp = eng.padded_states(p.K)
        blk = torch.empty(kp + 2, dtype=torch.float64, device="cuda")
        lnk = torch.empty(2, dtype=torch.float64, device="cuda")
        pp = _PackedParams([p])
        st = torch.cuda.Stream()  # a real stream: the shard calls and the events on it
        c = _native_config(eng.EngineConfig(), 0, 0, st.cuda_stream)
        err = nat.errbuf()

        def one():
            assert nat.lib().thmm_stitch_shard(dev._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                               1 if g == 1 else 0, blk.data_ptr(), err, len(err)) == 0, err.value
            if g > 1:
                assert nat.lib().thmm_stitch_link(dev._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                                  nat.c_void_p(blk.data_ptr()), kp + 2, lnk.data_ptr(), err,
                                                  len(err)) == 0, err.value

        for _ in range(3):
            one()
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            one()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        base = base or t
        print(f"{wl} g={g}: shard of {m} records {t:.3f} ms  (speed-up {base / t:.2f}x, "
              f"strong-scaling efficiency of the compute {base / t / g:.2f})", flush=True)
        dev.close()
