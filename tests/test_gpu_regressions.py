"""Regression tests for the CUDA-graph caches and argument validation of the
C ABI (round-1 advisor findings) -- needs a B200.

* a replayed host-pipeline graph must honour cfg->lo/hi (thmm_loglik_host);
* a replayed peer-exchange graph must notice that the handle's stream was
  replaced by a shorter one in the same buffers (thmm_peer_loglik);
* a call rejected for its cfg must leave the handle's records untouched.
Values are checked against the C oracle at the FP64 bar (1e-9).
"""

import os

import numpy as np
import pytest

import fixtures as fx
from oracle import coracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    return eng


def _pinned(pr, lo, la):
    import torch

    out = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (pr.view(np.uint8), lo, la)]
    return out, (out[0].numpy().view(np.bool_), out[1].numpy(), out[2].numpy())


def _host_call(eng, dev, plist, arrays, lo, hi):
    """thmm_loglik_host with a record range (the pipelined-copy entry)."""
    from paper_2003_03508_b200 import _native as nat
    from paper_2003_03508_b200.engine import _PackedParams, _native_config

    pr, lon, lat = arrays
    pp = _PackedParams(plist)
    out = np.empty(len(plist))
    status = np.empty(len(plist), dtype=np.int32)
    c = _native_config(eng.EngineConfig(), lo, hi, 0)
    err = nat.errbuf()
    rc = nat.lib().thmm_loglik_host(dev._handle, nat.as_ptr(pr.view(np.uint8), nat.c_uint8),
                                    nat.as_ptr(lon, nat.c_double), nat.as_ptr(lat, nat.c_double), pr.size,
                                    nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                    nat.as_ptr(out, nat.c_double), nat.as_ptr(status, nat.c_int32), err, len(err))
    return rc, out, err.value.decode()


def test_host_graph_keys_on_range(eng):
    rng = np.random.default_rng(5)
    plist = [fx.random_params(rng, 25)]
    pr, lo, la = fx.random_obs_arrays(rng, 20011, present_prob=0.3)
    keep, arrays = _pinned(pr, lo, la)
    dev = eng.DeviceObservations(pr[:16], lo[:16], la[:16])
    for a, b in ((0, 9000), (0, 9000), (9000, 20011), (9000, 20011), (0, 0), (5, 13001), (0, 9000)):
        rc, out, msg = _host_call(eng, dev, plist, arrays, a, b)
        assert rc == 0, msg
        hi = b if b else pr.size
        want = coracle.forward_loglik(plist[0], pr[a:hi], lo[a:hi], la[a:hi])
        assert abs(out[0] - want) <= 1e-9 * abs(want), (a, b, out[0], want)
    dev.close()
    del keep


def test_rejected_host_call_keeps_records(eng):
    rng = np.random.default_rng(6)
    plist = [fx.random_params(rng, 9)]
    pr, lo, la = fx.random_obs_arrays(rng, 5003)
    dev = eng.DeviceObservations(pr, lo, la)
    before = dev.loglik_batch(plist, eng.EngineConfig())
    pr2, lo2, la2 = fx.random_obs_arrays(rng, 40000)
    rc, _, msg = _host_call(eng, dev, plist, (pr2, lo2, la2), 0, 50000)  # hi beyond the new stream
    assert rc != 0 and msg
    from paper_2003_03508_b200 import _native as nat

    assert nat.lib().thmm_obs_length(dev._handle) == pr.size
    after = dev.loglik_batch(plist, eng.EngineConfig())
    assert np.array_equal(before, after)
    dev.close()


def test_peer_graph_notices_shorter_stream(eng):
    """World-1 process group, peer transport: graph captured on a stream of
    n records, then the stream is replaced by a shorter one in the same
    buffers (assign); the replay must evaluate the new records."""
    import socket

    import torch.distributed as dist

    from paper_2003_03508_b200.distributed import ShardedLoglik

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(7)
        plist = [fx.random_params(rng, 25)]
        pr, lo, la = fx.random_obs_arrays(rng, 30000, present_prob=0.3)
        sh = ShardedLoglik(pr, lo, la, device=0, transport="peer")
        import torch

        stream = torch.cuda.Stream()
        for _ in range(3):  # eager, capture, replay
            got = sh.loglik_batch(plist, eng.EngineConfig(), stream=stream.cuda_stream)
        want = coracle.forward_loglik(plist[0], pr, lo, la)
        assert sh.transport_used == "peer"
        assert abs(got[0] - want) <= 1e-9 * abs(want)
        m = 17001
        sh.obs.assign(pr[:m], lo[:m], la[:m])
        got2 = sh.loglik_batch(plist, eng.EngineConfig(), stream=stream.cuda_stream)
        want2 = coracle.forward_loglik(plist[0], pr[:m], lo[:m], la[:m])
        assert abs(got2[0] - want2) <= 1e-9 * abs(want2), (got2, want2)
        sh.close()
    finally:
        dist.destroy_process_group()
