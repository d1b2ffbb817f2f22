"""Multi-rank sharded likelihood with the REAL device kernels -- needs a B200.

In-round GPU access is a single GPU, so world sizes 2 and 3 run as several
processes sharing cuda:0 over gloo (ShardedLoglik stages the one packed
all-gather through the host; on NCCL the same buffers move over NVLink).
Everything else is the production multi-GPU path: each rank uploads only its
contiguous shard, reduces it with thmm_range_nodes_async, the per-rank
(nodes | exponents) blocks are gathered in rank order and folded with
thmm_fold_nodes_strided -- and every rank must return the single-GPU value.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import fixtures as fx
from oracle import coracle
from paper_2003_03508_b200.distributed import shard_bounds

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    rng = np.random.default_rng(31)
    plist = [fx.random_params(rng, k) for k in (25, 25, 25)]
    pr, lo, la = fx.random_obs_arrays(rng, 20011)
    return plist, pr, lo, la


def _worker_b1(rank, world, port, transport, q):
    import torch
    import torch.distributed as dist

    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200.distributed import ShardedLoglik

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(55)
        p = fx.random_params(rng, 25)
        pr, lo, la = fx.random_obs_arrays(rng, 50001)
        sh = ShardedLoglik(pr, lo, la, device=0, transport=transport)
        a = sh.loglik_batch([p], eng.EngineConfig())
        b = sh.loglik_batch([p], eng.EngineConfig())
        q.put((rank, a.tolist(), b.tolist(), sh.transport_used))
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_sharded_five_ranks_single_proposal(transport):
    """World 5 with one proposal: more ranks than one fold group (radix 4) and
    an odd per-rank node block -- the layout the 8-GPU default bench uses.
    'nccl' is the all-gather path (gloo staging here), 'peer' the
    peer-memory stores + flags (CUDA IPC between the processes)."""
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    rng = np.random.default_rng(55)
    p = fx.random_params(rng, 25)
    pr, lo, la = fx.random_obs_arrays(rng, 50001)
    want = eng.DeviceObservations(pr, lo, la).loglik_batch([p], eng.EngineConfig())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_b1, args=(r, 5, port, transport, q)) for r in range(5)]
    for pc in procs:
        pc.start()
    res = [q.get(timeout=300) for _ in range(5)]
    for pc in procs:
        pc.join(timeout=60)
        assert pc.exitcode == 0
    for rank, a, b, used in res:
        assert used == transport
        assert a == b == res[0][1]
        np.testing.assert_allclose(a, want, rtol=1e-12, atol=0)


def _worker(rank, world, port, precision, q):
    import torch
    import torch.distributed as dist

    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200.distributed import ShardedLoglik

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plist, pr, lo, la = _case()
        sh = ShardedLoglik(pr, lo, la, device=0)
        assert sh.n_local == eng.segment_bounds(pr.size, world)[rank][1] - eng.segment_bounds(pr.size, world)[rank][0]
        cfg = eng.EngineConfig(precision=precision)
        a = sh.loglik_batch(plist, cfg)
        b = sh.loglik_batch(plist, cfg)  # buffers reused
        lo_r, hi_r = eng.segment_bounds(pr.size, world)[rank]
        shard = tuple(np.ascontiguousarray(x[lo_r:hi_r]) for x in (pr, lo, la))
        c = sh.loglik_batch(plist, cfg, host_shard=shard)  # records re-sent from host, copy pipelined
        np.testing.assert_allclose(c, a, rtol=1e-12 if precision == "float64" else 1e-6, atol=0)
        q.put((rank, a.tolist(), b.tolist()))
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,precision", [(2, "float64"), (3, "float64"), (2, "tf32x3")])
def test_sharded_ranks_match_single_gpu(world, precision):
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    plist, pr, lo, la = _case()
    want = eng.DeviceObservations(pr, lo, la).loglik_batch(plist, eng.EngineConfig())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, precision, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tol = 1e-12 if precision == "float64" else 1e-6
    for rank, a, b in res:
        assert a == b, rank  # deterministic, identical on reuse
        np.testing.assert_allclose(a, want, rtol=tol, atol=0)
    assert all(r[1] == res[0][1] for r in res)  # every rank returns the same value


@pytest.mark.parametrize("workload", ["k25_n1e6", "k25_n1e6_b256", "k50_n1e7"])
def test_bench_torchrun_two_ranks_one_gpu(workload):
    """bench.py's torchrun path end to end with 2 ranks (gloo, both on cuda:0):
    chain-sharded for the single-proposal workload, proposal-sharded for the
    256-proposal batch."""
    env = dict(os.environ, THMM_BENCH_BACKEND="gloo", THMM_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "2", "--workload", workload,
           "--subconfigs", "none"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    import json

    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0 and rec["e2e"]["value"] > 0
    assert rec["e2e"]["pinned"]["value"] > 0 and rec["scaling"] == "strong"
    # strong scaling: the workload's N across both ranks, parity vs the golden at N=2
    assert rec["config"]["N"] == sum(rec["run"]["n_local_per_rank"]) or workload != "k25_n1e6"
    assert rec["parity_max_rel_vs_reference"] is not None and rec["parity_max_rel_vs_reference"] < 1e-9
    if workload == "k25_n1e6":
        assert rec["run"]["transport_used"] == "nccl" and rec["run"]["combine"] == "nodes"
        assert rec["run"]["n_local_per_rank"] == [500_000, 500_000]
    elif workload == "k50_n1e7":  # long shards: the stitched combine
        assert rec["run"]["combine"] == "stitched" and rec["run"]["n_local_per_rank"] == [5_000_000, 5_000_000]
    else:
        assert rec["config"]["N"] == rec["run"]["N_per_gpu"]
        assert "proposal-sharded" in rec["run"]["parallelism"]


def _replica_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200.distributed import ReplicaLoglik

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(41)
        plist = [fx.random_params(rng, 25) for _ in range(7)]
        pr, lo, la = fx.random_obs_arrays(rng, 30011)
        rep = ReplicaLoglik(pr, lo, la, device=0)
        a = rep.loglik_batch(plist, eng.EngineConfig())
        b = rep.loglik_batch(plist, eng.EngineConfig(), host=(pr, lo, la))
        q.put((rank, a.tolist(), b.tolist()))
        rep.close()
    finally:
        dist.destroy_process_group()


def test_replica_proposal_sharding_matches_single_gpu():
    """Batched proposals sharded over 3 ranks (all on cuda:0 over gloo):
    every rank returns all 7 values, equal to one single-GPU batch."""
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    rng = np.random.default_rng(41)
    plist = [fx.random_params(rng, 25) for _ in range(7)]
    pr, lo, la = fx.random_obs_arrays(rng, 30011)
    want = eng.DeviceObservations(pr, lo, la).loglik_batch(plist, eng.EngineConfig())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, a, b in res:
        np.testing.assert_allclose(a, want, rtol=1e-12, atol=0)
        np.testing.assert_allclose(b, want, rtol=1e-12, atol=0)


def _mcmc_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2003_03508_b200 import mcmc, synth
    from paper_2003_03508_b200.distributed import ReplicaLoglik

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        init, pr, lo, la = _mcmc_case()
        rep = ReplicaLoglik(pr, lo, la, device=0)
        res = mcmc.run_chains(6, rep, init, 4, rng=np.random.default_rng(3))
        q.put((rank, res.log_likelihood.tolist(), res.vectors.tolist()))
        rep.close()
    finally:
        dist.destroy_process_group()


def _mcmc_case():
    from paper_2003_03508_b200 import proposals, synth

    import paper_2003_03508_b200 as eng

    rng = np.random.default_rng(17)
    truth = synth.sample_prior_params(6, rng)
    _, pr, lo, la = synth.simulate_arrays(truth, 20000, rng)
    # strictly positive Gamma: the random walk moves log Gamma (reference bayes.py:406)
    start = eng.HmmParams(gamma=0.999 * np.asarray(truth.gamma) + 0.001 / 6, delta=truth.delta, states=truth.states)
    base = proposals.params_to_vectors([start])[0]
    init = np.stack([base] * 5)
    return init, pr, lo, la


def test_mcmc_chains_over_replica_ranks():
    """mcmc.run_chains with its proposals sharded over 2 ranks gives the
    single-GPU chains (same seed, same accept decisions)."""
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native, mcmc

    _native.require_device()
    init, pr, lo, la = _mcmc_case()
    want = mcmc.run_chains(6, eng.DeviceObservations(pr, lo, la), init, 4, rng=np.random.default_rng(3))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mcmc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ll, vecs in res:
        np.testing.assert_allclose(ll, want.log_likelihood, rtol=1e-12)
        np.testing.assert_allclose(vecs, want.vectors, rtol=0, atol=0)


def _shapes_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200.distributed import ShardedLoglik

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(808)
        pr, lo, la = fx.random_obs_arrays(rng, 30000)
        sh = ShardedLoglik(pr, lo, la, device=0, transport="auto")
        out = []
        for k, b in ((5, 1), (25, 2), (80, 3), (9, 4), (80, 1)):  # growing slots force re-setup
            plist = [fx.random_params(rng, k) for _ in range(b)]
            out.append((k, b, sh.loglik_batch(plist, eng.EngineConfig()).tolist(), sh.transport_used))
        q.put((rank, out))
        sh.close()
    finally:
        dist.destroy_process_group()


def test_sharded_shapes_sequence_peer():
    """One process group, a sequence of (K, B) shapes: the peer mailboxes are
    re-created collectively when a batch needs a larger slot, and every rank
    returns the single-GPU values for every shape."""
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shapes_worker, args=(r, 3, port, q)) for r in range(3)]
    for pc in procs:
        pc.start()
    res = [q.get(timeout=300) for _ in range(3)]
    for pc in procs:
        pc.join(timeout=60)
        assert pc.exitcode == 0
    rng = np.random.default_rng(808)
    pr, lo, la = fx.random_obs_arrays(rng, 30000)
    dev = eng.DeviceObservations(pr, lo, la)
    for k, b in ((5, 1), (25, 2), (80, 3), (9, 4), (80, 1)):
        plist = [fx.random_params(rng, k) for _ in range(b)]
        want = dev.loglik_batch(plist, eng.EngineConfig())
        for rank, out in res:
            kk, bb, vals, used = next(o for o in out if o[0] == k and o[1] == b)
            assert used == "peer"
            np.testing.assert_allclose(vals, want, rtol=1e-12, atol=0)


def _stitch_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native
    from paper_2003_03508_b200.distributed import ShardedLoglik

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _native.set_collapse_params(0.0, 256, -1.0)  # short shards take the stitched path too
        out = []
        # (the last case: 300k records per rank -- host shards staged by DMA in time chunks)
        for k, b, seed, n in ((25, 1, 61, 24_011), (50, 3, 62, 24_011), (9, 2, 63, 24_011), (33, 1, 64, 900_011)):
            rng = np.random.default_rng(seed)
            plist = [fx.random_params(rng, k) for _ in range(b)]
            pr, lo, la = fx.random_obs_arrays(rng, n, present_prob=0.3)
            sh = ShardedLoglik(pr, lo, la, device=0)
            a = sh.loglik_batch(plist, eng.EngineConfig())
            used = sh.combine_used
            c = sh.loglik_batch(plist, eng.EngineConfig(), host_shard=tuple(x[slice(*shard_bounds(pr.size, world)[rank])]
                                                                          for x in (pr, lo, la)))
            out.append((k, b, a.tolist(), c.tolist(), used, sh.combine_used))
            sh.close()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_stitched_combine_three_ranks():
    """The stitched multi-GPU combine (shard rows + links, two small
    all-gathers) over 3 ranks on cuda:0 (gloo): every rank returns the
    single-GPU value (<= 1e-11) and the C oracle's (1e-9), device-resident and
    from host shards."""
    import paper_2003_03508_b200 as eng
    from paper_2003_03508_b200 import _native

    _native.require_device()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stitch_worker, args=(r, 3, port, q)) for r in range(3)]
    for pc in procs:
        pc.start()
    res = [q.get(timeout=300) for _ in range(3)]
    for pc in procs:
        pc.join(timeout=60)
        assert pc.exitcode == 0
    for k, b, seed, n in ((25, 1, 61, 24_011), (50, 3, 62, 24_011), (9, 2, 63, 24_011), (33, 1, 64, 900_011)):
        rng = np.random.default_rng(seed)
        plist = [fx.random_params(rng, k) for _ in range(b)]
        pr, lo, la = fx.random_obs_arrays(rng, n, present_prob=0.3)
        want = np.array([coracle.forward_loglik(p, pr, lo, la) for p in plist])
        for rank, out in res:
            kk, bb, a, c, used, used2 = next(o for o in out if o[0] == k)
            assert used == "stitched" and used2 == "stitched", (rank, k, used, used2)
            np.testing.assert_allclose(a, want, rtol=1e-9, atol=0)
            np.testing.assert_allclose(c, a, rtol=1e-12, atol=0)
        assert all(next(o for o in out if o[0] == k)[2] == next(o for o in res[0][1] if o[0] == k)[2] for _, out in res)
