"""Multi-GPU host logic on CPU: world_size 2 (and 3) over gloo.

The device reduction/fold are replaced by the oracle (the only part that
needs a GPU); what is exercised is the sharding, that each rank keeps only
its shard, the all-gather order and the ordered fold -- the code path
ShardedLoglik runs over NCCL on B200s.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fixtures as fx
from oracle import thmm_oracle as npo
from paper_2003_03508_b200.distributed import ReplicaLoglik, ShardedLoglik, shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_reduce(shard, params_list, cfg):
    """Node per proposal: (m padded to K_p, natural-log scale) of the shard."""
    pr, lo, la = shard
    k = params_list[0].K
    kp = ((k + 7) // 8) * 8
    m = torch.zeros((len(params_list), kp, kp), dtype=torch.float64)
    e = torch.zeros((len(params_list),), dtype=torch.float64)
    for b, p in enumerate(params_list):
        ed = npo.emission_columns(p, pr, lo, la)
        mm, ls = npo.chain_segment(np.asarray(p.gamma), ed, 8)
        m[b, :k, :k] = torch.from_numpy(mm)
        e[b] = ls
    return m, e


def oracle_fold(params_list, gm, ge):
    k = params_list[0].K
    out = []
    for b, p in enumerate(params_list):
        parts = [(g, g + 1, gm[g, b, :k, :k].numpy(), float(ge[g, b])) for g in range(gm.shape[0])]
        out.append(npo.combine_segments(p.delta, parts))
    return np.array(out)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    plist = [fx.random_params(rng, 6) for _ in range(3)]
    pr, lo, la = fx.random_obs_arrays(rng, 301)
    sh = ShardedLoglik(pr, lo, la, reduce_fn=oracle_reduce, fold_fn=oracle_fold)
    a, b = shard_bounds(pr.size, world)[rank]
    assert sh.n_local == b - a
    assert np.array_equal(sh.shard[1], lo[a:b])
    vals = sh.loglik_batch(plist)
    q.put((rank, vals.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fold_matches_whole_chain(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    plist = [fx.random_params(rng, 6) for _ in range(3)]
    pr, lo, la = fx.random_obs_arrays(rng, 301)
    want = [npo.forward_loglik_arrays(p, pr, lo, la, 1) for p in plist]
    for r in range(world):
        assert res[r] == res[0]          # every rank folds to the identical value
    np.testing.assert_allclose(res[0], want, rtol=1e-12)


def test_shard_bounds():
    assert shard_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        shard_bounds(2, 3)


def _replica_worker(rank, world, port, nprop, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(9)
    plist = [fx.random_params(rng, 4) for _ in range(nprop)]
    pr, lo, la = fx.random_obs_arrays(rng, 120)
    seen = []

    def eval_fn(ps):
        seen.extend(id(p) for p in ps)
        return np.array([npo.forward_loglik_arrays(p, pr, lo, la, 1) for p in ps])

    rep = ReplicaLoglik(pr, lo, la, eval_fn=eval_fn)
    vals = rep.loglik_batch(plist)
    mine = [i for i, p in enumerate(plist) if id(p) in seen]
    q.put((rank, vals.tolist(), mine))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nprop", [(2, 7), (3, 7), (3, 2)])
def test_replica_proposal_sharding(world, nprop):
    """Proposals split contiguously across ranks, each evaluated once, every
    rank returns all B values in order (including B < world)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, world, port, nprop, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (v, m) for r, v, m in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(9)
    plist = [fx.random_params(rng, 4) for _ in range(nprop)]
    pr, lo, la = fx.random_obs_arrays(rng, 120)
    want = [npo.forward_loglik_arrays(p, pr, lo, la, 1) for p in plist]
    owned = sorted(i for r in res for i in res[r][1])
    assert owned == list(range(nprop))  # every proposal evaluated exactly once
    for r in res:
        np.testing.assert_allclose(res[r][0], want, rtol=1e-12)
