"""Multi-GPU likelihood: one contiguous shard of the chain per GPU.

The chain product is associative and the reference already cuts it into
contiguous segments combined in order (reference engine.py:97-111,
292-318).  Across GPUs:

1. rank r holds only records ``segment_bounds(N, world)[r]`` in its HBM;
2. each rank reduces its shard to one scaled product node per proposal
   (``thmm_range_nodes``: K_p x K_p FP64 matrix + base-2 exponent);
3. the nodes are exchanged with one NCCL all-gather over NVLink
   ((K_p^2 + 1) doubles per proposal per rank: 8.2 KB at K=25, 51 KB at K=80);
4. every rank folds the G nodes in rank order against delta on its own GPU
   (``thmm_fold_nodes``), so all ranks return the identical value.

Torch is used only for the process group and the collective (plumbing).
The reduction and fold are pluggable so the host logic (bounds, gather
order, fold order) can be exercised with gloo on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from .engine import DeviceObservations, EngineConfig, fold_nodes, padded_states, segment_bounds


def shard_bounds(n: int, world: int):
    """Contiguous per-rank ranges; earlier ranks take the remainder."""
    if n < world:
        raise ValueError(f"cannot shard a chain of {n} records over {world} ranks")
    return segment_bounds(n, world)


class ShardedLoglik:
    """Likelihood of one chain sharded over the ranks of a process group.

    ``present, lon, lat`` may be the whole chain (each rank keeps only its
    shard) or, with ``local=True``, already this rank's shard.
    """

    def __init__(self, present, lon, lat, *, group=None, device: Optional[int] = None, local: bool = False,
                 total: Optional[int] = None, reduce_fn: Optional[Callable] = None,
                 fold_fn: Optional[Callable] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if local:
            self.n_total = int(total) if total is not None else None
            shard = (present, lon, lat)
        else:
            self.n_total = int(np.asarray(present).size)
            lo, hi = shard_bounds(self.n_total, self.world)[self.rank]
            shard = (present[lo:hi], lon[lo:hi], lat[lo:hi])
        self.n_local = int(np.asarray(shard[0]).size)
        self._reduce = reduce_fn
        self._fold = fold_fn
        self.device = device
        self.obs = None
        self.last_launches = 0
        self.last_profile = (0.0, 0.0, 0)
        if reduce_fn is None:
            self.obs = DeviceObservations(*shard, device=device)
            self.device = self.obs.device
        else:
            self.shard = shard

    def _torch_device(self):
        import torch

        return torch.device("cuda", self.device) if self._reduce is None else torch.device("cpu")

    def loglik_batch(self, params_list, cfg: EngineConfig = EngineConfig(), stream: int = 0) -> np.ndarray:
        import torch

        params_list = list(params_list)
        b = len(params_list)
        k = int(params_list[0].K)
        kp = padded_states(k)
        dev = self._torch_device()
        if self._reduce is None:
            m = torch.empty((b, kp, kp), dtype=torch.float64, device=dev)
            e = torch.empty((b,), dtype=torch.float64, device=dev)
            with torch.cuda.device(self.device):
                s = stream or torch.cuda.current_stream().cuda_stream
                self.obs.range_nodes(params_list, cfg, 0, 0, m.data_ptr(), e.data_ptr(), stream=s)
            from . import _native
            self.last_launches = _native.last_launch_count()
            self.last_profile = _native.profile_last()
        else:
            m, e = self._reduce(self.shard, params_list, cfg)
        # output concatenated along dim 0 (accepted by NCCL and gloo), viewed [G][B]
        gm = torch.empty((self.world * b, kp, kp), dtype=torch.float64, device=dev)
        ge = torch.empty((self.world * b,), dtype=torch.float64, device=dev)
        self.dist.all_gather_into_tensor(gm, m.contiguous(), group=self.group)
        self.dist.all_gather_into_tensor(ge, e.contiguous(), group=self.group)
        gm = gm.view(self.world, b, kp, kp)
        ge = ge.view(self.world, b)
        if self._fold is not None:
            return self._fold(params_list, gm, ge)
        with torch.cuda.device(self.device):
            s = stream or torch.cuda.current_stream().cuda_stream
            out = fold_nodes(params_list, gm.data_ptr(), ge.data_ptr(), self.world, self.device, stream=s,
                             raise_on_collapse=False)
        from . import _native
        self.last_launches += _native.last_launch_count()
        return out

    def loglik(self, params, cfg: EngineConfig = EngineConfig()) -> float:
        v = float(self.loglik_batch([params], cfg)[0])
        if not np.isfinite(v):
            raise RuntimeError("running state vector collapsed to zero while combining segments")
        return v

    def close(self):
        if self.obs is not None:
            self.obs.close()
