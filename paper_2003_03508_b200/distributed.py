"""Multi-GPU likelihood: one contiguous shard of the chain per GPU.

The chain product is associative and the reference already cuts it into
contiguous segments combined in order (reference engine.py:97-111,
292-318).  Across GPUs:

1. rank r holds only records ``segment_bounds(N, world)[r]`` in its HBM;
2. each rank reduces its shard to one scaled product node per proposal
   (``thmm_range_nodes``: K_p x K_p FP64 matrix + base-2 exponent);
3. the nodes and exponents, packed in one block per rank, are exchanged with
   ONE NCCL all-gather over NVLink ((K_p^2 + 1) doubles per proposal per rank:
   8.2 KB at K=25, 51 KB at K=80), queued behind the range kernels on the
   same stream (no host synchronisation before the fold);
4. every rank folds the G nodes in rank order against delta on its own GPU
   (``thmm_fold_nodes``), so all ranks return the identical value.

Torch is used only for the process group and the collective (plumbing).
The reduction and fold are pluggable so the host logic (bounds, gather
order, fold order) can be exercised with gloo on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

from typing import Callable, Optional

import numpy as np

CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy

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
                 fold_fn: Optional[Callable] = None, transport: Optional[str] = None):
        import os

        import torch.distributed as dist

        # NCCL all-gather unless asked otherwise (argument, else THMM_TRANSPORT):
        # the peer-memory mailbox is opt-in ("peer", or "auto" = peer after a
        # bitwise check against NCCL on first use).
        if transport is None:
            transport = os.environ.get("THMM_TRANSPORT", "nccl")
        if transport not in ("auto", "peer", "nccl"):
            raise ValueError("transport must be 'auto', 'peer' or 'nccl'")
        self.transport = transport if reduce_fn is None else "nccl"
        self._peer = None        # native thmm_peer handle
        self._peer_slot = 0
        self._peer_checked = False
        self.transport_used = None
        self.combine_used = None
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

    # -- peer-memory transport (NVLink P2P stores + flags, thmm_peer_*) -------

    def _agree(self, ok: bool) -> bool:
        """All ranks agree (logical AND) -- a transport is used by all or none."""
        import torch

        dev = (torch.device("cuda", self.device) if self.dist.get_backend(self.group) == "nccl"
               else torch.device("cpu"))
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())

    def _peer_setup(self, slot: int) -> bool:
        import ctypes

        from . import _native as nat

        self._peer_close()
        handle = ctypes.create_string_buffer(64)
        peer = ctypes.c_void_p()
        err = nat.errbuf()
        try:
            ok = nat.lib().thmm_peer_create(int(self.device), self.rank, self.world, int(slot), ctypes.byref(peer),
                                            handle, err, len(err)) == nat.THMM_OK
        except Exception:  # pragma: no cover - defensive
            ok = False
        if not self._agree(ok):
            if ok:
                nat.lib().thmm_peer_destroy(peer)
            return False
        handles = [None] * self.world
        self.dist.all_gather_object(handles, handle.raw, group=self.group)
        blob = ctypes.create_string_buffer(b"".join(handles), 64 * self.world)
        ok = nat.lib().thmm_peer_open(peer, blob, err, len(err)) == nat.THMM_OK
        if not self._agree(ok):
            nat.lib().thmm_peer_destroy(peer)
            return False
        self._peer = peer
        self._peer_slot = int(slot)
        return True

    def _peer_close(self):
        if self._peer is not None:
            from . import _native as nat

            nat.lib().thmm_peer_destroy(self._peer)
            self._peer = None
            self._peer_slot = 0

    def _peer_loglik(self, params_list, cfg, s, host_shard):
        from . import _native as nat
        from .engine import _PackedParams, _auto_pin, _host_arrays, _native_config

        pp = _PackedParams(params_list)
        out = np.empty(pp.pack.B, dtype=np.float64)
        status = np.empty(pp.pack.B, dtype=np.int32)
        c = _native_config(cfg, 0, 0, s)
        err = nat.errbuf()
        if host_shard is not None:
            pr, lo, la = _host_arrays(*host_shard)
            _auto_pin(pr, lo, la)
            self._host_refs = (pr, lo, la)
            args = (nat.as_ptr(pr, nat.c_uint8), nat.as_ptr(lo, nat.c_double), nat.as_ptr(la, nat.c_double), pr.size)
        else:
            args = (None, None, None, 0)
        rc = nat.lib().thmm_peer_loglik(self._peer, self.obs._handle, *args, nat.ctypes.byref(pp.struct),
                                        nat.ctypes.byref(c), nat.as_ptr(out, nat.c_double),
                                        nat.as_ptr(status, nat.c_int32), err, len(err))
        if host_shard is not None:
            self.obs.n = int(args[3])
            self.n_local = int(args[3])
        if rc != nat.THMM_OK and rc != nat.THMM_ECOLLAPSE:
            nat.raise_for(rc, err)
        self.last_launches = nat.last_launch_count()
        self.last_profile = nat.profile_last()
        return out

    def _packed(self, b: int, kp: int, dev):
        """Per-rank block [B*KP*KP nodes | B exponents | pad to even] and the
        gathered [world][block] buffer, reused across calls of the same shape."""
        import torch

        key = (b, kp, str(dev))
        if getattr(self, "_buf_key", None) != key:
            blk = b * kp * kp + b + ((b * kp * kp + b) & 1)
            self._buf = torch.empty(blk, dtype=torch.float64, device=dev)
            self._gbuf = torch.empty(self.world * blk, dtype=torch.float64, device=dev)
            self._buf_key = key
        return self._buf, self._gbuf

    def loglik_batch(self, params_list, cfg: EngineConfig = EngineConfig(), stream: int = 0,
                     host_shard=None) -> np.ndarray:
        """One evaluation: shard nodes -> ONE all-gather of the packed
        (nodes | exponents) block -> ordered fold on every rank.  On the
        native path nothing synchronises the host before the fold's result
        read: the range kernels, the collective and the fold queue back to
        back on the launch stream.  ``host_shard=(present, lon, lat)``
        evaluates this rank's records from host memory (end-to-end
        evaluation): pinned arrays are read in place by the kernels over PCIe
        (zero-copy; the device copy is left as it was), pageable ones replace
        it with the copy pipelined against the chain."""
        import torch

        params_list = list(params_list)
        b = len(params_list)
        k = int(params_list[0].K)
        kp = padded_states(k)
        nd = b * kp * kp
        blk = nd + b + ((nd + b) & 1)  # even: every rank's block (node rows are read as double2) 16-B aligned
        if self.transport != "nccl" and self._reduce is None:
            s = stream or torch.cuda.current_stream(self.device).cuda_stream or CUDA_STREAM_LEGACY
            if blk > self._peer_slot and not self._peer_setup(blk):
                if self.transport == "peer":
                    raise RuntimeError("peer-memory transport unavailable on this process group")
                self.transport = "nccl"
            elif self._peer_checked:
                with torch.cuda.device(self.device):
                    out = self._peer_loglik(params_list, cfg, s, host_shard)
                self.transport_used = "peer"
                return out
            else:
                # First use: the peer result must equal the NCCL path's bitwise on
                # every rank (a peer that never publishes makes every rank's wait
                # time out, so failures are seen by all ranks alike).
                try:
                    with torch.cuda.device(self.device):
                        out = self._peer_loglik(params_list, cfg, s, host_shard)
                    ok = True
                except RuntimeError:
                    if self.transport == "peer":
                        raise
                    out, ok = None, False
                ref = self._nccl_loglik(params_list, cfg, stream, host_shard, b, kp, nd, blk)
                self._peer_checked = True
                if not self._agree(ok and bool(np.array_equal(out, ref))):
                    self._peer_close()
                    self.transport = "nccl"
                    self.transport_used = "nccl"
                    return ref
                self.transport_used = "peer"
                return out
        self.transport_used = "nccl"
        if self._reduce is None and cfg.precision == "float64" and cfg.segments is None:
            out = self._stitch_loglik(params_list, cfg, stream, host_shard, b, k, kp)
            if out is not None:
                self.combine_used = "stitched"
                return out
        self.combine_used = "nodes"
        return self._nccl_loglik(params_list, cfg, stream, host_shard, b, kp, nd, blk)

    # -- stitched combine (no K x K nodes; csrc/thmm_vec.cuh) -----------------

    def _stitch_ok(self, k: int, b: int) -> bool:
        """All ranks' shards long enough for the stitched chain (agreed once per (K, B))."""
        from . import _native as nat

        cache = self.__dict__.setdefault("_stitch_cache", {})
        key = (k, b, self.n_local)
        if key not in cache:
            mine = int(nat.lib().thmm_stitch_segments(self.obs._handle, k, b)) > 0
            cache[key] = self._agree(mine)
        return cache[key]

    def _stitch_loglik(self, params_list, cfg, stream, host_shard, b, k, kp):
        """One evaluation with the stitched combine: every rank reduces its
        shard to (final forward row, log-scale, flag) -- ONE all-gather of
        B (K_p + 2) doubles per rank -- then rank r links the previous rank's
        final row into its first segment -- ONE all-gather of 2 B doubles --
        and every rank sums the terms in rank order:
            log L = sum_r A_r + sum_{r>=1} link_r + log(w_{last} . 1).
        Returns None when the stitched path does not apply (the caller then
        exchanges nodes); a flagged link (did not converge) falls back the
        same way, on every rank alike."""
        import contextlib

        import torch

        from . import _native as nat
        from .engine import _PackedParams, _auto_pin, _host_arrays, _native_config

        staged = None
        if host_shard is not None:  # this rank's records from host memory
            pr, lo, la = _host_arrays(*host_shard)
            _auto_pin(pr, lo, la)
            if pr.size != self.n_local or self.obs.n != pr.size:
                self.obs.assign(pr, lo, la)  # new shard length: one synchronous copy, then the agreement below
            else:  # copied by DMA in time chunks under the main pass (thmm_stitch_shard_host)
                staged = (pr, lo, la)
                self._host_refs = staged  # alive until the stream has passed the copies
            self.n_local = int(pr.size)
        if not self._stitch_ok(k, b):
            if staged is not None:
                self.obs.assign(*staged)
            return None
        dev = torch.device("cuda", self.device)
        ctx = contextlib.nullcontext()
        with torch.cuda.device(self.device):
            if stream and torch.cuda.current_stream().cuda_stream != stream:
                ctx = torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev))
        with ctx, torch.cuda.device(self.device):
            s = torch.cuda.current_stream().cuda_stream or CUDA_STREAM_LEGACY
            pp = _PackedParams(params_list)
            c = _native_config(cfg, 0, 0, s)
            width = kp + 2
            key = (b, kp)
            if getattr(self, "_sbuf_key", None) != key:
                self._sblk = torch.empty(b * width, dtype=torch.float64, device=dev)
                self._sgblk = torch.empty(self.world * b * width, dtype=torch.float64, device=dev)
                self._slink = torch.zeros(2 * b, dtype=torch.float64, device=dev)
                self._sglink = torch.empty(self.world * 2 * b, dtype=torch.float64, device=dev)
                self._sbuf_key = key
            err = nat.errbuf()
            first = 1 if self.rank == 0 else 0
            if staged is not None:
                pr, lo, la = staged
                rc = nat.lib().thmm_stitch_shard_host(self.obs._handle, pr.ctypes.data, lo.ctypes.data, la.ctypes.data,
                                                      pr.size, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c), first,
                                                      self._sblk.data_ptr(), err, len(err))
            else:
                rc = nat.lib().thmm_stitch_shard(self.obs._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                                 first, self._sblk.data_ptr(), err, len(err))
            nat.raise_for(rc, err)
            launches = nat.last_launch_count()
            self._gather(self._sgblk, self._sblk)
            if self.rank > 0:
                prev = self._sgblk.data_ptr() + 8 * (self.rank - 1) * b * width
                rc = nat.lib().thmm_stitch_link(self.obs._handle, nat.ctypes.byref(pp.struct), nat.ctypes.byref(c),
                                                nat.c_void_p(prev), width, self._slink.data_ptr(), err, len(err))
                nat.raise_for(rc, err)
                launches += nat.last_launch_count()
            else:
                self._slink.zero_()
            self._gather(self._sglink, self._slink)
            g = self._sgblk.view(self.world, b, width).cpu().numpy()
            lk = self._sglink.view(self.world, b, 2).cpu().numpy()
        self.last_launches = launches
        nat.lib().thmm_profile_collect()  # the shard's events have passed (the gathers synchronised)
        self.last_profile = nat.profile_last()
        fail = (g[:, :, kp + 1] != 0).any(axis=0) | (lk[1:, :, 1] != 0).any(axis=0)
        if fail.any():
            return None
        acc = g[0, :, kp].copy()
        for r in range(1, self.world):  # rank order: identical on every rank
            acc = acc + g[r, :, kp] + lk[r, :, 0]
        tail = g[self.world - 1, :, :kp].sum(axis=1)
        with np.errstate(divide="ignore"):
            out = np.where(tail > 0, acc + np.log(tail), -np.inf)
        return out

    def _gather(self, out, inp):
        import torch

        if self.dist.get_backend(self.group) == "gloo":
            # gloo moves host tensors only (several ranks sharing one GPU in the tests)
            torch.cuda.synchronize(self.device)
            hg = torch.empty(out.numel(), dtype=torch.float64)
            self.dist.all_gather_into_tensor(hg, inp.cpu(), group=self.group)
            out.copy_(hg)
            torch.cuda.synchronize(self.device)
        else:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)

    def _nccl_loglik(self, params_list, cfg, stream, host_shard, b, kp, nd, blk):
        import contextlib

        import torch

        # The collective is ordered after torch's current stream: make the
        # caller's stream (if any) current so the range kernels, the all-gather
        # and the fold stay in one stream order.
        ctx = contextlib.nullcontext()
        if stream and self._reduce is None:
            with torch.cuda.device(self.device):
                if torch.cuda.current_stream().cuda_stream != stream:
                    ctx = torch.cuda.stream(torch.cuda.ExternalStream(stream, device=torch.device("cuda", self.device)))
        with ctx:
            return self._nccl_loglik_ordered(params_list, cfg, stream, host_shard, b, kp, nd, blk)

    def _nccl_loglik_ordered(self, params_list, cfg, stream, host_shard, b, kp, nd, blk):
        import torch

        dev = self._torch_device()
        buf, gbuf = self._packed(b, kp, dev)
        if self._reduce is None:
            from . import _native
            with torch.cuda.device(self.device):
                # The collective below is ordered after torch's current stream, so the
                # range kernels must be queued on that stream (the legacy default stream
                # is handle 0 in torch; passed as cudaStreamLegacy, not as "unset").
                s = stream or torch.cuda.current_stream().cuda_stream or CUDA_STREAM_LEGACY
                if host_shard is not None:  # new records for this rank, copy pipelined with the chain
                    self.obs.range_nodes_host(params_list, *host_shard, cfg, buf.data_ptr(),
                                              buf.data_ptr() + 8 * nd, stream=s)
                    self.n_local = int(np.asarray(host_shard[0]).size)
                else:
                    self.obs.range_nodes(params_list, cfg, 0, 0, buf.data_ptr(), buf.data_ptr() + 8 * nd,
                                         stream=s, sync=False)
            self.last_launches = _native.last_launch_count()
        else:
            m, e = self._reduce(self.shard, params_list, cfg)
            buf[:nd].copy_(m.reshape(-1))
            buf[nd:nd + b].copy_(e.reshape(-1))
        if self._reduce is None and self.dist.get_backend(self.group) == "gloo":
            # gloo moves host tensors only: several ranks sharing one GPU (the
            # multi-rank test of this path on a single-GPU box) stage via the host.
            torch.cuda.synchronize(self.device)  # the range kernels may run on the caller's stream
            hbuf = buf.cpu()
            hg = torch.empty(gbuf.numel(), dtype=torch.float64)
            self.dist.all_gather_into_tensor(hg, hbuf, group=self.group)
            gbuf.copy_(hg)
            torch.cuda.synchronize(self.device)
        else:
            self.dist.all_gather_into_tensor(gbuf, buf, group=self.group)
        if self._fold is not None:
            g2 = gbuf.view(self.world, blk)
            return self._fold(params_list, g2[:, :nd].reshape(self.world, b, kp, kp), g2[:, nd:nd + b])
        from . import _native
        with torch.cuda.device(self.device):
            s = stream or torch.cuda.current_stream().cuda_stream or CUDA_STREAM_LEGACY
            out = fold_nodes(params_list, gbuf.data_ptr(), gbuf.data_ptr() + 8 * nd, self.world, self.device,
                             stream=s, raise_on_collapse=False, m_stride_g=blk, e_stride_g=blk)
        self.last_launches += _native.last_launch_count()
        self.last_profile = _native.profile_last()
        return out

    def loglik(self, params, cfg: EngineConfig = EngineConfig()) -> float:
        v = float(self.loglik_batch([params], cfg)[0])
        if not np.isfinite(v):
            raise RuntimeError("running state vector collapsed to zero while combining segments")
        return v

    def close(self):
        self._peer_close()
        if self.obs is not None:
            self.obs.close()


class ReplicaLoglik:
    """Batched proposals sharded across ranks ("replicas").

    Every rank holds the WHOLE observation stream and evaluates its
    contiguous slice ``segment_bounds(B, world)[rank]`` of the B proposals in
    one launch; the B log-likelihoods are then exchanged with ONE all-gather
    (B doubles in total, padded to the largest slice) so every rank returns
    all B values in proposal order.  Compared with ``ShardedLoglik`` (one
    chain cut across the GPUs, B·(K_p²+1) doubles exchanged and folded) this
    is the natural layout for the many-chain MCMC driver: ``mcmc.run_chains``
    accepts it in place of a ``DeviceObservations`` (every rank draws the same
    proposals from the same seed, evaluates its slice, and gets all values
    back, so the accept decisions agree on every rank).

    ``eval_fn(params_slice) -> np.ndarray`` replaces the device evaluation
    (host-logic tests over gloo on CPU).
    """

    def __init__(self, present, lon, lat, *, group=None, device: Optional[int] = None,
                 eval_fn: Optional[Callable] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._eval = eval_fn
        self.obs = None
        self.device = device
        self.last_launches = 0
        if eval_fn is None:
            self.obs = DeviceObservations(present, lon, lat, device=device)
            self.device = self.obs.device
        self.n = int(np.asarray(present).size)

    def loglik_batch(self, params_list, cfg: EngineConfig = EngineConfig(), stream: int = 0,
                     host=None) -> np.ndarray:
        """All B log-likelihoods (collapsed proposals: -inf).  ``host=(present,
        lon, lat)`` replaces the stream from host memory first, the copy
        pipelined against this rank's chain kernels (end-to-end evaluation)."""
        import torch

        from .model import ParamPack

        packed = isinstance(params_list, ParamPack)  # pre-packed batch (mcmc.run_chains, proposals.py)
        if not packed:
            params_list = list(params_list)
        b = len(params_list)
        bounds = segment_bounds(b, self.world) if b >= self.world else \
            [(min(r, b), min(r + 1, b)) for r in range(self.world)]
        lo, hi = bounds[self.rank]
        width = max(h - l for l, h in bounds)
        mine = np.full(width, np.nan)
        if hi > lo:
            part = params_list.slice(lo, hi) if packed else params_list[lo:hi]
            if self._eval is not None:
                mine[:hi - lo] = self._eval(part)
            elif host is not None:
                mine[:hi - lo] = self.obs.loglik_host_batch(part, *host, cfg, stream=stream, mapped=True)
            else:
                mine[:hi - lo] = self.obs.loglik_batch(part, cfg, stream=stream)
                from . import _native
                self.last_launches = _native.last_launch_count()
        backend = self.dist.get_backend(self.group)
        dev = torch.device("cuda", self.device) if (backend == "nccl" and self._eval is None) else torch.device("cpu")
        t = torch.from_numpy(mine).to(dev)
        g = torch.empty(self.world * width, dtype=torch.float64, device=dev)
        self.dist.all_gather_into_tensor(g, t, group=self.group)
        g = g.view(self.world, width).cpu().numpy()
        return np.concatenate([g[r, :h - l] for r, (l, h) in enumerate(bounds)])

    def close(self):
        if self.obs is not None:
            self.obs.close()
