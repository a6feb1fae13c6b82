"""Pose-sharded multi-GPU rendering.

Poses are independent units: the reference guarantees ray and pose
independence (``SPEC.md:237``) and runs its population study as independent
registrations in parallel processes (``cli.py:133-145``, ``SPEC.md:407``).  So
the path shards over a batch of poses with no collective inside the render:

1. the CT is broadcast once from rank ``src`` (NCCL over NVLink on the GPU
   box, gloo in the CPU tests) -- :func:`broadcast_volume`;
2. every rank walks its contiguous block of the global pose batch
   (:func:`shard_range`);
3. the results go to the collecting rank ``dst`` through peer memory: ``dst``
   exports its output buffers once (:class:`PeerRows`, ``drr_peer_export``),
   every other rank opens them (``drr_peer_open``), and the kernels of each
   rank store their images / loss values / pose gradients straight into
   ``dst``'s HBM over NVLink -- the render and the gather are one kernel per
   rank, with no all-gather afterwards (:func:`gather_rows` is the NCCL
   all-gather this replaces, kept as the measured baseline);
4. one tiny stream-ordered all-reduce per call marks completion (and, at
   entry, that ``dst`` has finished with the previous call's rows).  A shared
   batched-registration loss would be the only data all-reduce
   (:func:`allreduce_sum`); the population study has none.

:class:`ShardedDRR` is the product entry point: ``render`` (C4: images
gathered), ``loss_and_gradient`` (C2 / C5: per-pose value and 7-gradient
gathered) and ``register_batch`` (the population study, traces gathered).
Under a world of one process every call is the single-GPU path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


def shard_range(n: int, rank: int, world: int):
    """Balanced contiguous block [start, stop) of n items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(int(n), world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def _world(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _global_rank(group, rank):
    return dist.get_global_rank(group, rank) if group is not None else rank


def broadcast_volume(vol: torch.Tensor | None, shape, device, dtype=torch.float32, src: int = 0,
                     group=None) -> torch.Tensor:
    """Every rank gets rank `src`'s volume (one collective, before any render)."""
    world, rank = _world(group)
    if world == 1:
        return vol.to(device=device, dtype=dtype)
    if rank == src:
        buf = vol.to(device=device, dtype=dtype).contiguous()
    else:
        buf = torch.empty(tuple(shape), device=device, dtype=dtype)
    dist.broadcast(buf, src=_global_rank(group, src), group=group)
    return buf


def gather_rows(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather per-pose rows (images (b, H, W) or gradients (b, k)) from
    uneven contiguous shards back into global order (n_total, ...).  The NCCL
    baseline of the peer-memory gather (:class:`PeerRows`)."""
    world, _ = _world(group)
    if world == 1:
        return local
    rows = [shard_range(n_total, r, world) for r in range(world)]
    cap = max(stop - start for start, stop in rows)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * cap,) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        dist.all_gather_into_tensor(out, pad, group=group)
        bufs = list(out.split(cap))
    else:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:stop - start] for b, (start, stop) in zip(bufs, rows)], dim=0)


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """Shared-loss reduction for batched registration (a few floats)."""
    if _world(group)[0] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def max_over_ranks(value: float, device, group=None) -> float:
    """Timing rule: report the slowest rank."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if _world(group)[0] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def rank_sync(device, group=None) -> None:
    """Stream-ordered rendezvous of all ranks: NCCL all-reduce of one int on the
    current stream (work issued after it waits for every rank's earlier work);
    other backends synchronise the device and barrier on the host."""
    world, _ = _world(group)
    if world == 1:
        return
    if dist.get_backend(group) == "nccl":
        flag = _sync_flag(device)
        dist.all_reduce(flag, group=group)
    else:
        if torch.device(device).type == "cuda":
            torch.cuda.synchronize(device)
        dist.barrier(group=group)


_FLAGS: dict = {}


def _sync_flag(device):
    key = str(device)
    if key not in _FLAGS:
        _FLAGS[key] = torch.zeros(1, dtype=torch.int32, device=device)
    return _FLAGS[key]


class PeerRows:
    """An (n_rows, *row_shape) buffer in rank ``dst``'s HBM that every rank's
    kernels can store into.

    ``dst`` allocates it and exports it (``drr_peer_export``); the handle goes
    to the other ranks over the process group once, and each opens it on its
    own device (``drr_peer_open``: a pointer valid for its kernels, peer access
    over NVLink).  ``ptr(row)`` is that rank's address of a global row.
    Collective: every rank of ``group`` constructs it with the same arguments.

    If any rank cannot open the handle (no peer access between its GPU and
    ``dst``'s, e.g. a launcher that hides the other GPUs from each process),
    every rank falls back to a local buffer for its own rows ``[lo, hi)`` and
    :meth:`collect` gathers them into ``dst``'s buffer with one NCCL
    all-gather (``mode == "collective"``; the peer path is ``"peer"``)."""

    def __init__(self, n_rows: int, row_shape, dtype, device, group=None, dst: int = 0,
                 shard=None):
        self.world, self.rank = _world(group)
        self.group, self.dst = group, dst
        self.n_rows = int(n_rows)
        self.row_shape = tuple(int(x) for x in row_shape)
        self.dtype = dtype
        self.device = torch.device(device)
        self.row_bytes = int(np.prod(self.row_shape, dtype=np.int64)) * torch.empty(
            (), dtype=dtype).element_size()
        self.lo, self.hi = shard if shard is not None else shard_range(self.n_rows, self.rank,
                                                                       self.world)
        self.buf = None
        self.local = None
        self._opened = None
        self.mode = "peer"
        self.row0 = 0  # global row at self.base
        lib = _lib.load()
        if self.rank == dst:
            self.buf = torch.empty((max(self.n_rows, 1),) + self.row_shape, dtype=dtype,
                                   device=self.device)
            self.base = self.buf.data_ptr()
        if self.world == 1:
            return
        forced = os.environ.get("DRR_PEER_MODE") == "collective"  # test knob
        ok = 0 if forced else 1
        if not forced:
            msg = [None]
            if self.rank == dst:
                h = _lib.DrrPeerHandle()
                _lib.check(lib.drr_peer_export(self.buf.data_ptr(), ctypes.byref(h)))
                msg = [bytes(h)]
            dist.broadcast_object_list(msg, src=_global_rank(group, dst), group=group)
            if self.rank != dst:
                h = _lib.DrrPeerHandle.from_buffer_copy(msg[0])
                p = ctypes.c_void_p()
                if lib.drr_peer_open(ctypes.byref(h), ctypes.byref(p)) == _lib.DRR_OK:
                    self.base = int(p.value)
                    self._opened = (self.base, int(h.offset))
                else:
                    ok = 0
            flag = torch.tensor([ok], dtype=torch.int32,
                                device=self.device if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            ok = int(flag.item())
        if ok == 0:
            self.close()
            self.mode = "collective"
            if self.rank != dst:
                self.local = torch.empty((max(self.hi - self.lo, 1),) + self.row_shape,
                                         dtype=dtype, device=self.device)
                self.base = self.local.data_ptr()
                self.row0 = self.lo

    def shard_view(self) -> torch.Tensor:
        """This rank's rows [lo, hi) as a tensor it may write (collective mode,
        or the collecting rank)."""
        if self.rank == self.dst:
            return self.buf[self.lo:self.hi]
        if self.local is None:
            raise RuntimeError("peer mode: this rank's rows live in the collecting rank's HBM")
        return self.local[:self.hi - self.lo]

    def ptr(self, row: int = 0) -> int:
        return self.base + (int(row) - self.row0) * self.row_bytes

    def collect(self) -> None:
        """Collective mode only: bring every rank's rows into ``dst``'s buffer."""
        if self.mode != "collective":
            return
        allrows = gather_rows(self.shard_view(), self.n_rows, self.group)
        if self.rank == self.dst:
            self.buf[:self.n_rows].copy_(allrows)

    def rows(self, n: int | None = None) -> torch.Tensor | None:
        """The buffer's first n rows on ``dst`` (None on the other ranks)."""
        if self.buf is None:
            return None
        return self.buf[: self.n_rows if n is None else n]

    def close(self) -> None:
        if self._opened is not None:
            _lib.check(_lib.load().drr_peer_close(ctypes.c_void_p(self._opened[0]),
                                                  self._opened[1]))
            self._opened = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


class ShardedDRR:
    """The C2/C4/C5 workloads and the population study over the ranks of a
    process group (one process per GPU), results collected on rank ``dst``.

    ``volume`` (nx, ny, nz), indexed like ``Volume.data``, is needed on rank
    ``src`` only; it is broadcast once, in the device's x-fastest fp32 layout.
    Every rank passes the same global pose batch to each call (the reference's
    population study also draws every initialisation from one seed,
    ``registration.py:128-147``) and walks its own ``shard_range``.
    Collective: all ranks call every method, in the same order.
    """

    def __init__(self, volume, spacing, sdr: float, height: int, delx: float,
                 width: int | None = None, dely: float | None = None,
                 origin=(0.0, 0.0, 0.0), device=None, group=None, src: int = 0,
                 dst: int = 0, ray_split: int = 0):
        from .renderer import Detector, DeviceVolume
        self.world, self.rank = _world(group)
        self.group, self.src, self.dst = group, src, dst
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        if self.rank == src:
            dv = DeviceVolume(volume, spacing, origin, device=self.device)
            meta = [dv.dims]
        else:
            meta = [None]
        if self.world > 1:
            dist.broadcast_object_list(meta, src=_global_rank(group, src), group=group)
        dims = tuple(meta[0])
        if self.rank != src:
            dv = DeviceVolume.empty(dims, spacing, origin, device=self.device)
        if self.world > 1:
            dist.broadcast(dv.flat, src=_global_rank(group, src), group=group)
        if self.rank != src:  # same data, so the same occupied box as rank src's
            dv.trim = True
            dv.refresh_bounds()
        self.volume = dv
        self.detector = Detector(height, width if width is not None else height, delx, dely,
                                 ray_split=ray_split)
        self.sdr = float(sdr)
        self._peer = {}
        self._bufs = {}

    def with_detector(self, detector) -> "ShardedDRR":
        """The same (already broadcast) volume with another detector."""
        other = ShardedDRR.__new__(ShardedDRR)
        other.__dict__.update(self.__dict__)
        other.detector = detector
        other._peer, other._bufs = {}, {}
        return other

    # ------------------------------------------------------------ plumbing
    def shard(self, n: int):
        return shard_range(n, self.rank, self.world)

    def _rows(self, name, n, row_shape, dtype):
        key = (name, n)
        if key not in self._peer:
            self._peer[key] = PeerRows(n, row_shape, dtype, self.device, self.group, self.dst)
        return self._peer[key]

    def _local_eta(self, eta):
        """This rank's rows of the global (n, 7) pose batch, on the device."""
        n = int(eta.shape[0])
        lo, hi = self.shard(n)
        if isinstance(eta, torch.Tensor):
            e = eta[lo:hi].to(self.device, torch.float64, non_blocking=True)
        else:
            e = torch.as_tensor(np.asarray(eta, dtype=np.float64)[lo:hi], device=self.device)
        return n, lo, e.contiguous()

    def _finish(self, out, copy, peers=()):
        for p in peers:
            p.collect()
        rank_sync(self.device, self.group)
        if self.rank != self.dst:
            return None
        return tuple(o.clone() for o in out) if copy else out

    # -------------------------------------------------------------- calls
    def pose_vectors(self, rotation, translation) -> np.ndarray:
        rot = np.asarray(rotation, dtype=np.float64).reshape(-1, 3)
        tra = np.asarray(translation, dtype=np.float64).reshape(-1, 3)
        return np.concatenate([np.full((rot.shape[0], 1), self.sdr), rot, tra], axis=1)

    def render(self, eta, copy: bool = True, sync_entry: bool = True):
        """(n, H, W) fp32 images of the global pose batch on ``dst`` (None on
        the other ranks): ``drr_pose_frames`` + ``drr_forward`` per rank, the
        forward kernel storing its image rows into ``dst``'s buffer."""
        from .registration import _iso
        n, lo, e = self._local_eta(eta)
        det = self.detector
        out = self._rows("img", n, (det.height, det.width), torch.float32)
        if sync_entry:
            rank_sync(self.device, self.group)  # dst is done with the previous rows
        b = e.shape[0]
        if b:
            lib = _lib.load()
            st = torch.cuda.current_stream(self.device).cuda_stream
            fr = self._buf("frames", (b, 12), torch.float64)
            _lib.check(lib.drr_pose_frames(e.data_ptr(), b, _iso(self.volume, None),
                                           fr.data_ptr(), st))
            for c0 in range(0, b, 65535):
                c1 = min(b, c0 + 65535)
                _lib.check(lib.drr_forward(self.volume.flat.data_ptr(), self.volume.vol_dtype,
                                           self.volume.grid, fr[c0:].data_ptr(), c1 - c0, det.c,
                                           out.ptr(lo + c0), 0, st))
        r = self._finish((out.rows(),), copy, (out,))
        return None if r is None else r[0]

    def loss_and_gradient(self, eta, fixed, loss_kind: str = "neg_zncc", copy: bool = True,
                          sync_entry: bool = True):
        """Batched ``gradients.loss_and_gradient`` (``gradients.py:61-69``) over
        the global pose batch: (value (n,), grad (n, 7)) on ``dst``.  Each rank
        runs the native chain on its shard; the loss kernel stores the values
        and the reduction kernel the gradients straight into ``dst``'s
        buffers."""
        from .registration import LOSS_KINDS, _launch_loss_grad, _prep_fixed, _Buffers, _iso
        n, lo, e = self._local_eta(eta)
        vals = self._rows("value", n, (), torch.float64)
        grads = self._rows("grad", n, (7,), torch.float64)
        if sync_entry:
            rank_sync(self.device, self.group)
        b = e.shape[0]
        if b:
            key = ("lg", b)
            if key not in self._bufs:
                self._bufs[key] = _Buffers(self.volume, self.detector, b)
            buf = self._bufs[key]
            fx = fixed
            if isinstance(fixed, torch.Tensor) and fixed.ndim == 3 and fixed.shape[0] == n and n > 1:
                fx = fixed[lo:lo + b]
            elif not isinstance(fixed, torch.Tensor):
                fa = np.asarray(fixed)
                fx = fa[lo:lo + b] if fa.ndim == 3 and fa.shape[0] == n and n > 1 else fa
            fixed_t, stride = _prep_fixed(fx, b, self.detector, self.device)
            lib = _lib.load()
            st = torch.cuda.current_stream(self.device).cuda_stream
            _launch_loss_grad(lib, self.volume, self.detector, _iso(self.volume, None), e,
                              fixed_t, stride, LOSS_KINDS[loss_kind], buf, st,
                              value_ptr=vals.ptr(lo), grad_eta_ptr=grads.ptr(lo),
                              grad_frames=False)
        return self._finish((vals.rows(), grads.rows()), copy, (vals, grads))

    def register_batch(self, fixed_images, poses0, config=None, use_graph: bool = True):
        """The population study (``cli.py:133-145``): ``len(poses0)`` independent
        registrations, each rank running its shard as one device-resident
        engine (one CUDA graph); the traces are collected on ``dst`` in global
        order (None on the other ranks)."""
        from .registration import RegistrationEngine
        poses0 = np.asarray(poses0, dtype=np.float64).reshape(-1, 7)
        n = poses0.shape[0]
        lo, hi = self.shard(n)
        fx = fixed_images
        fa = fx if isinstance(fx, torch.Tensor) else np.asarray(fx)
        if fa.ndim == 3 and fa.shape[0] == n and n > 1:
            fx = fa[lo:hi]
        traces = []
        if hi > lo:
            eng = RegistrationEngine(self.volume, self.detector, fx, hi - lo, config)
            eng.reset(poses0[lo:hi])
            eng.run(use_graph=use_graph)
            traces = eng.traces()
        if self.world == 1:
            return traces
        got = [None] * self.world if self.rank == self.dst else None
        dist.gather_object(traces, got, dst=_global_rank(self.group, self.dst), group=self.group)
        if self.rank != self.dst:
            return None
        return [t for part in got for t in part]

    def _buf(self, name, shape, dtype):
        key = (name, tuple(shape), dtype)
        if key not in self._bufs:
            self._bufs[key] = torch.empty(shape, dtype=dtype, device=self.device)
        return self._bufs[key]

    def close(self):
        for p in self._peer.values():
            p.close()
        self._peer.clear()


def init_from_env(backend: str | None = None):
    """torchrun convenience: one process per GPU (LOCAL_RANK), NCCL over
    NVLink; returns (rank, world, device)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        be = backend or "nccl"
        if be == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(be)
    return rank, world, dev


__all__ = ["shard_range", "broadcast_volume", "gather_rows", "allreduce_sum", "max_over_ranks",
           "rank_sync", "PeerRows", "ShardedDRR", "init_from_env"]
