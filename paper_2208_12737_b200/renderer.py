"""The drop-in north-star API: ``DRR(volume, spacing, sdr, height, delx)``.

``DRR`` is an ``nn.Module`` whose ``forward(rotation, translation)`` returns a
differentiable (B, H, W) float32 image.  It is the batched, device-resident
equivalent of the reference's ``render`` / ``render_with_gradient`` /
``loss_and_gradient`` chain (``raytrace.py:132-142``, ``gradients.py:45-69``):

* ``rotation`` = (theta, phi, gamma) radians and ``translation`` = the shift
  (bx, by, bz) in mm relative to the isocentre (``geometry.py:24,142-143``);
* ``sdr`` is rho, half the source-detector distance (``PAPER.md:144``);
* ``delx`` (and ``dely``) is the pixel pitch; the isocentre is the volume
  centre (``DetectorSpec.for_volume``, ``geometry.py:94-97``);
* the volume is indexed [i, j, k] = (x, y, z) like ``Volume.data`` and kept
  on the device as float32 in the reference's x-fastest flat layout
  (``volume.py:77-79``).

With a gradient requested, the image and every ray's endpoint Jacobian come
from one walk (``drr_forward_jac``) and backward is a walk-free contraction
(``drr_backward_jac``); without one, ``drr_forward`` alone runs.  The pose ->
frame map and its gradient are ``drr_pose_frames`` / ``drr_pose_grad``
(``geometry.pose_frames`` is the same map as torch ops, used on the host side).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError
from .geometry import (canonical_sdr_to_rho, check_gimbal, check_pose_vectors, pose_frames,
                       volume_center)


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise InvalidArgumentError(f"{name} must be a CUDA tensor (no CPU fallback)")


_SRC_CODES = {torch.float32: _lib.DRR_SRC_F32, torch.float64: _lib.DRR_SRC_F64,
              torch.int16: _lib.DRR_SRC_I16, torch.uint8: _lib.DRR_SRC_U8}


def pack_volume(src: torch.Tensor, dims, order: int, dtype=torch.float32,
                clamp_negative: bool = False) -> torch.Tensor:
    """``drr_volume_pack``: a device tensor holding the volume in ``order``
    (``DRR_ORDER_XFASTEST`` flat, or ``DRR_ORDER_ZFASTEST`` = a C-ordered
    (nx, ny, nz) array) -> the walk's x-fastest flat layout in ``dtype``, cast
    (and clamped) in the same pass."""
    import ctypes
    _require_cuda(src, "volume")
    if src.dtype not in _SRC_CODES:
        src = src.to(torch.float64)
    src = src.contiguous()
    n = [int(x) for x in dims]
    out = torch.empty(n[0] * n[1] * n[2], dtype=dtype, device=src.device)
    d = (ctypes.c_int64 * 3)(*n)
    _lib.check(_lib.load().drr_volume_pack(
        src.data_ptr(), _SRC_CODES[src.dtype], order, d, 1 if clamp_negative else 0,
        out.data_ptr(), _lib.DRR_VOL_F32 if dtype == torch.float32 else _lib.DRR_VOL_F64,
        _stream_ptr(src.device)))
    return out


def volume_bounds(flat: torch.Tensor, grid, vol_dtype: int, hull: bool = False):
    """``drr_volume_bounds``: ((lo0, lo1, lo2), (hi0, hi1, hi2)), the voxel box
    outside of which the device volume is exactly zero; with ``hull`` also
    ``drr_volume_hull``'s (lo[n], hi[n]) (None for an all-zero volume).
    One sync."""
    out = torch.empty(6 + 32, dtype=torch.int32, device=flat.device)
    lib = _lib.load()
    _lib.check(lib.drr_volume_bounds(flat.data_ptr(), vol_dtype, grid, out.data_ptr(),
                                     _stream_ptr(flat.device)))
    if hull:
        _lib.check(lib.drr_volume_hull(flat.data_ptr(), vol_dtype, grid, out[6:].data_ptr(),
                                       _stream_ptr(flat.device)))
    b = [int(x) for x in out.cpu().tolist()]
    box = (tuple(b[:3]), tuple(b[3:6]))
    if not hull:
        return box
    nd = lib.drr_volume_hull_dirs()
    empty = box == ((0, 0, 0), (0, 0, 0))
    return box, (None if empty else (tuple(b[6:6 + nd]), tuple(b[22:22 + nd])))


def trim_grid(flat: torch.Tensor, dims, spacing, origin, vol_dtype: int, trim=True):
    """(grid, occupied box, hull) for a device volume: ``trim`` True = the box
    and the 14-direction hull, "box" = the box only, False = the whole volume."""
    grid = _lib.make_grid(dims, spacing, origin)
    if not trim or flat.numel() == 0:
        return grid, None, None
    box, hull = volume_bounds(flat, grid, vol_dtype, hull=True)
    if trim == "box":
        hull = None
    return _lib.make_grid(dims, spacing, origin, box, hull), box, hull


class DeviceVolume:
    """A CT volume resident in HBM: float32, x-fastest, plus its grid.

    ``trim`` (default True): the grid carries the volume's occupied box and
    hull (:func:`volume_bounds`); every ray is walked only between where it
    enters and leaves them, so the exactly-zero margins are skipped --
    bit-identical results, fewer voxel-steps.  ``trim="box"`` keeps the box
    only, ``False`` walks the whole volume.  Call ``refresh_bounds`` after
    writing into ``flat``."""

    def __init__(self, data, spacing, origin=(0.0, 0.0, 0.0), device=None,
                 dtype=torch.float32, trim=True):
        spacing = tuple(float(s) for s in np.broadcast_to(np.asarray(spacing, dtype=np.float64), (3,)))
        origin = tuple(float(s) for s in np.broadcast_to(np.asarray(origin, dtype=np.float64), (3,)))
        if isinstance(data, torch.Tensor):
            t = data.detach()
        else:
            arr = np.asarray(data)
            t = torch.as_tensor(arr if arr.flags.writeable else arr.copy())
        if t.ndim != 3:
            raise InvalidArgumentError(f"volume must be 3-D (nx, ny, nz), got shape {tuple(t.shape)}")
        if any(n < 1 for n in t.shape):
            raise InvalidArgumentError(f"dims must be >= 1, got {tuple(t.shape)}")
        if any(not (s > 0 and np.isfinite(s)) for s in spacing):
            raise InvalidArgumentError(f"spacing must be three positive reals, got {spacing}")
        device = torch.device(device) if device is not None else torch.device("cuda")
        self.dims = tuple(int(n) for n in t.shape)
        self.spacing = spacing
        self.origin = origin
        self.dtype = dtype
        # [i, j, k] (C order: z fastest) -> the x-fastest flat layout, on the device
        self.flat = pack_volume(t.to(device), self.dims, _lib.DRR_ORDER_ZFASTEST, dtype)
        self.vol_dtype = _lib.DRR_VOL_F32 if dtype == torch.float32 else _lib.DRR_VOL_F64
        self.trim = trim
        self.refresh_bounds()

    def refresh_bounds(self):
        """(Re)compute the grid: with ``trim``, the occupied box (and hull) of ``flat``."""
        self.grid, self.occupied, self.hull = trim_grid(
            self.flat, self.dims, self.spacing, self.origin, self.vol_dtype,
            getattr(self, "trim", False))
        return self

    @property
    def full_grid(self):
        """The grid without the occupied box (the reference's whole-volume walk)."""
        return _lib.make_grid(self.dims, self.spacing, self.origin)

    @classmethod
    def from_flat(cls, flat, dims, spacing, origin=(0.0, 0.0, 0.0), device=None,
                  dtype=torch.float32, clamp_negative: bool = False, trim=True):
        """From an x-fastest flat array (the reference's ``flat_data()``, .dvol /
        raw payloads): uploaded as-is, cast (and clamped) by drr_volume_pack."""
        dims = tuple(int(n) for n in dims)
        if isinstance(flat, torch.Tensor):
            src = flat.detach().reshape(-1)
        else:
            arr = np.asarray(flat).reshape(-1)
            src = torch.as_tensor(arr if arr.flags.writeable else arr.copy())
        if src.numel() != int(np.prod(dims)):
            raise InvalidArgumentError(
                f"data has {src.numel()} values, expected {int(np.prod(dims))} for dims {dims}")
        self = cls.empty(dims, spacing, origin, device=device, dtype=dtype, allocate=False)
        self.flat = pack_volume(src.to(self.flat.device), dims, _lib.DRR_ORDER_XFASTEST, dtype,
                                clamp_negative)
        self.trim = trim
        return self.refresh_bounds()

    @classmethod
    def empty(cls, dims, spacing, origin=(0.0, 0.0, 0.0), device=None, dtype=torch.float32,
              allocate: bool = True):
        """Uninitialised device volume of the given dims (filled by the caller,
        e.g. a broadcast of another rank's ``flat``)."""
        self = cls.__new__(cls)
        self.dims = tuple(int(n) for n in dims)
        self.spacing = tuple(float(s) for s in np.broadcast_to(np.asarray(spacing, np.float64), (3,)))
        self.origin = tuple(float(s) for s in np.broadcast_to(np.asarray(origin, np.float64), (3,)))
        if len(self.dims) != 3 or any(n < 1 for n in self.dims):
            raise InvalidArgumentError(f"dims must be three integers >= 1, got {self.dims}")
        if any(not (s > 0 and np.isfinite(s)) for s in self.spacing):
            raise InvalidArgumentError(f"spacing must be three positive reals, got {self.spacing}")
        if any(not np.isfinite(b) for b in self.origin):
            raise InvalidArgumentError(f"plane_origin must be finite, got {self.origin}")
        self.dtype = dtype
        device = torch.device(device) if device is not None else torch.device("cuda")
        self.flat = (torch.empty(int(np.prod(self.dims)), dtype=dtype, device=device)
                     if allocate else torch.empty(0, dtype=dtype, device=device))
        self.vol_dtype = _lib.DRR_VOL_F32 if dtype == torch.float32 else _lib.DRR_VOL_F64
        self.trim = False  # contents unknown until filled: refresh_bounds(trim) then
        self.occupied = None
        self.hull = None
        self.grid = _lib.make_grid(self.dims, self.spacing, self.origin)
        return self

    @property
    def center(self):
        return volume_center(self.dims, self.spacing, self.origin)

    @property
    def device(self):
        return self.flat.device


class Detector:
    """H x W detector with pitch (x along W, y along H), geometry.py:71-97.

    ``ray_split`` = threads per ray in the kernels: 1 walks each ray in one
    thread (sums bit-identical to the reference's sequential accumulation);
    2/4/8 cut rays at dominant-axis crossings (same segments, ~1e-16 relative
    summation-order differences); 0 = auto (split only when the batch has too
    few rays to fill the GPU, e.g. a single pose)."""

    def __init__(self, height: int, width: int, pitch_x: float, pitch_y: float | None = None,
                 ray_split: int = 0):
        pitch_y = pitch_x if pitch_y is None else pitch_y
        if int(height) < 1 or int(width) < 1:
            raise InvalidArgumentError(f"detector must be at least 1x1, got {height}x{width}")
        if not (pitch_x > 0 and pitch_y > 0 and np.isfinite(pitch_x) and np.isfinite(pitch_y)):
            raise InvalidArgumentError(f"pixel pitch must be positive, got {(pitch_x, pitch_y)}")
        if int(ray_split) not in (0, 1, 2, 4, 8):
            raise InvalidArgumentError(f"ray_split must be 0, 1, 2, 4 or 8, got {ray_split}")
        self.height, self.width = int(height), int(width)
        self.pitch_x, self.pitch_y = float(pitch_x), float(pitch_y)
        self.ray_split = int(ray_split)
        self.c = _lib.make_detector(self.height, self.width, self.pitch_x, self.pitch_y,
                                    self.ray_split)


# One launch covers at most this many poses (the grid's z extent); larger
# batches are split into launches of this size (rays are independent, so the
# split does not change any result).
MAX_POSES_PER_LAUNCH = 65535


def _pose_chunks(B: int):
    for lo in range(0, B, MAX_POSES_PER_LAUNCH):
        yield lo, min(B, lo + MAX_POSES_PER_LAUNCH)


def render_frames(vol: DeviceVolume, det: Detector, frames: torch.Tensor,
                  out_dtype=torch.float32) -> torch.Tensor:
    """(B, 12) float64 frames -> (B, H, W) images via ``drr_forward``."""
    _require_cuda(frames, "frames")
    frames = frames.detach().to(torch.float64).contiguous()
    B = frames.shape[0]
    img = torch.empty((B, det.height, det.width), dtype=out_dtype, device=frames.device)
    lib = _lib.load()
    for lo, hi in _pose_chunks(B):
        _lib.check(lib.drr_forward(vol.flat.data_ptr(), vol.vol_dtype, vol.grid,
                                   frames[lo:hi].data_ptr(), hi - lo, det.c, img[lo:hi].data_ptr(),
                                   1 if out_dtype == torch.float64 else 0,
                                   _stream_ptr(frames.device)))
    return img


def backward_frames(vol: DeviceVolume, det: Detector, frames: torch.Tensor,
                    grad_img: torch.Tensor, want_image: bool = False):
    """dL/d(frame) (B, 12) float64 for an upstream (B, H, W) pixel gradient."""
    frames = frames.detach().to(torch.float64).contiguous()
    if grad_img.dtype not in (torch.float32, torch.float64):
        grad_img = grad_img.to(torch.float32)
    grad_img = grad_img.contiguous()
    B = frames.shape[0]
    lib = _lib.load()
    ws_bytes = lib.drr_backward_workspace_size(min(B, MAX_POSES_PER_LAUNCH), det.c)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=frames.device)
    grad_frames = torch.empty((B, 12), dtype=torch.float64, device=frames.device)
    img = None
    if want_image:
        img = torch.empty((B, det.height, det.width), dtype=torch.float32, device=frames.device)
    for lo, hi in _pose_chunks(B):
        _lib.check(lib.drr_backward(
            vol.flat.data_ptr(), vol.vol_dtype, vol.grid, frames[lo:hi].data_ptr(), hi - lo, det.c,
            grad_img[lo:hi].data_ptr(), 1 if grad_img.dtype == torch.float64 else 0,
            grad_frames[lo:hi].data_ptr(), img[lo:hi].data_ptr() if img is not None else None, 0,
            ws.data_ptr(), ws_bytes, _stream_ptr(frames.device)))
    return (grad_frames, img) if want_image else grad_frames


def jac_bytes(det: Detector, n_poses: int) -> int:
    """Bytes of the stored ray Jacobian for n_poses (6 float64 per pixel)."""
    return 6 * 8 * int(n_poses) * det.height * det.width


def render_frames_jac(vol: DeviceVolume, det: Detector, frames: torch.Tensor,
                      out_dtype=torch.float32):
    """Image (B, H, W) plus the per-ray Jacobian (6, B*H*W) float64 from ONE
    walk (``drr_forward_jac``); :func:`backward_from_jac` turns it into dL/dframe.
    One launch: B <= MAX_POSES_PER_LAUNCH."""
    _require_cuda(frames, "frames")
    frames = frames.detach().to(torch.float64).contiguous()
    B = frames.shape[0]
    img = torch.empty((B, det.height, det.width), dtype=out_dtype, device=frames.device)
    jac = torch.empty((6, B * det.height * det.width), dtype=torch.float64, device=frames.device)
    lib = _lib.load()
    _lib.check(lib.drr_forward_jac(vol.flat.data_ptr(), vol.vol_dtype, vol.grid, frames.data_ptr(),
                                   B, det.c, img.data_ptr(),
                                   1 if out_dtype == torch.float64 else 0, jac.data_ptr(),
                                   _stream_ptr(frames.device)))
    return img, jac


def backward_from_jac(det: Detector, jac: torch.Tensor, grad_img: torch.Tensor) -> torch.Tensor:
    """dL/d(frame) (B, 12) from a stored ray Jacobian (``drr_backward_jac``, no walk)."""
    if grad_img.dtype not in (torch.float32, torch.float64):
        grad_img = grad_img.to(torch.float32)
    grad_img = grad_img.contiguous()
    B = grad_img.shape[0]
    lib = _lib.load()
    ws_bytes = lib.drr_backward_workspace_size(B, det.c)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=grad_img.device)
    grad_frames = torch.empty((B, 12), dtype=torch.float64, device=grad_img.device)
    _lib.check(lib.drr_backward_jac(jac.data_ptr(), B, det.c, grad_img.data_ptr(),
                                    1 if grad_img.dtype == torch.float64 else 0,
                                    grad_frames.data_ptr(), ws.data_ptr(), ws_bytes,
                                    _stream_ptr(grad_img.device)))
    return grad_frames


def count_steps(vol: DeviceVolume, det: Detector, frames: torch.Tensor,
                full: bool = False) -> torch.Tensor:
    """Used voxel-steps per ray (B, H, W) int32 (python_ref.ray_structure's `use`).
    ``full``: of the reference's whole-volume walk (SURVEY 8(d)'s S), else of
    the walk the kernels take (the occupied box only)."""
    frames = frames.detach().to(torch.float64).contiguous()
    B = frames.shape[0]
    steps = torch.empty((B, det.height, det.width), dtype=torch.int32, device=frames.device)
    lib = _lib.load()
    grid = vol.full_grid if full else vol.grid
    for lo, hi in _pose_chunks(B):
        _lib.check(lib.drr_count_steps(vol.flat.data_ptr(), vol.vol_dtype, grid,
                                       frames[lo:hi].data_ptr(), hi - lo, det.c,
                                       steps[lo:hi].data_ptr(), _stream_ptr(frames.device)))
    return steps


# Above this many bytes of stored ray Jacobian, autograd re-walks the rays in
# backward instead (drr_backward) and batched loss_and_gradient takes the fused
# walk.  8 GiB (4.4% of a B200's HBM) keeps C5 (64 poses at 1024^2: 3.2 GB) on
# the stored-Jacobian chain: 53.9 ms vs 56.6 for the fused walk
# (scripts/c5_modes.py, profiles/r02/SUMMARY.md).
JAC_BUDGET_BYTES = 8 << 30


class _RenderFrames(torch.autograd.Function):
    """frames (B, 12) -> image (B, H, W).

    When a gradient is needed, forward is ``drr_forward_jac`` (one walk: image
    plus per-ray Jacobian) and backward the walk-free ``drr_backward_jac``;
    above ``JAC_BUDGET_BYTES`` (or one launch's pose limit) forward is
    ``drr_forward`` and backward the fused re-walk ``drr_backward``."""

    @staticmethod
    def forward(ctx, frames, vol, det):
        ctx.vol, ctx.det = vol, det
        if (ctx.needs_input_grad[0] and frames.shape[0] <= MAX_POSES_PER_LAUNCH
                and jac_bytes(det, frames.shape[0]) <= JAC_BUDGET_BYTES):
            img, jac = render_frames_jac(vol, det, frames)
            ctx.save_for_backward(frames, jac)
            return img
        ctx.save_for_backward(frames)
        return render_frames(vol, det, frames)

    @staticmethod
    def backward(ctx, grad_img):
        saved = ctx.saved_tensors
        frames = saved[0]
        if len(saved) == 2:
            grad_frames = backward_from_jac(ctx.det, saved[1], grad_img)
        else:
            grad_frames = backward_frames(ctx.vol, ctx.det, frames, grad_img)
        return grad_frames.to(frames.dtype), None, None


class _PoseFrames(torch.autograd.Function):
    """(B, 7) pose vectors -> (B, 12) frames with ``drr_pose_frames``; backward
    is ``drr_pose_grad`` (dL/dframe -> dL/deta).  Two launches instead of the
    ~60 small torch ops of ``geometry.pose_frames``, the same map
    (``geometry.py:120-149``)."""

    @staticmethod
    def forward(ctx, eta, isocenter):
        import ctypes
        eta = eta.detach().to(torch.float64).contiguous()
        B = eta.shape[0]
        frames = torch.empty((B, 12), dtype=torch.float64, device=eta.device)
        iso = (ctypes.c_double * 3)(*isocenter)
        lib = _lib.load()
        _lib.check(lib.drr_pose_frames(eta.data_ptr(), B, iso, frames.data_ptr(),
                                       _stream_ptr(eta.device)))
        ctx.save_for_backward(eta)
        return frames

    @staticmethod
    def backward(ctx, grad_frames):
        (eta,) = ctx.saved_tensors
        B = eta.shape[0]
        grad_frames = grad_frames.to(torch.float64).contiguous()
        grad_eta = torch.empty((B, 7), dtype=torch.float64, device=eta.device)
        lib = _lib.load()
        _lib.check(lib.drr_pose_grad(eta.data_ptr(), grad_frames.data_ptr(), B,
                                     grad_eta.data_ptr(), _stream_ptr(eta.device)))
        return grad_eta, None


def render_pose_vectors(vol: DeviceVolume, det: Detector, eta: torch.Tensor,
                        isocenter=None) -> torch.Tensor:
    """Differentiable render of (B, 7) pose vectors (rho, theta, phi, gamma, shift)."""
    iso = vol.center if isocenter is None else isocenter
    frames = pose_frames(eta.to(torch.float64), iso)
    return _RenderFrames.apply(frames, vol, det)


class DRR(torch.nn.Module):
    """Differentiable DRR renderer: ``DRR(volume, spacing, sdr, height, delx)``.

    ``forward(rotation, translation)`` takes (B, 3) or (3,) tensors and returns
    (B, H, W) or (H, W) float32 images.  Gradients flow to rotation,
    translation and (if given as a tensor to ``forward``) ``sdr``.
    ``strict=True`` keeps the reference's validation (finite poses, and the
    |sin phi| > 1e-6 gimbal guard when a gradient is requested,
    ``gradients.py:39-42``); it synchronises with the device, so latency-bound
    loops (and CUDA-graph capture) pass ``strict=False``.
    """

    def __init__(self, volume, spacing, sdr: float, height: int, delx: float,
                 width: int | None = None, dely: float | None = None,
                 origin=(0.0, 0.0, 0.0), isocenter=None, device=None,
                 strict: bool = True, ray_split: int = 0):
        super().__init__()
        self.volume = DeviceVolume(volume, spacing, origin, device=device)
        self.detector = Detector(height, width if width is not None else height, delx, dely,
                                 ray_split=ray_split)
        self.sdr = canonical_sdr_to_rho(float(sdr))
        self.isocenter = tuple(self.volume.center if isocenter is None else
                               (float(v) for v in isocenter))
        self.strict = strict

    @classmethod
    def from_device_volume(cls, volume: DeviceVolume, sdr: float, detector: Detector,
                           isocenter=None, strict: bool = True) -> "DRR":
        """A module over an already resident volume (e.g. one broadcast by
        distributed.ShardedDRR): no upload, no copy."""
        self = cls.__new__(cls)
        torch.nn.Module.__init__(self)
        self.volume, self.detector = volume, detector
        self.sdr = canonical_sdr_to_rho(float(sdr))
        self.isocenter = tuple(volume.center if isocenter is None else
                               (float(v) for v in isocenter))
        self.strict = strict
        return self

    @property
    def height(self):
        return self.detector.height

    @property
    def width(self):
        return self.detector.width

    def pose_vectors(self, rotation, translation, sdr=None) -> torch.Tensor:
        dev = self.volume.device
        rot = torch.as_tensor(rotation, device=dev)
        tra = torch.as_tensor(translation, device=dev)
        if rot.ndim == 1:
            rot = rot[None]
        if tra.ndim == 1:
            tra = tra[None]
        if rot.shape[-1] != 3 or tra.shape[-1] != 3 or rot.shape[0] != tra.shape[0]:
            raise InvalidArgumentError(
                f"rotation/translation must be (B, 3), got {tuple(rot.shape)} / {tuple(tra.shape)}")
        rot = rot.to(torch.float64)
        tra = tra.to(torch.float64)
        if sdr is None:
            rho = torch.full((rot.shape[0], 1), self.sdr, dtype=torch.float64, device=dev)
        else:
            rho = torch.as_tensor(sdr, device=dev).to(torch.float64).reshape(-1, 1)
            rho = rho.expand(rot.shape[0], 1)
        return torch.cat([rho, rot, tra], dim=1)

    def forward(self, rotation, translation, sdr=None):
        single = torch.as_tensor(rotation).ndim == 1
        eta = self.pose_vectors(rotation, translation, sdr)
        if self.strict:
            check_pose_vectors(eta.detach())
            if torch.is_grad_enabled() and eta.requires_grad:
                check_gimbal(eta.detach())
        frames = _PoseFrames.apply(eta, self.isocenter)
        img = _RenderFrames.apply(frames, self.volume, self.detector)
        return img[0] if single else img
