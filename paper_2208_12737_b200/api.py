"""drrtrace-compatible functional API on the GPU path.

The reference's public functions for this path, with its argument meaning,
types and errors, so a caller can switch ``import drrtrace as dt`` to
``from paper_2208_12737_b200 import api as dt``:

* ``render`` / ``render_iterative`` (``raytrace.py:132-152``) -> ``Image``;
* ``render_with_gradient`` (``gradients.py:45-58``) -> ``(Image, d_image)``
  with ``d_image`` (H, W, 7) against (rho, theta, phi, gamma, bx, by, bz);
* ``loss_and_gradient`` (``gradients.py:61-69``) -> ``GradientRecord``;
* ``register`` (``registration.py:89-125``) -> ``RegistrationTrace``.

``Volume``, ``PoseParameters``, ``DetectorSpec``, ``Image`` and
``GradientRecord`` mirror the reference's dataclasses (``volume.py:24-83``,
``geometry.py:32-97``, ``raytrace.py:29-47``, ``gradients.py:31-36``), and the
reference's own objects are accepted too (duck-typed on the same fields).

Precision: the volume goes to the device as float64 (as the reference keeps
it), so images are bit-identical to the reference's ``render``; the
derivatives come from the one-walk reverse-mode kernels and agree with the
reference's forward-mode tangents to ~1e-12 relative.  The device copy of a
volume is cached per volume object (volumes are immutable).
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import (GradientUndefinedError, InvalidArgumentError, KernelError,
                     MetricUndefinedError)
from .geometry import MIN_ABS_SIN_PHI
from .registration import OptimizerConfig, RegistrationTrace, RegistrationEngine
from .renderer import Detector, DeviceVolume, render_frames, render_frames_jac, _stream_ptr

__all__ = ["Volume", "PoseParameters", "DetectorSpec", "Image", "GradientRecord",
           "OptimizerConfig", "RegistrationTrace", "render", "render_iterative",
           "render_with_gradient", "loss_and_gradient", "register"]


# ------------------------------------------------------------------ types
@dataclass(frozen=True)
class Volume:
    """volume.py:24-83: dims, spacing, plane_origin, data indexed [i, j, k]."""

    dims: tuple
    spacing: tuple
    plane_origin: tuple
    data: np.ndarray

    def __post_init__(self):
        dims = tuple(int(n) for n in np.broadcast_to(self.dims, (3,)))
        spacing = tuple(float(s) for s in np.broadcast_to(self.spacing, (3,)))
        origin = tuple(float(b) for b in np.broadcast_to(self.plane_origin, (3,)))
        if any(n < 1 for n in dims):
            raise InvalidArgumentError(f"dims must be three integers >= 1, got {self.dims}")
        if any(not np.isfinite(s) or s <= 0 for s in spacing):
            raise InvalidArgumentError(f"spacing must be three positive reals, got {self.spacing}")
        if any(not np.isfinite(b) for b in origin):
            raise InvalidArgumentError(f"plane_origin must be finite, got {self.plane_origin}")
        data = np.asfortranarray(self.data, dtype=np.float64)
        if data.shape != dims:
            if data.size != int(np.prod(dims)):
                raise InvalidArgumentError(
                    f"data has {data.size} values, expected {int(np.prod(dims))} for dims {dims}")
            data = np.asfortranarray(data.reshape(dims, order="F"))
        data.flags.writeable = False
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "plane_origin", origin)
        object.__setattr__(self, "data", data)

    @property
    def center(self):
        return tuple(b + 0.5 * n * s for b, n, s in zip(self.plane_origin, self.dims, self.spacing))

    def flat_data(self) -> np.ndarray:
        return self.data.ravel(order="F")


@dataclass(frozen=True)
class PoseParameters:
    """geometry.py:32-68: (rho, theta, phi, gamma, shift)."""

    rho: float
    theta: float
    phi: float
    gamma: float = 0.0
    shift: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        vals = (self.rho, self.theta, self.phi, self.gamma, *self.shift)
        if len(vals) != 7 or not all(np.isfinite(v) for v in vals):
            raise InvalidArgumentError(f"pose parameters must be 7 finite reals, got {self}")
        if self.rho <= 0:
            raise InvalidArgumentError(f"rho must be positive, got {self.rho}")
        for name in ("rho", "theta", "phi", "gamma"):
            object.__setattr__(self, name, float(getattr(self, name)))
        object.__setattr__(self, "shift", tuple(float(v) for v in self.shift))

    def to_vector(self) -> np.ndarray:
        return np.array([self.rho, self.theta, self.phi, self.gamma, *self.shift])

    @classmethod
    def from_vector(cls, eta) -> "PoseParameters":
        eta = np.asarray(eta, dtype=np.float64)
        if eta.shape != (7,):
            raise InvalidArgumentError(f"pose vector must have 7 components, got shape {eta.shape}")
        return cls(eta[0], eta[1], eta[2], eta[3], tuple(eta[4:7]))


@dataclass(frozen=True)
class DetectorSpec:
    """geometry.py:71-97: height, width, pixel_pitch (x, y), isocenter."""

    height: int
    width: int
    pixel_pitch: tuple = (1.0, 1.0)
    isocenter: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if self.height < 1 or self.width < 1:
            raise InvalidArgumentError(f"detector must be at least 1x1, got {self.height}x{self.width}")
        pitch = self.pixel_pitch
        if np.isscalar(pitch):
            pitch = (pitch, pitch)
        pitch = tuple(float(p) for p in pitch)
        if any(p <= 0 or not np.isfinite(p) for p in pitch):
            raise InvalidArgumentError(f"pixel pitch must be positive, got {self.pixel_pitch}")
        object.__setattr__(self, "height", int(self.height))
        object.__setattr__(self, "width", int(self.width))
        object.__setattr__(self, "pixel_pitch", pitch)
        object.__setattr__(self, "isocenter", tuple(float(v) for v in self.isocenter))

    @classmethod
    def for_volume(cls, volume, height: int, width: int, pixel_pitch=(1.0, 1.0)) -> "DetectorSpec":
        return cls(height, width, pixel_pitch, tuple(volume.center))


@dataclass
class Image:
    """raytrace.py:29-47: an H x W float64 DRR."""

    values: np.ndarray

    def __post_init__(self):
        values = np.asarray(self.values, dtype=np.float64)
        if values.ndim != 2:
            raise InvalidArgumentError(f"image values must be 2-D, got shape {values.shape}")
        self.values = values

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]


@dataclass
class GradientRecord:
    """gradients.py:31-36: loss value and its 7-gradient."""

    value: float
    grad: np.ndarray = field(default_factory=lambda: np.zeros(7))


# ---------------------------------------------------------------- helpers
_VOLUMES: dict = {}  # id(volume) -> (weakref to the volume, its DeviceVolume)


def _device():
    if not torch.cuda.is_available():
        raise KernelError("this API runs on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _device_volume(volume) -> DeviceVolume:
    """The volume's float64 device copy, uploaded once per volume object."""
    key = id(volume)
    hit = _VOLUMES.get(key)
    if hit is not None and hit[0]() is volume:
        return hit[1]
    flat = np.asarray(volume.flat_data() if hasattr(volume, "flat_data")
                      else np.asarray(volume.data).ravel(order="F"), dtype=np.float64)
    dv = DeviceVolume.from_flat(flat, volume.dims, volume.spacing, volume.plane_origin,
                                device=_device(), dtype=torch.float64)
    try:
        ref = weakref.ref(volume, lambda _r, k=key: _VOLUMES.pop(k, None))
        _VOLUMES[key] = (ref, dv)
    except TypeError:  # not weak-referenceable: no caching
        pass
    return dv


def _detector(spec) -> Detector:
    px, py = (spec.pixel_pitch if not np.isscalar(spec.pixel_pitch)
              else (spec.pixel_pitch, spec.pixel_pitch))
    return Detector(spec.height, spec.width, float(px), float(py), ray_split=1)


def _eta(pose) -> np.ndarray:
    return np.asarray(pose.to_vector(), dtype=np.float64).reshape(7)


def _frames(eta: np.ndarray, isocenter, dev) -> torch.Tensor:
    """The frame computed on the host in float64 (geometry.pose_frames on CPU
    tensors is bit-identical to the reference's numpy _pose_frame, so the
    pixel positions -- and the image -- are too; device sin/cos may differ
    from glibc's in the last ulp)."""
    from .geometry import pose_frames
    f = pose_frames(torch.tensor(eta[None], dtype=torch.float64), isocenter)
    return f.to(dev)


def _frame_jacobian(eta: np.ndarray, dev) -> torch.Tensor:
    """d frame / d eta (12 x 7): drr_pose_grad applied to the 12 unit rows."""
    e = torch.tensor(np.repeat(eta[None], 12, axis=0), dtype=torch.float64, device=dev)
    eye = torch.eye(12, dtype=torch.float64, device=dev)
    out = torch.empty((12, 7), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().drr_pose_grad(e.data_ptr(), eye.data_ptr(), 12, out.data_ptr(),
                                         _stream_ptr(dev)))
    return out


def _check_pose(pose) -> None:
    """gradients.py:39-42."""
    if abs(math.sin(pose.phi)) <= MIN_ABS_SIN_PHI:
        raise GradientUndefinedError(
            f"pose is gimbal-degenerate: |sin(phi)| <= {MIN_ABS_SIN_PHI} at phi={pose.phi}")


def _check_backend(backend) -> None:
    if backend not in (None, "cuda"):
        raise InvalidArgumentError(f"this module renders on the GPU only; backend={backend!r}")


# ------------------------------------------------------------- functions
def render(volume, pose, spec, backend=None, chunk_size=None) -> Image:
    """raytrace.py:138-142: the DRR (bit-identical to the reference's)."""
    _check_backend(backend)
    dv = _device_volume(volume)
    f = _frames(_eta(pose), tuple(spec.isocenter), dv.device)
    img = render_frames(dv, _detector(spec), f, out_dtype=torch.float64)
    return Image(img[0].cpu().numpy())


def render_iterative(volume, pose, spec, backend=None, chunk_size=None) -> Image:
    """raytrace.py:145-152: the plane-by-plane variant -- the GPU walk already
    is incremental, so this is :func:`render`."""
    return render(volume, pose, spec, backend, chunk_size)


def _render_jac(volume, pose, spec):
    dv = _device_volume(volume)
    eta = _eta(pose)
    f = _frames(eta, tuple(spec.isocenter), dv.device)
    det = _detector(spec)
    img, jac = render_frames_jac(dv, det, f, out_dtype=torch.float64)
    return dv, det, eta, img[0], jac


def render_with_gradient(volume, pose, spec, backend=None):
    """gradients.py:45-58: (image, d_image (H, W, 7))."""
    _check_backend(backend)
    _check_pose(pose)
    dv, det, eta, img, jac = _render_jac(volume, pose, spec)
    F = _frame_jacobian(eta, dv.device)                         # (12, 7)
    H, W = spec.height, spec.width
    px, py = det.pitch_x, det.pitch_y
    ah = (torch.arange(H, dtype=torch.float64, device=dv.device) - (H - 1) / 2.0) * py
    aw = (torch.arange(W, dtype=torch.float64, device=dv.device) - (W - 1) / 2.0) * px
    ah = ah[:, None].expand(H, W).reshape(-1)
    aw = aw[None, :].expand(H, W).reshape(-1)
    js, jp = jac[:3], jac[3:]                                   # (3, HW) each
    # p = c + a_h e1 + a_w e2  (geometry.py:171-174)
    d = js.T @ F[0:3] + jp.T @ F[3:6] + (jp * ah).T @ F[6:9] + (jp * aw).T @ F[9:12]
    return Image(img.cpu().numpy()), d.reshape(H, W, 7).cpu().numpy()


def loss_and_gradient(volume, pose, spec, fixed_image, loss_kind: str = "neg_zncc",
                      backend=None) -> GradientRecord:
    """gradients.py:61-69: loss of the DRR against ``fixed_image`` and its
    exact 7-gradient, reduced over pixels in a fixed order.  One native call
    (``drr_forward_loss_grad``, float64 image and fixed image): one walk per
    ray, the loss on the device, no stored Jacobian; one host read at the end."""
    from .registration import LOSS_KINDS
    _check_backend(backend)
    _check_pose(pose)
    if loss_kind not in LOSS_KINDS:
        raise InvalidArgumentError(f"loss kind must be one of ('neg_zncc', 'l2'), got {loss_kind!r}")
    fixed = np.asarray(getattr(fixed_image, "values", fixed_image), dtype=np.float64)
    if fixed.shape != (spec.height, spec.width):
        raise InvalidArgumentError(
            f"image shapes differ: {(spec.height, spec.width)} vs {fixed.shape}")
    dv = _device_volume(volume)
    eta = _eta(pose)
    dev = dv.device
    f = _frames(eta, tuple(spec.isocenter), dev)
    det = _detector(spec)
    lib = _lib.load()
    e = torch.tensor(eta[None], dtype=torch.float64, device=dev)
    fx = torch.as_tensor(fixed, device=dev)
    img = torch.empty((1, spec.height, spec.width), dtype=torch.float64, device=dev)
    out = torch.empty(9, dtype=torch.float64, device=dev)   # value, status, grad (7)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws_bytes = lib.drr_loss_grad_workspace_size(1, det.c)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dev)
    _lib.check(lib.drr_forward_loss_grad(
        dv.flat.data_ptr(), dv.vol_dtype, dv.grid, f.data_ptr(), e.data_ptr(), 1, det.c,
        fx.data_ptr(), 0, LOSS_KINDS[loss_kind], img.data_ptr(), 1, out.data_ptr(),
        status.data_ptr(), None, out[2:].data_ptr(), ws.data_ptr(), ws_bytes, _stream_ptr(dev)))
    out[1] = status[0].to(torch.float64)
    host = out.cpu().numpy()
    if host[1] != 0:
        raise MetricUndefinedError("moving or fixed image has zero variance")
    return GradientRecord(value=float(host[0]), grad=host[2:].copy())


def register(fixed_image, volume, pose0, spec, config=None):
    """registration.py:89-125: momentum GD from ``pose0``; the loop runs on the
    device (RegistrationEngine, one CUDA graph), rendering and scoring in
    float64 as the reference does.  ``config`` may be this module's or the
    reference's OptimizerConfig.  Like the reference, a pose where the loss is
    undefined -- here also a fixed image of the wrong shape -- ends the run
    as failed instead of raising."""
    config = config or OptimizerConfig()
    eta0 = _eta(pose0)
    fixed = np.asarray(getattr(fixed_image, "values", fixed_image), dtype=np.float64)
    if fixed.shape != (spec.height, spec.width):   # metrics._check_pair raises -> failed run
        return RegistrationTrace(rho=float(eta0[0]), poses=eta0[None, 1:].copy(),
                                 losses=np.array([np.inf]), converged=False, failed=True)
    dv = _device_volume(volume)
    eng = RegistrationEngine(dv, _detector(spec), fixed, 1, config,
                             isocenter=tuple(spec.isocenter), image_dtype=torch.float64)
    eng.reset(eta0[None])
    eng.run(use_graph=True)
    return eng.traces()[0]
