"""Loss + gradient and slice-to-volume registration on the device.

Mirrors the reference's ``gradients.loss_and_gradient`` (``gradients.py:61-69``)
and ``registration.register`` (``registration.py:89-125``), batched:

* :func:`loss_and_gradient` -- B poses at once: ``drr_pose_frames`` -> one
  walk per ray -> the fused neg-ZNCC / L2 value and pixel gradient -> dL/dframe
  -> dL/deta, as native launches only (no host round trip, no torch
  autograd).  Two chains (:class:`_Buffers`): the stored ray Jacobian and
  ``drr_loss_grad_jac`` (loss + pixel gradient + contraction + pose gradient
  in one launch), or ``drr_forward_loss_grad`` (no Jacobian: per-CTA
  sums of the ray Jacobian weighted by 1, the image and the fixed image,
  combined with the loss kernel's affine pixel-gradient coefficients).
* :class:`RegistrationEngine` -- B independent momentum-GD registrations
  (``OptimizerConfig`` defaults = the paper's hyper-parameters,
  ``registration.py:41-58``).  Each iteration is the chain above plus
  ``drr_register_update``, which keeps the reference's convergence / failure
  bookkeeping on the device; the whole ``max_iters + 1`` loop is captured in
  one CUDA graph.

Images are float32 by default (the product path); ``image_dtype=torch.float64``
renders and scores in float64 as the reference does (``api.register``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError
from .renderer import Detector, DeviceVolume

LOSS_KINDS = {"neg_zncc": _lib.DRR_LOSS_NEG_ZNCC, "l2": _lib.DRR_LOSS_L2}


@dataclass
class OptimizerConfig:
    """registration.py:41-58 (paper section 3.2 hyper-parameters)."""

    lr_rotation: float = 5.3e-2
    lr_translation: float = 7.5e1
    momentum: float = 0.9
    max_iters: int = 250
    converged_threshold: float = -0.999
    loss_kind: str = "neg_zncc"

    def __post_init__(self):
        if self.lr_rotation <= 0 or self.lr_translation <= 0:
            raise InvalidArgumentError("learning rates must be positive")
        if not 0.0 <= self.momentum < 1.0:
            raise InvalidArgumentError(f"momentum must be in [0, 1), got {self.momentum}")
        if self.max_iters < 1:
            raise InvalidArgumentError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.loss_kind not in LOSS_KINDS:
            raise InvalidArgumentError(f"loss kind must be one of {tuple(LOSS_KINDS)}")

    def c(self):
        return reg_config_c(self)


def reg_config_c(config) -> "_lib.DrrRegConfig":
    """The C-ABI settings from any config with the reference's fields
    (``registration.py:41-58``): this module's OptimizerConfig or the
    reference's own (duck-typed, no method needed)."""
    cfg = _lib.DrrRegConfig()
    cfg.lr_rotation = float(config.lr_rotation)
    cfg.lr_translation = float(config.lr_translation)
    cfg.momentum = float(config.momentum)
    cfg.converged_threshold = float(config.converged_threshold)
    cfg.max_iters = int(config.max_iters)
    return cfg


@dataclass
class RegistrationTrace:
    """registration.py:61-86: per-iteration (theta..bz) and losses."""

    rho: float
    poses: np.ndarray
    losses: np.ndarray
    converged: bool
    failed: bool = False

    @property
    def iterations_used(self) -> int:
        return len(self.losses) - 1

    @property
    def final_loss(self) -> float:
        return float(self.losses[-1])

    def final_pose(self):
        """registration.py:84-85: the last recorded pose with the fixed rho."""
        from .api import PoseParameters
        return PoseParameters.from_vector(np.concatenate([[self.rho], self.poses[-1]]))


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


class _Buffers:
    """Device buffers for B poses; reused across calls (no allocation in the loop).

    Two native chains compute the same step (``mode``):

    * ``"jac"`` -- ``drr_forward_jac`` stores each ray's 6-double Jacobian
      (48 B/pixel) and ``drr_loss_grad_jac`` computes the loss, its float64
      pixel gradient and their contraction (and the pose gradient) in one
      cluster launch per image: measured faster at C2 (the fused walk's
      per-CTA 36-sum epilogue costs more; profiles/r02/SUMMARY.md);
    * ``"fused"`` -- ``drr_forward_loss_grad``: no Jacobian, the pixel gradient
      as an affine map of the two images reduced inside the walk; float64
      pixel gradients (used for float64 images) and any batch size.

    ``"auto"`` takes ``"jac"`` for float32 images whose Jacobian fits
    ``renderer.JAC_BUDGET_BYTES`` (8 GiB; C2's 256 poses hold 0.5 GB, C5's 64
    poses at 1024^2 3.2 GB), else ``"fused"``."""

    def __init__(self, vol: DeviceVolume, det: Detector, B: int, image_dtype=torch.float32,
                 mode: str = "auto"):
        from .renderer import JAC_BUDGET_BYTES, jac_bytes
        dev = vol.device
        if mode not in ("auto", "jac", "fused"):
            raise InvalidArgumentError(f"mode must be 'auto', 'jac' or 'fused', got {mode!r}")
        if mode == "auto":
            mode = ("jac" if image_dtype == torch.float32 and jac_bytes(det, B) <= JAC_BUDGET_BYTES
                    else "fused")
        if mode == "jac" and image_dtype != torch.float32:
            raise InvalidArgumentError("the stored-Jacobian chain takes float32 images")
        self.mode = mode
        self.B = B
        self.image_dtype = image_dtype
        self.img_code = 1 if image_dtype == torch.float64 else 0
        self.frames = torch.empty((B, 12), dtype=torch.float64, device=dev)
        self.img = torch.empty((B, det.height, det.width), dtype=image_dtype, device=dev)
        self.value = torch.empty(B, dtype=torch.float64, device=dev)
        self.status = torch.zeros(B, dtype=torch.int32, device=dev)
        self.grad_frames = torch.empty((B, 12), dtype=torch.float64, device=dev)
        self.grad_eta = torch.empty((B, 7), dtype=torch.float64, device=dev)
        lib = _lib.load()
        if mode == "jac":
            self.jac = torch.empty((6, B * det.height * det.width), dtype=torch.float64, device=dev)
            self.ws_bytes = 0
        else:
            self.ws_bytes = lib.drr_loss_grad_workspace_size(B, det.c)
        self.ws = torch.empty(max(self.ws_bytes, 8), dtype=torch.uint8, device=dev)


def _launch_loss_grad(lib, vol, det, iso, eta, fixed, fixed_stride, kind, buf, stream,
                      value_ptr=None, grad_eta_ptr=None, grad_frames=True):
    """pose frames -> one walk per ray -> loss value + pixel gradient -> dL/dframe
    (buf.grad_frames) -> dL/deta (``grad_eta_ptr``, when given); the loss values
    go to ``value_ptr`` (or buf.value).  The output pointers may be another
    rank's buffers (distributed.PeerRows).  ``buf.mode`` picks the chain:
    three launches either way."""
    B = buf.B
    value_ptr = buf.value.data_ptr() if value_ptr is None else value_ptr
    _lib.check(lib.drr_pose_frames(eta.data_ptr(), B, iso, buf.frames.data_ptr(), stream))
    if buf.mode == "fused":
        _lib.check(lib.drr_forward_loss_grad(
            vol.flat.data_ptr(), vol.vol_dtype, vol.grid, buf.frames.data_ptr(), eta.data_ptr(),
            B, det.c, fixed.data_ptr(), fixed_stride, kind, buf.img.data_ptr(), buf.img_code,
            value_ptr, buf.status.data_ptr(), buf.grad_frames.data_ptr() if grad_frames else None,
            grad_eta_ptr, buf.ws.data_ptr(), buf.ws_bytes, stream))
        return
    _lib.check(lib.drr_forward_jac(vol.flat.data_ptr(), vol.vol_dtype, vol.grid,
                                   buf.frames.data_ptr(), B, det.c, buf.img.data_ptr(), 0,
                                   buf.jac.data_ptr(), stream))
    # loss + float64 pixel gradient + contraction (+ pose gradient): one launch
    _lib.check(lib.drr_loss_grad_jac(buf.jac.data_ptr(), buf.img.data_ptr(), fixed.data_ptr(), 0,
                                     fixed_stride, B, det.c, kind, value_ptr,
                                     buf.status.data_ptr(),
                                     buf.grad_frames.data_ptr() if grad_frames else None,
                                     eta.data_ptr(), grad_eta_ptr, stream))


def _prep_fixed(fixed, B, det, dev, dtype=torch.float32):
    if not isinstance(fixed, (torch.Tensor, np.ndarray)) and hasattr(fixed, "values"):
        fixed = fixed.values  # a reference Image
    fixed = torch.as_tensor(fixed, device=dev, dtype=dtype)
    if fixed.shape[-2:] != (det.height, det.width):
        raise InvalidArgumentError(
            f"fixed image shape {tuple(fixed.shape)} does not match detector {det.height}x{det.width}")
    if fixed.ndim == 2 or fixed.shape[0] == 1:
        return fixed.reshape(det.height, det.width).contiguous(), 0
    if fixed.shape[0] != B:
        raise InvalidArgumentError(f"need 1 or {B} fixed images, got {fixed.shape[0]}")
    return fixed.contiguous(), det.height * det.width


def loss_and_gradient(vol: DeviceVolume, det: Detector, eta, fixed, loss_kind: str = "neg_zncc",
                      isocenter=None, buffers: _Buffers | None = None,
                      image_dtype=torch.float32, mode: str = "auto"):
    """Batched ``gradients.loss_and_gradient``: (value (B,), grad (B, 7)) for
    pose vectors eta (B, 7) = (rho, theta, phi, gamma, bx, by, bz).

    Device tensors in and out; undefined metrics give NaN values (status in
    ``buffers.status``) instead of raising, so the call never synchronises."""
    if loss_kind not in LOSS_KINDS:
        raise InvalidArgumentError(f"loss kind must be one of {tuple(LOSS_KINDS)}, got {loss_kind!r}")
    dev = vol.device
    eta = torch.as_tensor(eta, device=dev, dtype=torch.float64)
    if eta.ndim == 1:
        eta = eta[None]
    eta = eta.contiguous()
    B = eta.shape[0]
    from .renderer import MAX_POSES_PER_LAUNCH
    if B > MAX_POSES_PER_LAUNCH:  # one launch covers at most 65535 poses: chunk
        per_pose = isinstance(fixed, (torch.Tensor, np.ndarray)) and fixed.ndim == 3
        parts = [loss_and_gradient(vol, det, eta[lo:lo + MAX_POSES_PER_LAUNCH],
                                   fixed[lo:lo + MAX_POSES_PER_LAUNCH] if per_pose else fixed,
                                   loss_kind, isocenter, None, image_dtype, mode)
                 for lo in range(0, B, MAX_POSES_PER_LAUNCH)]
        return torch.cat([v for v, _ in parts]), torch.cat([g for _, g in parts])
    buf = (buffers if buffers is not None and buffers.B == B
           and buffers.image_dtype == image_dtype else _Buffers(vol, det, B, image_dtype, mode))
    fixed_t, stride = _prep_fixed(fixed, B, det, dev, image_dtype)
    iso = _iso(vol, isocenter)
    lib = _lib.load()
    st = _stream(dev)
    _launch_loss_grad(lib, vol, det, iso, eta, fixed_t, stride, LOSS_KINDS[loss_kind], buf, st,
                      grad_eta_ptr=buf.grad_eta.data_ptr(), grad_frames=False)
    return buf.value.clone(), buf.grad_eta.clone()


def _iso(vol, isocenter):
    import ctypes
    c = vol.center if isocenter is None else tuple(float(v) for v in isocenter)
    return (ctypes.c_double * 3)(*c)


class RegistrationEngine:
    """B independent registrations of fixed image(s) against one CT volume.

    ``mode="fused"`` (default): each iteration is ``drr_register_step`` --
    the Jacobian-free walk, the loss, and a reduction that also applies the
    momentum step and writes the next frames: three launches (C3 at C2, one
    pose, one CUDA graph: 0.0854 ms per step vs 0.0880 for the four-launch
    stored-Jacobian iteration, ``scripts/c3_modes.py``).  ``mode="jac"``: the
    stored-Jacobian chain (pose frames, ``drr_forward_jac``,
    ``drr_loss_grad_jac``) + ``drr_register_update``."""

    def __init__(self, vol: DeviceVolume, det: Detector, fixed, B: int = 1,
                 config: OptimizerConfig | None = None, isocenter=None,
                 image_dtype=torch.float32, mode: str = "fused"):
        self.vol, self.det, self.B = vol, det, int(B)
        self.config = config or OptimizerConfig()
        dev = vol.device
        self.fixed, self.fixed_stride = _prep_fixed(fixed, self.B, det, dev, image_dtype)
        self.iso = _iso(vol, isocenter)
        self.buf = _Buffers(vol, det, self.B, image_dtype, mode)
        T = self.config.max_iters + 1
        self.eta = torch.zeros((self.B, 7), dtype=torch.float64, device=dev)
        self.vel = torch.zeros((self.B, 6), dtype=torch.float64, device=dev)
        self.state = torch.zeros(self.B, dtype=torch.int32, device=dev)
        self.n_rec = torch.zeros(self.B, dtype=torch.int32, device=dev)
        self.trace_eta = torch.zeros((self.B, T, 6), dtype=torch.float64, device=dev)
        self.trace_loss = torch.zeros((self.B, T), dtype=torch.float64, device=dev)
        self.graph = None
        kind = getattr(self.config, "loss_kind", "neg_zncc")
        if kind not in LOSS_KINDS:
            raise InvalidArgumentError(f"loss kind must be one of {tuple(LOSS_KINDS)}, got {kind!r}")
        self.kind = LOSS_KINDS[kind]
        self._cfg = reg_config_c(self.config)

    def reset(self, poses0):
        p = torch.as_tensor(poses0, dtype=torch.float64, device=self.vol.device).reshape(self.B, 7)
        self.eta.copy_(p)
        self.vel.zero_()
        self.state.zero_()
        self.n_rec.zero_()

    def _iteration(self, it: int, stream: int):
        lib = _lib.load()
        buf = self.buf
        if buf.mode == "fused":
            # three launches: walk, loss, reduction + update + the next frames
            if it == 0:
                _lib.check(lib.drr_pose_frames(self.eta.data_ptr(), self.B, self.iso,
                                               buf.frames.data_ptr(), stream))
            _lib.check(lib.drr_register_step(
                self.vol.flat.data_ptr(), self.vol.vol_dtype, self.vol.grid, buf.frames.data_ptr(),
                self.eta.data_ptr(), self.vel.data_ptr(), self.B, self.det.c,
                self.fixed.data_ptr(), self.fixed_stride, self.kind, buf.img.data_ptr(),
                buf.img_code, buf.value.data_ptr(), buf.status.data_ptr(), self.iso, self._cfg,
                it, self.state.data_ptr(), self.n_rec.data_ptr(), self.trace_eta.data_ptr(),
                self.trace_loss.data_ptr(), buf.ws.data_ptr(), buf.ws_bytes, stream))
            return
        _launch_loss_grad(lib, self.vol, self.det, self.iso, self.eta, self.fixed,
                          self.fixed_stride, self.kind, buf, stream)
        _lib.check(lib.drr_register_update(
            self.eta.data_ptr(), self.vel.data_ptr(), self.buf.grad_frames.data_ptr(),
            self.buf.value.data_ptr(), self.buf.status.data_ptr(), self._cfg, it,
            self.state.data_ptr(), self.n_rec.data_ptr(), self.trace_eta.data_ptr(),
            self.trace_loss.data_ptr(), self.B, stream))

    def run(self, use_graph: bool = True):
        """All max_iters + 1 iterations (converged / failed registrations are
        frozen on the device).  With use_graph the loop is one CUDA graph."""
        dev = self.vol.device
        if not use_graph:
            st = _stream(dev)
            for it in range(self.config.max_iters + 1):
                self._iteration(it, st)
            return
        if self.graph is None:
            saved = [t.clone() for t in (self.eta, self.vel, self.state, self.n_rec)]
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):  # warm-up outside capture (loads the kernels)
                self._iteration(0, side.cuda_stream)
            torch.cuda.current_stream(dev).wait_stream(side)
            for t, s in zip((self.eta, self.vel, self.state, self.n_rec), saved):
                t.copy_(s)  # the warm-up iteration must not advance the registrations
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                st = _stream(dev)
                for it in range(self.config.max_iters + 1):
                    self._iteration(it, st)
        self.graph.replay()

    def traces(self):
        n = self.n_rec.cpu().numpy()
        state = self.state.cpu().numpy()
        te = self.trace_eta.cpu().numpy()
        tl = self.trace_loss.cpu().numpy()
        rho = self.eta[:, 0].cpu().numpy()
        out = []
        for b in range(self.B):
            k = int(n[b])
            out.append(RegistrationTrace(rho=float(rho[b]), poses=te[b, :k].copy(),
                                         losses=tl[b, :k].copy(),
                                         converged=bool(state[b] == _lib.DRR_REG_CONVERGED),
                                         failed=bool(state[b] == _lib.DRR_REG_FAILED)))
        return out


def register(fixed_image, vol: DeviceVolume, pose0, det: Detector,
             config: OptimizerConfig | None = None, use_graph: bool = False) -> RegistrationTrace:
    """``registration.register`` for one pose vector (rho, theta, ..., bz)."""
    eng = RegistrationEngine(vol, det, fixed_image, 1, config)
    eng.reset(np.asarray(pose0, dtype=np.float64)[None])
    eng.run(use_graph=use_graph)
    return eng.traces()[0]


def register_batch(fixed_images, vol: DeviceVolume, poses0, det: Detector,
                   config: OptimizerConfig | None = None, use_graph: bool = True):
    """B independent registrations (the population study, cli.py:133-145)."""
    poses0 = np.asarray(poses0, dtype=np.float64).reshape(-1, 7)
    eng = RegistrationEngine(vol, det, fixed_images, poses0.shape[0], config)
    eng.reset(poses0)
    eng.run(use_graph=use_graph)
    return eng.traces()


# ---------------------------------------------------------------- landscape
OPTIMIZED_PARAMS = ("theta", "phi", "gamma", "bx", "by", "bz")
NARROW_HALF_WIDTHS = {"theta": math.radians(45.0), "phi": math.radians(45.0),
                      "gamma": math.radians(22.5), "bx": 15.0, "by": 15.0, "bz": 15.0}


@dataclass
class LandscapeGrid:
    """registration.py:150-156."""

    axes: tuple
    coords: tuple
    losses: np.ndarray


def loss_landscape(vol: DeviceVolume, det: Detector, truth, loss_kind: str = "neg_zncc",
                   axes=("theta",), samples=41, half_widths=None, chunk: int = 1024,
                   isocenter=None) -> LandscapeGrid:
    """``registration.loss_landscape`` (registration.py:159-203) as batched
    renders: the fixed image renders once at ``truth``; every grid pose is one
    row of a (B, 7) batch -> drr_pose_frames -> drr_forward -> drr_image_loss
    (value only), ``chunk`` poses per launch.  Undefined metrics give +inf."""
    import ctypes
    if isinstance(axes, str):
        axes = (axes,)
    axes = tuple(axes)
    if not 1 <= len(axes) <= 2:
        raise InvalidArgumentError(f"axes must name one or two parameters, got {axes}")
    for name in axes:
        if name not in OPTIMIZED_PARAMS:
            raise InvalidArgumentError(f"unknown sweep axis {name!r}, expected one of {OPTIMIZED_PARAMS}")
    if loss_kind not in LOSS_KINDS:
        raise InvalidArgumentError(f"loss kind must be one of {tuple(LOSS_KINDS)}, got {loss_kind!r}")
    samples = np.broadcast_to(np.asarray(samples, dtype=int), (len(axes),))
    if np.any(samples < 3):
        raise InvalidArgumentError(f"grid resolution must be >= 3 per axis, got {samples}")
    if half_widths is None:
        half_widths = [NARROW_HALF_WIDTHS[name] for name in axes]
    half_widths = np.broadcast_to(np.asarray(half_widths, dtype=np.float64), (len(axes),))
    center = np.asarray(truth, dtype=np.float64).reshape(7)
    index = {name: i for i, name in enumerate(OPTIMIZED_PARAMS, start=1)}
    coords = tuple(center[index[name]] + np.linspace(-hw, hw, int(ns))
                   for name, hw, ns in zip(axes, half_widths, samples))
    if len(axes) == 1:
        grid = coords[0][:, None]
    else:
        grid = np.stack(np.meshgrid(coords[0], coords[1], indexing="ij"), -1).reshape(-1, 2)
    etas = np.repeat(center[None], grid.shape[0], axis=0)
    for j, name in enumerate(axes):
        etas[:, index[name]] = grid[:, j]
    dev = vol.device
    lib = _lib.load()
    st = _stream(dev)
    iso = _iso(vol, isocenter)
    npix = det.height * det.width
    # fixed image at the truth pose
    one = torch.tensor(center[None], device=dev)
    fr = torch.empty((1, 12), dtype=torch.float64, device=dev)
    fixed = torch.empty((1, det.height, det.width), dtype=torch.float32, device=dev)
    _lib.check(lib.drr_pose_frames(one.data_ptr(), 1, iso, fr.data_ptr(), st))
    _lib.check(lib.drr_forward(vol.flat.data_ptr(), vol.vol_dtype, vol.grid, fr.data_ptr(), 1,
                               det.c, fixed.data_ptr(), 0, st))
    out = torch.empty(etas.shape[0], dtype=torch.float64, device=dev)
    status = torch.empty(etas.shape[0], dtype=torch.int32, device=dev)
    all_eta = torch.tensor(etas, device=dev)
    frames = torch.empty((min(chunk, etas.shape[0]), 12), dtype=torch.float64, device=dev)
    img = torch.empty((min(chunk, etas.shape[0]), det.height, det.width), dtype=torch.float32,
                      device=dev)
    for s in range(0, etas.shape[0], chunk):
        n = min(chunk, etas.shape[0] - s)
        e = all_eta[s:s + n]
        _lib.check(lib.drr_pose_frames(e.data_ptr(), n, iso, frames.data_ptr(), st))
        _lib.check(lib.drr_forward(vol.flat.data_ptr(), vol.vol_dtype, vol.grid, frames.data_ptr(),
                                   n, det.c, img.data_ptr(), 0, st))
        _lib.check(lib.drr_image_loss(img.data_ptr(), fixed.data_ptr(), 0, 0, n, npix,
                                      LOSS_KINDS[loss_kind], out[s:].data_ptr(), None,
                                      status[s:].data_ptr(), st))
    losses = torch.where(status != 0, torch.full_like(out, math.inf), out).cpu().numpy()
    if len(axes) == 2:
        losses = losses.reshape(len(coords[0]), len(coords[1]))
    return LandscapeGrid(axes=axes, coords=coords, losses=losses)
