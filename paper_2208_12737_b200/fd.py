"""Finite-difference checks of the pose gradient, on the device.

Restates the reference's validation oracle (``gradients.py:72-167``), batched:

* :func:`default_fd_steps` -- 1e-3 for rho and lengths, 1e-5 rad for angles
  (``gradients.py:72-74``);
* :func:`finite_difference_gradient` -- central (or forward) differences of
  the rendered loss (``gradients.py:77-121``): the 2 x 7 bumped poses (+ the
  centre for the forward scheme) render as ONE float64 batch
  (``drr_pose_frames`` + ``drr_forward``) and are scored by ``drr_image_loss``
  -- primal renders only, independent of the reverse-mode kernels they check;
* :func:`detect_fd_boundaries` -- which stencils straddle a change of the
  discrete traversal structure (``gradients.py:145-167``): the 15 poses'
  per-pose signatures (``drr_signature``) against the centre's;
* :func:`fd_report` -- exact vs FD per component, the relative error the
  reference's test bars (``test_gradients.py:119-148``: < 1e-5 wherever the
  stencil is kink-free), and which components a boundary explains.

Float64 throughout (float32 images would put ~1e-7 rounding into losses that
differ by ~1e-5 x gradient).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import GradientUndefinedError, InvalidArgumentError
from .geometry import MIN_ABS_SIN_PHI
from .renderer import Detector, DeviceVolume


def default_fd_steps() -> np.ndarray:
    """gradients.py:72-74."""
    return np.array([1e-3, 1e-5, 1e-5, 1e-5, 1e-3, 1e-3, 1e-3])


def _steps(steps):
    s = default_fd_steps() if steps is None else np.broadcast_to(
        np.asarray(steps, dtype=np.float64), (7,)).copy()
    if np.any(s <= 0):
        raise InvalidArgumentError(f"steps must be positive, got {s}")
    return s


def _stencil(eta, steps, scheme):
    """(rows (n, 7), index of the centre row or None): +/- bumps per component."""
    eta = np.asarray(eta, dtype=np.float64).reshape(7)
    rows = [eta.copy()]
    for i in range(7):
        for sign in (+1.0, -1.0):
            if scheme == "forward" and sign < 0:
                continue
            r = eta.copy()
            r[i] += sign * steps[i]
            rows.append(r)
    return np.stack(rows)


def _frames(vol: DeviceVolume, eta_rows: np.ndarray, isocenter=None):
    dev = vol.device
    e = torch.tensor(eta_rows, dtype=torch.float64, device=dev)
    fr = torch.empty((e.shape[0], 12), dtype=torch.float64, device=dev)
    c = vol.center if isocenter is None else tuple(float(v) for v in isocenter)
    _lib.check(_lib.load().drr_pose_frames(e.data_ptr(), e.shape[0], (ctypes.c_double * 3)(*c),
                                           fr.data_ptr(),
                                           torch.cuda.current_stream(dev).cuda_stream))
    return fr


def _losses(vol, det, eta_rows, fixed, loss_kind, isocenter=None):
    from .registration import LOSS_KINDS
    dev = vol.device
    lib = _lib.load()
    st = torch.cuda.current_stream(dev).cuda_stream
    fr = _frames(vol, eta_rows, isocenter)
    n = fr.shape[0]
    img = torch.empty((n, det.height, det.width), dtype=torch.float64, device=dev)
    _lib.check(lib.drr_forward(vol.flat.data_ptr(), vol.vol_dtype, vol.grid, fr.data_ptr(), n,
                               det.c, img.data_ptr(), 1, st))
    fx = torch.as_tensor(np.asarray(fixed, dtype=np.float64), device=dev).contiguous()
    val = torch.empty(n, dtype=torch.float64, device=dev)
    status = torch.zeros(n, dtype=torch.int32, device=dev)
    _lib.check(lib.drr_image_loss(img.data_ptr(), fx.data_ptr(), 1, 0, n,
                                  det.height * det.width, LOSS_KINDS[loss_kind], val.data_ptr(),
                                  None, status.data_ptr(), st))
    return val.cpu().numpy(), status.cpu().numpy()


def _check_pose(eta):
    if abs(np.sin(eta[2])) <= MIN_ABS_SIN_PHI:  # gradients.py:39-42
        raise GradientUndefinedError(
            f"pose is gimbal-degenerate: |sin(phi)| <= {MIN_ABS_SIN_PHI} at phi={eta[2]}")


def finite_difference_gradient(vol: DeviceVolume, det: Detector, eta, fixed,
                               loss_kind: str = "neg_zncc", steps=None,
                               scheme: str = "central", isocenter=None) -> np.ndarray:
    """gradients.py:100-121: FD gradient of the rendered loss at pose eta (7,)."""
    if scheme not in ("forward", "central"):
        raise InvalidArgumentError(f"scheme must be 'forward' or 'central', got {scheme!r}")
    eta = np.asarray(eta, dtype=np.float64).reshape(7)
    _check_pose(eta)
    s = _steps(steps)
    rows = _stencil(eta, s, scheme)
    val, _ = _losses(vol, det, rows, fixed, loss_kind, isocenter)
    grad = np.zeros(7)
    for i in range(7):
        if scheme == "central":
            grad[i] = (val[1 + 2 * i] - val[2 + 2 * i]) / (2.0 * s[i])
        else:
            grad[i] = (val[1 + i] - val[0]) / s[i]
    return grad


def signatures(vol: DeviceVolume, det: Detector, eta_rows, isocenter=None) -> np.ndarray:
    """Per-pose traversal-structure signatures (uint64) of the (n, 7) poses."""
    fr = _frames(vol, np.asarray(eta_rows, dtype=np.float64).reshape(-1, 7), isocenter)
    sig = torch.empty(fr.shape[0], dtype=torch.int64, device=fr.device)
    _lib.check(_lib.load().drr_signature(vol.flat.data_ptr(), vol.vol_dtype, vol.grid,
                                         fr.data_ptr(), fr.shape[0], det.c, sig.data_ptr(),
                                         torch.cuda.current_stream(fr.device).cuda_stream))
    return sig.cpu().numpy().view(np.uint64)


def detect_fd_boundaries(vol: DeviceVolume, det: Detector, eta, steps=None,
                         isocenter=None) -> np.ndarray:
    """gradients.py:145-167: component i is True when the traversal structure
    differs anywhere across [eta - steps_i e_i, eta + steps_i e_i]."""
    s = _steps(steps)
    rows = _stencil(eta, s, "central")
    sig = signatures(vol, det, rows, isocenter)
    return np.array([sig[1 + 2 * i] != sig[0] or sig[2 + 2 * i] != sig[0] for i in range(7)])


def fd_report(vol: DeviceVolume, det: Detector, eta, fixed, loss_kind: str = "neg_zncc",
              steps=None, exact=None, isocenter=None) -> dict:
    """Exact (float64 fused kernel) vs central FD at one pose, with boundary
    attribution: the reference's bar is rel < 1e-5 on every component whose
    stencil is kink-free (test_gradients.py:119-148; |exact| <= 1e-8 counts as
    agreeing)."""
    from .registration import loss_and_gradient
    eta = np.asarray(eta, dtype=np.float64).reshape(7)
    if exact is None:
        _, g = loss_and_gradient(vol, det, eta[None], np.asarray(fixed, dtype=np.float64),
                                 loss_kind, isocenter=isocenter, image_dtype=torch.float64)
        exact = g[0].cpu().numpy()
    fd = finite_difference_gradient(vol, det, eta, fixed, loss_kind, steps, "central", isocenter)
    boundary = detect_fd_boundaries(vol, det, eta, steps, isocenter)
    denom = np.maximum(np.abs(exact), np.abs(fd))
    rel = np.where(np.abs(exact) > 1e-8, np.abs(exact - fd) / np.where(denom > 0, denom, 1.0),
                   0.0)
    clean = ~boundary
    return {"exact": exact.tolist(), "fd": fd.tolist(), "rel": rel.tolist(),
            "boundary": boundary.tolist(),
            "max_rel_kink_free": float(rel[clean].max()) if clean.any() else None,
            "n_kink_free": int(clean.sum()),
            "unexplained": bool(((rel >= 1e-5) & clean).any())}
