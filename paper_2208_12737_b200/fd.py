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


def ray_signatures(vol: DeviceVolume, det: Detector, eta_rows, isocenter=None) -> np.ndarray:
    """Per-ray traversal-structure signatures (n, H, W) uint64 of the (n, 7)
    poses (``drr_ray_signatures``; a pose's :func:`signatures` entry is the
    wrapping sum of its rays')."""
    fr = _frames(vol, np.asarray(eta_rows, dtype=np.float64).reshape(-1, 7), isocenter)
    sig = torch.empty((fr.shape[0], det.height, det.width), dtype=torch.int64, device=fr.device)
    _lib.check(_lib.load().drr_ray_signatures(vol.flat.data_ptr(), vol.vol_dtype, vol.grid,
                                              fr.data_ptr(), fr.shape[0], det.c, sig.data_ptr(),
                                              torch.cuda.current_stream(fr.device).cuda_stream))
    return sig.cpu().numpy().view(np.uint64)


def ray_fd_report(vol: DeviceVolume, det: Detector, eta, steps=None, isocenter=None) -> dict:
    """Central FD of every ray's energy against its exact pose gradient, with
    the boundary test of ``detect_fd_boundaries`` (gradients.py:145-167)
    applied ray by ray.

    On a full detector nearly every pose-level stencil straddles some ray's
    structure change (C2: all 7 components), so the image-level report has no
    kink-free component to test; per ray most stencils are kink-free, and
    there the reference's bar (rel < 1e-5, test_gradients.py:119-148) applies
    to each (ray, component).  Exact: the float64 energy Jacobian of one walk
    (``drr_forward_jac``: dE/ds, dE/dp) chained through the frame map
    (geometry.py:120-149).  FD: float64 renders of the bumped poses at the
    steps and at half the steps (a pair is kink-free when neither stencil
    changes its ray's structure).  A pair above the bar whose Richardson
    extrapolation (4 FD(h/2) - FD(h)) / 3 meets it is FD truncation error
    (O(h^2): a grazing ray's crossings curve fast), not a gradient error;
    ``unexplained`` counts the pairs that fail both."""
    from .geometry import pixel_offsets, pose_frames
    from .renderer import render_frames, render_frames_jac
    eta = np.asarray(eta, dtype=np.float64).reshape(7)
    _check_pose(eta)
    s = _steps(steps)
    H, W = det.height, det.width

    def central(step):
        rows = _stencil(eta, step, "central")
        img = render_frames(vol, det, _frames(vol, rows, isocenter),
                            out_dtype=torch.float64).cpu().numpy()
        fd = np.stack([(img[1 + 2 * i] - img[2 + 2 * i]) / (2.0 * step[i]) for i in range(7)], -1)
        sig = ray_signatures(vol, det, rows, isocenter)
        kink = np.stack([(sig[1 + 2 * i] != sig[0]) | (sig[2 + 2 * i] != sig[0])
                         for i in range(7)], -1)  # (H, W, 7)
        return img[0], fd, kink

    E, fd, kink = central(s)
    _, fd2, kink2 = central(0.5 * s)
    rich = (4.0 * fd2 - fd) / 3.0
    _, jac = render_frames_jac(vol, det, _frames(vol, eta[None], isocenter),
                               out_dtype=torch.float64)
    jac = jac.cpu().numpy().reshape(6, H, W)
    iso = vol.center if isocenter is None else tuple(float(v) for v in isocenter)
    Jf = torch.autograd.functional.jacobian(
        lambda e: pose_frames(e[None], iso)[0], torch.tensor(eta)).numpy()  # (12, 7)
    ah, aw = (np.asarray(v) for v in pixel_offsets(H, W, det.pitch_x, det.pitch_y))
    dp = (Jf[3:6][None, None] + ah[:, None, None, None] * Jf[6:9][None, None]
          + aw[None, :, None, None] * Jf[9:12][None, None])  # (H, W, 3, 7)
    exact = (np.einsum("ahw,aj->hwj", jac[0:3], Jf[0:3])
             + np.einsum("ahw,hwaj->hwj", jac[3:6], dp))  # (H, W, 7)

    def rel(f):
        den = np.maximum(np.abs(exact), np.abs(f))
        return np.abs(exact - f) / np.where(den > 0, den, 1.0), den

    r, den = rel(fd)
    rr, _ = rel(rich)
    # The FD quotients' own rounding: a ray energy sums a few hundred segments
    # in float64 (~1e-13 |E| relative at most), divided by 2 h (x3 for the
    # extrapolation).  A pair is resolvable at the 1e-5 bar when its gradient
    # is above that noise / 1e-5 (the per-ray counterpart of the reference's
    # |exact| > 1e-8 for O(1) losses).
    noise = 3e-13 * np.abs(E)[..., None] / s[None, None, :]
    hit = (E != 0.0)[..., None] & np.ones(7, dtype=bool)
    boundary = hit & (kink | kink2)
    tested = hit & ~boundary & (den > noise / 1e-5)
    over = tested & (r >= 1e-5)
    bad = over & (rr >= 1e-5)
    return {"rays": int(H * W), "rays_nonzero": int(hit[..., 0].sum()),
            "pairs": int(hit.sum()), "pairs_boundary": int(boundary.sum()),
            "pairs_tested": int(tested.sum()),
            "max_rel_kink_free": float(r[tested].max()) if tested.any() else None,
            "p99_rel_kink_free": float(np.quantile(r[tested], 0.99)) if tested.any() else None,
            "n_over_1e-5": int(over.sum()),
            "n_over_1e-5_truncation": int((over & ~bad).sum()),
            "max_rel_richardson": float(rr[tested].max()) if tested.any() else None,
            "unexplained": int(bad.sum()),
            "per_component_tested": tested.sum(axis=(0, 1)).tolist(),
            "max_rel_boundary": float(r[boundary].max()) if boundary.any() else None}
