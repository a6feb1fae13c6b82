"""Pose -> detector frame, as differentiable torch ops on the device.

Restates ``geometry._pose_frame`` (reference ``pkg/src/drrtrace/geometry.py:120-149``)
for a batch of poses.  The seven-vector order is the reference's
``POSE_PARAM_NAMES`` = (rho, theta, phi, gamma, bx, by, bz) (``geometry.py:24``):

    u       = (sin phi cos theta, sin phi sin theta, cos phi)
    e_theta = (-sin theta, cos theta, 0);  e_phi = (cos phi cos theta, cos phi sin theta, -sin phi)
    s  = iso + shift + rho u              c  = iso + shift - rho u
    e1 = cos g e_phi - sin g e_theta      e2 = cos g e_theta + sin g e_phi

The frame (s, c, e1, e2) is the 12-number interface of the CUDA kernels: the
forward kernel generates pixel p[h, w] = (c + a_h e1) + a_w e2 itself
(``geometry.py:152-175``) and the backward kernel returns dL/d(frame), which
torch autograd chains through this function to (rho, theta, phi, gamma, shift).
That replaces the reference's forward-mode dual numbers (``dual.py``) and its
(H, W, 3, 7) pixel-tangent array (``geometry.py:178-202``).
"""

from __future__ import annotations

import math

import torch

from .errors import GradientUndefinedError, InvalidArgumentError

POSE_PARAM_NAMES = ("rho", "theta", "phi", "gamma", "bx", "by", "bz")
MIN_ABS_SIN_PHI = 1e-6  # gradients.py:28


def pose_frames(eta: torch.Tensor, isocenter) -> torch.Tensor:
    """(B, 7) float64 pose vectors -> (B, 12) frames (s, c, e1, e2)."""
    if eta.ndim != 2 or eta.shape[1] != 7:
        raise InvalidArgumentError(f"pose vectors must be (B, 7), got {tuple(eta.shape)}")
    iso = torch.as_tensor(isocenter, dtype=eta.dtype, device=eta.device)
    rho = eta[:, 0:1]
    theta, phi, gamma = eta[:, 1], eta[:, 2], eta[:, 3]
    shift = eta[:, 4:7]
    st, ct = torch.sin(theta), torch.cos(theta)
    sp, cp = torch.sin(phi), torch.cos(phi)
    sg, cg = torch.sin(gamma), torch.cos(gamma)
    zero = torch.zeros_like(st)
    u = torch.stack([sp * ct, sp * st, cp], dim=-1)
    e_theta = torch.stack([-st, ct, zero], dim=-1)
    e_phi = torch.stack([cp * ct, cp * st, -sp], dim=-1)
    source = shift + rho * u
    center = shift - rho * u
    e1 = cg[:, None] * e_phi - sg[:, None] * e_theta
    e2 = cg[:, None] * e_theta + sg[:, None] * e_phi
    return torch.cat([iso + source, iso + center, e1, e2], dim=-1)


def check_pose_vectors(eta: torch.Tensor) -> None:
    """The reference's PoseParameters validation (geometry.py:47-53):
    finite values and rho > 0.  Synchronises with the device."""
    if not bool(torch.isfinite(eta).all()):
        raise InvalidArgumentError("pose parameters must be finite")
    if not bool((eta[:, 0] > 0).all()):
        raise InvalidArgumentError("rho must be positive")


def check_gimbal(eta: torch.Tensor) -> None:
    """The gradient path's guard, ``gradients._check_pose`` (gradients.py:39-42)."""
    bad = torch.sin(eta[:, 2]).abs() <= MIN_ABS_SIN_PHI
    if bool(bad.any()):
        phi = float(eta[:, 2][bad][0])
        raise GradientUndefinedError(
            f"pose is gimbal-degenerate: |sin(phi)| <= {MIN_ABS_SIN_PHI} at phi={phi}")


def pixel_offsets(height: int, width: int, pitch_x: float, pitch_y: float):
    """a_h, a_w in mm (geometry.py:152-157); host-side float64 lists."""
    a_h = [(h - (height - 1) / 2.0) * pitch_y for h in range(height)]
    a_w = [(w - (width - 1) / 2.0) * pitch_x for w in range(width)]
    return a_h, a_w


def volume_center(dims, spacing, origin):
    """Physical centre of a grid (volume.py:71-74)."""
    return tuple(b + 0.5 * n * s for b, n, s in zip(origin, dims, spacing))


def canonical_sdr_to_rho(sdr: float) -> float:
    """North-star ``sdr`` is the source-to-detector RADIUS, i.e. the reference's
    rho (half the source-detector distance)."""
    if not (sdr > 0 and math.isfinite(sdr)):
        raise InvalidArgumentError(f"sdr must be positive, got {sdr}")
    return float(sdr)
