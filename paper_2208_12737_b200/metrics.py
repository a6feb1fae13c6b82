"""Image-similarity losses on the device (restating ``metrics.py`` of the
reference, ``pkg/src/drrtrace/metrics.py:26-91``).

``neg_zncc`` uses the population standard deviation (``metrics.py:26-31``) and
clips the correlation to [-1, 1] (``metrics.py:48-49``); its analytic pixel
gradient is -(b_hat - raw a_hat) / (N sigma_a) (``metrics.py:78-84``).

On the device, for float32 moving AND fixed images, both losses run as one
fused kernel (``drr_image_loss``: value and the reference's analytic pixel
gradient, ``loss_value_and_pixel_grad``) wrapped in an autograd Function;
elsewhere (host tensors, float64 images -- which the kernel would otherwise
round -- a fixed image that requires grad) they are plain differentiable torch
with the same value.  An undefined ZNCC (a constant image, metrics.py:29-30)
gives NaN value and NaN gradient on both paths.
"""

from __future__ import annotations

import torch

from .errors import InvalidArgumentError

LOSS_KINDS = ("neg_zncc", "l2")


def _standardize(x: torch.Tensor):
    mu = x.mean(dim=(-2, -1), keepdim=True)
    sigma = torch.sqrt(((x - mu) ** 2).mean(dim=(-2, -1), keepdim=True))
    return (x - mu) / sigma, sigma


class _ImageLoss(torch.autograd.Function):
    """Value (B,) float64 and stored pixel gradient from ``drr_image_loss``;
    backward scales the stored gradient by the upstream value gradient."""

    @staticmethod
    def forward(ctx, moving, fixed, kind):
        from . import _lib
        single = moving.ndim == 2
        m = moving.detach().reshape(-1, *moving.shape[-2:]).contiguous()
        B, npix = m.shape[0], m.shape[-2] * m.shape[-1]
        f = fixed.detach()
        if f.ndim == 3 and f.shape[0] == 1:
            f = f[0]
        if f.ndim == 3 and f.shape[0] != B:
            raise InvalidArgumentError(f"need 1 or {B} fixed images, got {f.shape[0]}")
        f = f.contiguous()
        stride = 0 if f.ndim == 2 else npix
        value = torch.empty(B, dtype=torch.float64, device=m.device)
        grad = torch.empty_like(m)
        lib = _lib.load()
        _lib.check(lib.drr_image_loss(m.data_ptr(), f.data_ptr(), 0, stride, B, npix,
                                      _lib.DRR_LOSS_NEG_ZNCC if kind == "neg_zncc" else _lib.DRR_LOSS_L2,
                                      value.data_ptr(), grad.data_ptr(), None,
                                      torch.cuda.current_stream(m.device).cuda_stream))
        ctx.save_for_backward(grad)
        ctx.shape = moving.shape
        return value[0] if single else value

    @staticmethod
    def backward(ctx, grad_value):
        (grad,) = ctx.saved_tensors
        g = grad_value.reshape(-1, 1, 1).to(grad.dtype) * grad
        return g.reshape(ctx.shape), None, None


def _fused_ok(moving: torch.Tensor, fixed: torch.Tensor) -> bool:
    """One fixed image, or one per moving image (no other broadcasting)."""
    if not (moving.is_cuda and moving.dtype == torch.float32 and moving.ndim in (2, 3)):
        return False
    if not isinstance(fixed, torch.Tensor) or fixed.requires_grad:
        return False
    if fixed.dtype != torch.float32 or fixed.device != moving.device:
        return False
    B = moving.shape[0] if moving.ndim == 3 else 1
    return fixed.ndim == 2 or (fixed.ndim == 3 and fixed.shape[0] in (1, B) and moving.ndim == 3)


def neg_zncc(moving: torch.Tensor, fixed: torch.Tensor) -> torch.Tensor:
    """Per-image -ZNCC over the last two dims (B,) ; -1 at a perfect match."""
    if moving.shape[-2:] != fixed.shape[-2:]:
        raise InvalidArgumentError(f"image shapes differ: {tuple(moving.shape)} vs {tuple(fixed.shape)}")
    if _fused_ok(moving, fixed):
        return _ImageLoss.apply(moving, fixed, "neg_zncc")
    a_hat, _ = _standardize(moving.to(torch.float64))
    b_hat, _ = _standardize(fixed.to(torch.float64))
    raw = (a_hat * b_hat).mean(dim=(-2, -1))
    return -torch.clamp(raw, -1.0, 1.0)


def l2(moving: torch.Tensor, fixed: torch.Tensor) -> torch.Tensor:
    """Per-image Euclidean norm of the difference (metrics.py:56-59)."""
    if moving.shape[-2:] != fixed.shape[-2:]:
        raise InvalidArgumentError(f"image shapes differ: {tuple(moving.shape)} vs {tuple(fixed.shape)}")
    if _fused_ok(moving, fixed):
        return _ImageLoss.apply(moving, fixed, "l2")
    diff = (moving.to(torch.float64) - fixed.to(torch.float64))
    return torch.sqrt((diff * diff).sum(dim=(-2, -1)))


def loss(kind: str, moving: torch.Tensor, fixed: torch.Tensor) -> torch.Tensor:
    if kind == "neg_zncc":
        return neg_zncc(moving, fixed)
    if kind == "l2":
        return l2(moving, fixed)
    raise InvalidArgumentError(f"loss kind must be one of {LOSS_KINDS}, got {kind!r}")
