"""Image-similarity losses on the device (restating ``metrics.py`` of the
reference, ``pkg/src/drrtrace/metrics.py:26-91``).

``neg_zncc`` uses the population standard deviation (``metrics.py:26-31``) and
clips the correlation to [-1, 1] (``metrics.py:48-49``); its analytic pixel
gradient is -(b_hat - raw a_hat) / (N sigma_a) (``metrics.py:78-84``).  Written
as plain differentiable torch so autograd produces the same pixel gradient that
``drr_backward`` consumes.
"""

from __future__ import annotations

import torch

from .errors import InvalidArgumentError

LOSS_KINDS = ("neg_zncc", "l2")


def _standardize(x: torch.Tensor):
    mu = x.mean(dim=(-2, -1), keepdim=True)
    sigma = torch.sqrt(((x - mu) ** 2).mean(dim=(-2, -1), keepdim=True))
    return (x - mu) / sigma, sigma


def neg_zncc(moving: torch.Tensor, fixed: torch.Tensor) -> torch.Tensor:
    """Per-image -ZNCC over the last two dims (B,) ; -1 at a perfect match."""
    if moving.shape[-2:] != fixed.shape[-2:]:
        raise InvalidArgumentError(f"image shapes differ: {tuple(moving.shape)} vs {tuple(fixed.shape)}")
    a_hat, _ = _standardize(moving.to(torch.float64))
    b_hat, _ = _standardize(fixed.to(torch.float64))
    raw = (a_hat * b_hat).mean(dim=(-2, -1))
    return -torch.clamp(raw, -1.0, 1.0)


def l2(moving: torch.Tensor, fixed: torch.Tensor) -> torch.Tensor:
    """Per-image Euclidean norm of the difference (metrics.py:56-59)."""
    diff = (moving.to(torch.float64) - fixed.to(torch.float64))
    return torch.sqrt((diff * diff).sum(dim=(-2, -1)))


def loss(kind: str, moving: torch.Tensor, fixed: torch.Tensor) -> torch.Tensor:
    if kind == "neg_zncc":
        return neg_zncc(moving, fixed)
    if kind == "l2":
        return l2(moving, fixed)
    raise InvalidArgumentError(f"loss kind must be one of {LOSS_KINDS}, got {kind!r}")
