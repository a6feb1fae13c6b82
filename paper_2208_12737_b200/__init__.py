"""paper_2208_12737_b200: a B200-native vectorised-Siddon DRR renderer.

Drop-in for the hot path of arXiv 2208.12737 (DiffDRR) as restated by the
reference package ``drrtrace``: ``DRR(volume, spacing, sdr, height, delx)``
(north-star module API), ``api`` (drrtrace's functional API: render,
render_with_gradient, loss_and_gradient, register, with its types) and the
``"cuda"`` kernel-protocol backend (the reference's ``_kernels.get_backend``
plugin boundary).  All compute runs in
hand-written sm_100a CUDA behind the C ABI of ``include/drr_b200.h``.
"""

from .errors import (DegenerateRayError, DrrTraceError, GradientUndefinedError,
                     InvalidArgumentError, KernelError, MetricUndefinedError)
from .geometry import POSE_PARAM_NAMES, pose_frames
from .renderer import (DRR, DeviceVolume, Detector, backward_frames, backward_from_jac, count_steps,
                       render_frames, render_frames_jac, render_pose_vectors)

__all__ = [
    "DRR", "DeviceVolume", "Detector", "render_frames", "backward_frames",
    "render_frames_jac", "backward_from_jac",
    "count_steps", "render_pose_vectors", "pose_frames", "POSE_PARAM_NAMES",
    "DrrTraceError", "InvalidArgumentError", "DegenerateRayError",
    "MetricUndefinedError", "GradientUndefinedError", "KernelError",
]
