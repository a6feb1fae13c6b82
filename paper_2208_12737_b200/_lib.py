"""ctypes binding of the C ABI in ``include/drr_b200.h``.

The shared library ``_lib/libdrr_b200.so`` is built in-tree by
``paper_2208_12737_b200.build`` (nvcc, sm_100a).  There is no fallback: if the
library is missing every entry point raises, so a GPU run can never silently
route through anything but the CUDA kernels.
"""

from __future__ import annotations

import ctypes
import os

from .errors import GradientUndefinedError, InvalidArgumentError, KernelError

LIB_PATH = os.environ.get("DRR_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libdrr_b200.so")

DRR_OK = 0
DRR_ERR_INVALID_ARGUMENT = -1
DRR_ERR_CUDA = -2
DRR_ERR_GRADIENT_UNDEFINED = -3
DRR_ERR_WORKSPACE = -4

DRR_VOL_F32 = 0
DRR_VOL_F64 = 1

# Every symbol include/drr_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "drr_last_error",
    "drr_version",
    "drr_struct_sizes",
    "drr_raysum",
    "drr_raysum_endpoint_grad",
    "drr_raysum_tangents",
    "drr_forward",
    "drr_backward_workspace_size",
    "drr_backward",
    "drr_forward_jac",
    "drr_backward_jac",
    "drr_count_steps",
    "drr_volume_pack",
    "drr_volume_bounds",
    "drr_volume_hull_dirs",
    "drr_volume_hull",
    "drr_signature",
    "drr_ray_signatures",
    "drr_pose_frames",
    "drr_pose_grad",
    "drr_image_loss",
    "drr_register_update",
    "drr_register_step",
    "drr_loss_grad_jac",
    "drr_loss_grad_workspace_size",
    "drr_forward_loss_grad",
    "drr_peer_export",
    "drr_peer_open",
    "drr_peer_close",
)


class DrrGrid(ctypes.Structure):
    _fields_ = [("dims", ctypes.c_int64 * 3),
                ("spacing", ctypes.c_double * 3),
                ("origin", ctypes.c_double * 3),
                ("occ_lo", ctypes.c_int64 * 3),
                ("occ_hi", ctypes.c_int64 * 3),
                ("hull_valid", ctypes.c_int32),
                ("hull_lo", ctypes.c_int32 * 16),
                ("hull_hi", ctypes.c_int32 * 16)]


class DrrRegConfig(ctypes.Structure):
    _fields_ = [("lr_rotation", ctypes.c_double),
                ("lr_translation", ctypes.c_double),
                ("momentum", ctypes.c_double),
                ("converged_threshold", ctypes.c_double),
                ("max_iters", ctypes.c_int32)]


class DrrDetector(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32),
                ("width", ctypes.c_int32),
                ("pitch_x", ctypes.c_double),
                ("pitch_y", ctypes.c_double),
                ("ray_split", ctypes.c_int32)]


class DrrPeerHandle(ctypes.Structure):
    _fields_ = [("ipc", ctypes.c_ubyte * 64),
                ("offset", ctypes.c_uint64),
                ("bytes", ctypes.c_uint64)]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_int = ctypes.c_int
_sz = ctypes.c_size_t
_GP = ctypes.POINTER(DrrGrid)
_DP = ctypes.POINTER(DrrDetector)

_SIGNATURES = {
    "drr_last_error": ([], ctypes.c_char_p),
    "drr_version": ([], _int),
    "drr_struct_sizes": ([_vp, _vp, _vp, _vp], _int),
    "drr_raysum": ([_vp, _int, _GP, _vp, _vp, _i64, _vp, _vp], _int),
    "drr_raysum_endpoint_grad": ([_vp, _int, _GP, _vp, _vp, _i64, _vp, _vp, _vp, _vp], _int),
    "drr_raysum_tangents": ([_vp, _int, _GP, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp],
                            _int),
    "drr_forward": ([_vp, _int, _GP, _vp, _i32, _DP, _vp, _int, _vp], _int),
    "drr_backward_workspace_size": ([_i32, _DP], _sz),
    "drr_backward": ([_vp, _int, _GP, _vp, _i32, _DP, _vp, _int, _vp, _vp, _int, _vp, _sz, _vp], _int),
    "drr_forward_jac": ([_vp, _int, _GP, _vp, _i32, _DP, _vp, _int, _vp, _vp], _int),
    "drr_backward_jac": ([_vp, _i32, _DP, _vp, _int, _vp, _vp, _sz, _vp], _int),
    "drr_count_steps": ([_vp, _int, _GP, _vp, _i32, _DP, _vp, _vp], _int),
    "drr_volume_pack": ([_vp, _int, _int, ctypes.POINTER(_i64), _int, _vp, _int, _vp], _int),
    "drr_volume_hull_dirs": ([], _int),
    "drr_volume_hull": ([_vp, _int, _GP, _vp, _vp], _int),
    "drr_volume_bounds": ([_vp, _int, _GP, _vp, _vp], _int),
    "drr_signature": ([_vp, _int, _GP, _vp, _i32, _DP, _vp, _vp], _int),
    "drr_ray_signatures": ([_vp, _int, _GP, _vp, _i32, _DP, _vp, _vp], _int),
    "drr_pose_frames": ([_vp, _i32, ctypes.POINTER(ctypes.c_double), _vp, _vp], _int),
    "drr_pose_grad": ([_vp, _vp, _i32, _vp, _vp], _int),
    "drr_image_loss": ([_vp, _vp, _int, _i64, _i32, _i64, _int, _vp, _vp, _vp, _vp], _int),
    "drr_register_update": ([_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(DrrRegConfig), _i32,
                             _vp, _vp, _vp, _vp, _i32, _vp], _int),
    "drr_loss_grad_workspace_size": ([_i32, _DP], _sz),
    "drr_loss_grad_jac": ([_vp, _vp, _vp, _int, _i64, _i32, _DP, _int, _vp, _vp, _vp, _vp, _vp,
                           _vp], _int),
    "drr_forward_loss_grad": ([_vp, _int, _GP, _vp, _vp, _i32, _DP, _vp, _i64, _int, _vp, _int,
                               _vp, _vp, _vp, _vp, _vp, _sz, _vp], _int),
    "drr_register_step": ([_vp, _int, _GP, _vp, _vp, _vp, _i32, _DP, _vp, _i64, _int, _vp, _int,
                           _vp, _vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(DrrRegConfig),
                           _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp], _int),
    "drr_peer_export": ([_vp, ctypes.POINTER(DrrPeerHandle)], _int),
    "drr_peer_open": ([ctypes.POINTER(DrrPeerHandle), ctypes.POINTER(_vp)], _int),
    "drr_peer_close": ([_vp, ctypes.c_uint64], _int),
}

DRR_SRC_F32, DRR_SRC_F64, DRR_SRC_I16, DRR_SRC_U8 = 0, 1, 2, 3
DRR_ORDER_XFASTEST, DRR_ORDER_ZFASTEST = 0, 1

DRR_LOSS_NEG_ZNCC = 0
DRR_LOSS_L2 = 1
DRR_REG_RUNNING, DRR_REG_CONVERGED, DRR_REG_FAILED, DRR_REG_DONE = 0, 1, 2, 3

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the native library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"native DRR library not built: {path} is missing; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _check_layouts(lib)
    _lib = lib
    return lib


def _check_layouts(lib) -> None:
    """The ctypes mirrors must have the library's struct sizes (a stale
    library or binding would otherwise pass misaligned arguments)."""
    got = [ctypes.c_size_t() for _ in range(4)]
    lib.drr_struct_sizes(*[ctypes.byref(g) for g in got])
    want = [ctypes.sizeof(t) for t in (DrrGrid, DrrDetector, DrrRegConfig, DrrPeerHandle)]
    if [g.value for g in got] != want:
        raise ImportError(f"{LIB_PATH}: ABI struct sizes {[g.value for g in got]} differ from "
                          f"the ctypes layouts {want}; rebuild the library")


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception classes."""
    if rc == DRR_OK:
        return
    msg = load().drr_last_error().decode("utf-8", "replace")
    if rc == DRR_ERR_INVALID_ARGUMENT:
        raise InvalidArgumentError(msg)
    if rc == DRR_ERR_GRADIENT_UNDEFINED:
        raise GradientUndefinedError(msg)
    raise KernelError(f"drr status {rc}: {msg}")


def make_grid(dims, spacing, origin, occupied=None, hull=None) -> DrrGrid:
    """The C grid; ``occupied`` = ((lo0, lo1, lo2), (hi0, hi1, hi2)), the voxel
    box outside of which the volume is exactly zero (None: the whole volume);
    ``hull`` = (lo[n], hi[n]) from drr_volume_hull (None: box only)."""
    g = DrrGrid()
    if hull is not None:
        g.hull_valid = len(hull[0])
        for q in range(len(hull[0])):
            g.hull_lo[q] = int(hull[0][q])
            g.hull_hi[q] = int(hull[1][q])
    for a in range(3):
        g.dims[a] = int(dims[a])
        g.spacing[a] = float(spacing[a])
        g.origin[a] = float(origin[a])
        g.occ_lo[a] = int(occupied[0][a]) if occupied is not None else 0
        g.occ_hi[a] = int(occupied[1][a]) if occupied is not None else 0
    return g


def make_detector(height, width, pitch_x, pitch_y, ray_split: int = 0) -> DrrDetector:
    d = DrrDetector()
    d.height = int(height)
    d.width = int(width)
    d.pitch_x = float(pitch_x)
    d.pitch_y = float(pitch_y)
    d.ray_split = int(ray_split)
    return d
