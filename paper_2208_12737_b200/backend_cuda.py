"""Kernel-protocol backend ``"cuda"``: the reference's plugin boundary.

The reference selects its hot kernels with ``drrtrace._kernels.get_backend``
(``pkg/src/drrtrace/_kernels/__init__.py:40-51``); a backend is a module with
``BACKEND_NAME`` and three functions over a flat x-fastest float64 volume and
numpy rays (``_native.pyx:140,196,285``; ``python_ref.py:130,141,204``).  This
module has exactly that surface, so the reference's callers
(``raytrace.ray_energies``, ``ray_energies_with_tangents``) and its tests
(``test_kernel_properties.py``) run unchanged against the GPU:

* ``siddon_raysum``      -> ``drr_raysum`` (one CUDA walk per ray);
* ``siddon_raysum_grad`` -> ``drr_raysum_endpoint_grad`` + the contraction
  d_energy[r, t] = dE/ds_r . d_source[:, t] + dE/dp_r . d_pixels[r, :, t]
  (on the device, torch f64);
* ``jacobs_raysum``      -> the same walk: the GPU traversal already advances
  plane by plane, so the reference's iterative oracle and its vectorised
  kernel coincide here (the reference requires them to agree within 1e-9,
  ``test_raytrace.py:143-148``).

The volume stays float64 on this path (``DRR_VOL_F64``) so energies are
bit-identical to the reference's native backend.  Inputs are coerced with
``np.ascontiguousarray(..., float64)`` like the reference (``_native.pyx:142-145``);
outputs are fresh numpy arrays owned by the caller.

The reference's dispatchers call a backend once per chunk of rays
(``raytrace.py:96-103,122-128``: 16384 rays, 2048 for the gradient) with the
same ``volume.flat_data()`` each time, so the device copy of a READ-ONLY flat
volume (the reference's ``Volume`` freezes its data, ``volume.py:52``) is
cached, keyed on its buffer and geometry; a writeable array is uploaded on
every call (its contents may change between calls).
"""

from __future__ import annotations

import warnings

import numpy as np
import torch

from . import _lib
from .errors import KernelError

BACKEND_NAME = "cuda"


def _device():
    if not torch.cuda.is_available():
        raise KernelError("the cuda backend needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _upload(arr, dev):
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    with warnings.catch_warnings():  # read-only host arrays are only read (copied to the device)
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr).to(dev)


# (buffer address, bytes, dtype, dims, device) -> (the host array, kept alive so
# the address cannot be reused while cached; its device copy); last few volumes
_VOL_CACHE: dict = {}
_VOL_CACHE_MAX = 2


def _device_volume(flat_data, dims, dev):
    """(device volume, its occupied box) -- cached for read-only volumes."""
    arr = np.asarray(flat_data).reshape(-1)
    if arr.flags.writeable:
        d = _upload(arr, dev)
        return d, _bounds(d, dims)
    key = (arr.__array_interface__["data"][0], arr.nbytes, arr.dtype.str,
           tuple(int(n) for n in dims), str(dev))
    hit = _VOL_CACHE.get(key)
    if hit is not None:
        return hit[1]
    while len(_VOL_CACHE) >= _VOL_CACHE_MAX:
        _VOL_CACHE.pop(next(iter(_VOL_CACHE)))
    d = _upload(arr, dev)
    _VOL_CACHE[key] = (arr, (d, _bounds(d, dims)))
    return _VOL_CACHE[key][1]


def _bounds(vol, dims):
    """(occupied box, hull) of a device volume (drr_volume_bounds / _hull)."""
    from .renderer import volume_bounds
    return volume_bounds(vol, _lib.make_grid(dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)),
                         _lib.DRR_VOL_F64, hull=True)


def _prep(flat_data, dims, spacing, origin, source, pixels):
    dev = _device()
    pix = np.ascontiguousarray(np.atleast_2d(pixels), dtype=np.float64)
    vol, (occupied, hull) = _device_volume(flat_data, dims, dev)
    grid = _lib.make_grid(dims, spacing, origin, occupied, hull)
    src = _upload(np.asarray(source).reshape(3), dev)
    return dev, grid, vol, src, _upload(pix, dev), pix.shape[0]


def siddon_raysum(flat_data, dims, spacing, origin, source, pixels):
    """Energies (N,) float64 -- contract of ``_native.siddon_raysum``."""
    dev, grid, vol, src, pix, n = _prep(flat_data, dims, spacing, origin, source, pixels)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.drr_raysum(vol.data_ptr(), _lib.DRR_VOL_F64, grid, src.data_ptr(),
                              pix.data_ptr(), n, out.data_ptr(),
                              torch.cuda.current_stream(dev).cuda_stream))
    return out.cpu().numpy()


def siddon_raysum_grad(flat_data, dims, spacing, origin, source, d_source,
                       pixels, d_pixels):
    """(energy (N,), d_energy (N, T)) -- contract of ``_native.siddon_raysum_grad``."""
    dev, grid, vol, src, pix, n = _prep(flat_data, dims, spacing, origin, source, pixels)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    dEds = torch.empty((n, 3), dtype=torch.float64, device=dev)
    dEdp = torch.empty((n, 3), dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.drr_raysum_endpoint_grad(
        vol.data_ptr(), _lib.DRR_VOL_F64, grid, src.data_ptr(), pix.data_ptr(), n,
        out.data_ptr(), dEds.data_ptr(), dEdp.data_ptr(),
        torch.cuda.current_stream(dev).cuda_stream))
    dsrc = _upload(d_source, dev)                              # (3, T)
    dpix = _upload(d_pixels, dev).reshape(n, 3, -1)            # (N, 3, T)
    d_energy = dEds @ dsrc + torch.einsum("na,nat->nt", dEdp, dpix)
    return out.cpu().numpy(), d_energy.cpu().numpy()


def jacobs_raysum(flat_data, dims, spacing, origin, source, pixels):
    """Iterative variant (``_native.pyx:285-382``): the same incremental walk."""
    return siddon_raysum(flat_data, dims, spacing, origin, source, pixels)


def ray_endpoint_grad(flat_data, dims, spacing, origin, source, pixels):
    """(energy, dE/ds (N, 3), dE/dp (N, 3)) -- the reverse-mode form."""
    dev, grid, vol, src, pix, n = _prep(flat_data, dims, spacing, origin, source, pixels)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    dEds = torch.empty((n, 3), dtype=torch.float64, device=dev)
    dEdp = torch.empty((n, 3), dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.drr_raysum_endpoint_grad(
        vol.data_ptr(), _lib.DRR_VOL_F64, grid, src.data_ptr(), pix.data_ptr(), n,
        out.data_ptr(), dEds.data_ptr(), dEdp.data_ptr(),
        torch.cuda.current_stream(dev).cuda_stream))
    return out.cpu().numpy(), dEds.cpu().numpy(), dEdp.cpu().numpy()
