"""Deterministic synthetic inputs for tests and the benchmark.

* ``make_phantom`` restates the reference's test phantoms
  (``pkg/src/drrtrace/volume.py:93-140``) as an (nx, ny, nz) float64 array;
* ``chest_phantom`` is the "chest-CT-shaped" volume SURVEY.md section 8(d)
  fixes for the benchmark configs (body ellipse, two lungs, spine, noise);
* ``sample_poses`` restates ``registration.sample_initializations``
  (``registration.py:128-141``) with the narrow half-widths (``:29-35``).
"""

from __future__ import annotations

import math

import numpy as np

NARROW_HALF_WIDTHS = (0.0, math.radians(45.0), math.radians(45.0), math.radians(22.5),
                      15.0, 15.0, 15.0)


def make_phantom(kind: str, dims, spacing=1.0, density: float = 1.0,
                 origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    if np.isscalar(dims):
        dims = (dims, dims, dims)
    dims = tuple(int(n) for n in dims)
    spacing = tuple(float(s) for s in np.broadcast_to(np.asarray(spacing, float), (3,)))
    origin = tuple(float(s) for s in np.broadcast_to(np.asarray(origin, float), (3,)))
    data = np.zeros(dims, dtype=np.float64, order="F")
    if kind == "uniform":
        data[:] = density
    elif kind == "single_voxel":
        data[dims[0] // 2, dims[1] // 2, dims[2] // 2] = density
    elif kind == "sphere":
        centers = [origin[a] + (np.arange(dims[a]) + 0.5) * spacing[a] for a in range(3)]
        extent = [n * s for n, s in zip(dims, spacing)]
        mid = [b + 0.5 * e for b, e in zip(origin, extent)]
        radius = 0.4 * min(extent)
        r2 = (np.square(centers[0] - mid[0])[:, None, None]
              + np.square(centers[1] - mid[1])[None, :, None]
              + np.square(centers[2] - mid[2])[None, None, :])
        data[r2 <= radius * radius] = density
    elif kind == "off_center_cube":
        box = [((np.arange(dims[a]) + 0.5) / dims[a] >= 0.25) &
               ((np.arange(dims[a]) + 0.5) / dims[a] <= 0.5) for a in range(3)]
        data[box[0][:, None, None] & box[1][None, :, None] & box[2][None, None, :]] = density
    else:
        raise ValueError(f"unknown phantom kind {kind!r}")
    return data


def blob_phantom(n: int = 64, spacing: float = 4.0) -> np.ndarray:
    """Sphere + 3x off-centre cube (the reference acceptance suite's blob64,
    test_acceptance.py:25-30, generalised in size)."""
    return make_phantom("sphere", n, spacing) + make_phantom("off_center_cube", n, spacing, 3.0)


def chest_phantom(dims=(512, 512, 133), seed: int = 0, dtype=np.float32) -> np.ndarray:
    """SURVEY.md 8(d) chest-shaped volume, (nx, ny, nz) array."""
    nx, ny, nz = dims
    x = (np.arange(nx) + 0.5) / nx - 0.5
    y = (np.arange(ny) + 0.5) / ny - 0.5
    X, Y = np.meshgrid(x, y, indexing="ij")
    body = (X / 0.45) ** 2 + (Y / 0.35) ** 2 <= 1.0
    lungs = ((((X - 0.18) / 0.14) ** 2 + (Y / 0.2) ** 2 <= 1.0) |
             (((X + 0.18) / 0.14) ** 2 + (Y / 0.2) ** 2 <= 1.0)) & body
    spine = (X / 0.05) ** 2 + ((Y + 0.25) / 0.05) ** 2 <= 1.0
    sl = np.zeros((nx, ny), dtype=np.float64)
    sl[body] = 1.0
    sl[lungs] = 0.2
    sl[spine] = 2.0
    vol = np.repeat(sl[:, :, None], nz, axis=2)
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal(size=vol.shape)
    vol = np.where(body[:, :, None], vol + 0.01 * noise, vol)
    return np.clip(vol, 0.0, None).astype(dtype)


def sample_poses(truth, half_widths, n: int, seed: int) -> np.ndarray:
    """(n, 7) uniform samples around ``truth`` (registration.py:128-141)."""
    center = np.asarray(truth, dtype=np.float64)
    hw = np.broadcast_to(np.asarray(half_widths, dtype=np.float64), (7,))
    rng = np.random.default_rng(seed)
    return rng.uniform(center - hw, center + hw, size=(n, 7))
