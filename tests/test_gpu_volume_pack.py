"""drr_volume_pack: the one-time ingest into the walk's
x-fastest layout -- from x-fastest or C-ordered (nx, ny, nz) sources, f32 /
f64 / i16 / u8 elements cast without rescaling (volume.py:211-218), optional
negative clamp -- against numpy, bit for bit, at ragged sizes
that exercise every edge of the 32 x 32 transpose tiles."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(1, 1, 1), (33, 5, 70), (64, 31, 32), (7, 100, 3)])
@pytest.mark.parametrize("src", ["f32", "f64", "i16", "u8"])
def test_pack_matches_numpy(cuda_device, dims, src):
    from paper_2208_12737_b200 import _lib
    from paper_2208_12737_b200.renderer import pack_volume
    rng = np.random.default_rng(sum(dims))
    np_t = {"f32": np.float32, "f64": np.float64, "i16": np.int16, "u8": np.uint8}[src]
    if src in ("f32", "f64"):
        data = (rng.standard_normal(dims) * 100).astype(np_t)
    elif src == "i16":
        data = rng.integers(-1000, 2000, dims).astype(np_t)
    else:
        data = rng.integers(0, 255, dims).astype(np_t)
    flat_ref = data.ravel(order="F")  # x-fastest (volume.py:77-79)
    for clamp in (False, True):
        want64 = flat_ref.astype(np.float64)
        if clamp:
            want64 = np.maximum(want64, 0.0)
        for dtype in (torch.float32, torch.float64):
            want = want64.astype(np.float32 if dtype == torch.float32 else np.float64)
            z = pack_volume(torch.from_numpy(np.ascontiguousarray(data)).to(cuda_device), dims,
                            _lib.DRR_ORDER_ZFASTEST, dtype, clamp).cpu().numpy()
            x = pack_volume(torch.from_numpy(np.ascontiguousarray(flat_ref)).to(cuda_device), dims,
                            _lib.DRR_ORDER_XFASTEST, dtype, clamp).cpu().numpy()
            np.testing.assert_array_equal(z, want)
            np.testing.assert_array_equal(x, want)


def test_pack_errors(cuda_device):
    import ctypes
    from paper_2208_12737_b200 import InvalidArgumentError, _lib
    lib = _lib.load()
    buf = torch.zeros(8, device=cuda_device)
    d = (ctypes.c_int64 * 3)(2, 2, 0)
    with pytest.raises(InvalidArgumentError):
        _lib.check(lib.drr_volume_pack(buf.data_ptr(), 0, 0, d, 0, buf.data_ptr(), 0, None))
    d = (ctypes.c_int64 * 3)(2, 2, 2)
    with pytest.raises(InvalidArgumentError):
        _lib.check(lib.drr_volume_pack(buf.data_ptr(), 9, 0, d, 0, buf.data_ptr(), 0, None))
    with pytest.raises(InvalidArgumentError):
        _lib.check(lib.drr_volume_pack(buf.data_ptr(), 0, 5, d, 0, buf.data_ptr(), 0, None))
