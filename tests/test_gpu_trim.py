"""Occupied-box trimming (drr_volume_bounds; GridDev tlo / thi): the walks
skip the exactly-zero margins of the volume, and every output must be
bit-identical to the reference's whole-volume walk -- images, ray Jacobians,
re-walk gradients, fused loss gradients, explicit-ray energies -- at C2 scale
(the chest phantom's air margins), for a single split pose, and on volumes
whose occupied box touches or misses the faces; the box itself against numpy
(NaN counts as occupied, -0.0 as empty)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TRUTH = (300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)


def _np_bounds(v):
    nz = np.argwhere(~(v == 0))
    if len(nz) == 0:
        return (0, 0, 0), (0, 0, 0)
    return tuple(int(x) for x in nz.min(0)), tuple(int(x) + 1 for x in nz.max(0))


def test_bounds_match_numpy(cuda_device):
    from paper_2208_12737_b200 import DeviceVolume
    rng = np.random.default_rng(0)
    for shape, box in (((17, 9, 12), (slice(3, 7), slice(2, 5), slice(4, 9))),
                       ((5, 5, 5), (slice(1, 3), slice(0, 5), slice(2, 3)))):
        v = np.zeros(shape)
        v[box] = rng.random(v[box].shape) + 0.5
        v[1, shape[1] - 1, shape[2] - 1] = np.nan  # occupied
        v[0, 0, 0] = -0.0                          # empty
        for dtype in (torch.float32, torch.float64):
            dv = DeviceVolume(v, 1.0, device=cuda_device, dtype=dtype)
            assert dv.occupied == _np_bounds(v), (dv.occupied, _np_bounds(v))
    empty = DeviceVolume(np.zeros((4, 4, 4)), 1.0, device=cuda_device)
    assert empty.occupied == ((0, 0, 0), (0, 0, 0))


def _pair(data, spacing, dev, dtype=torch.float32):
    from paper_2208_12737_b200 import DeviceVolume
    a = DeviceVolume(data, spacing, device=dev, dtype=dtype)
    b = DeviceVolume(data, spacing, device=dev, dtype=dtype, trim=False)
    return a, b


def test_c2_trimmed_walks_are_bitwise(cuda_device):
    from paper_2208_12737_b200 import (Detector, backward_frames, backward_from_jac, count_steps,
                                       pose_frames, render_frames, render_frames_jac, synthetic)
    chest = synthetic.chest_phantom()
    tv, fv = _pair(chest, (0.703125, 0.703125, 2.5), cuda_device)
    assert tv.occupied != ((0, 0, 0), tuple(chest.shape))  # the phantom has air margins
    det = Detector(200, 200, 3.6)
    eta = torch.tensor(synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, 12, seed=4),
                       device=cuda_device)
    fr = pose_frames(eta, tv.center).detach()
    for vol_a, vol_b in ((tv, fv),):
        ia, ja = render_frames_jac(vol_a, det, fr)
        ib, jb = render_frames_jac(vol_b, det, fr)
        torch.testing.assert_close(ia, ib, rtol=0, atol=0)
        torch.testing.assert_close(ja, jb, rtol=0, atol=0)
        torch.testing.assert_close(render_frames(vol_a, det, fr), render_frames(vol_b, det, fr),
                                   rtol=0, atol=0)
        g = torch.randn((12, 200, 200), device=cuda_device)
        torch.testing.assert_close(backward_frames(vol_a, det, fr, g),
                                   backward_frames(vol_b, det, fr, g), rtol=0, atol=0)
        torch.testing.assert_close(backward_from_jac(det, ja, g), backward_from_jac(det, jb, g),
                                   rtol=0, atol=0)
    sa = count_steps(tv, det, fr).sum().item()
    sb = count_steps(tv, det, fr, full=True).sum().item()
    assert sb == count_steps(fv, det, fr).sum().item() and sa < sb
    # one pose: the ray is split over 4 lanes at dominant-axis crossings of the
    # range it walks, so trimming moves the cuts -- the same segments summed in
    # other groups (the split walk's own ~1e-16 summation-order freedom);
    # images stay bitwise, Jacobians agree to 1e-11 relative
    one = fr[:1].contiguous()
    ia, ja = render_frames_jac(tv, det, one)
    ib, jb = render_frames_jac(fv, det, one)
    torch.testing.assert_close(ia, ib, rtol=1e-14, atol=0)
    scale = jb.abs().max(dim=1, keepdim=True).values
    assert bool(((ja - jb).abs() <= 1e-11 * scale).all())


def test_fused_loss_and_explicit_rays_trimmed(cuda_device):
    from paper_2208_12737_b200 import Detector, synthetic
    from paper_2208_12737_b200.registration import loss_and_gradient
    from paper_2208_12737_b200 import backend_cuda
    data = synthetic.blob_phantom(40, 2.0)
    tv, fv = _pair(data, 2.0, cuda_device, torch.float64)
    det = Detector(37, 31, 3.0, ray_split=1)  # one thread per ray: bitwise
    eta = torch.tensor(synthetic.sample_poses((150.0, 0.4, 1.3, 0.1, 0, 0, 0),
                                              synthetic.NARROW_HALF_WIDTHS, 9, seed=2),
                       device=cuda_device)
    fixed = np.random.default_rng(1).random((37, 31)) * 40
    for mode, dt in (("fused", torch.float64), ("fused", torch.float32), ("jac", torch.float32)):
        va, ga = loss_and_gradient(tv, det, eta, fixed, mode=mode, image_dtype=dt)
        vb, gb = loss_and_gradient(fv, det, eta, fixed, mode=mode, image_dtype=dt)
        torch.testing.assert_close(va, vb, rtol=0, atol=0)
        torch.testing.assert_close(ga, gb, rtol=0, atol=0)
    # the plugin backend trims with the cached volume's box: energies equal the
    # reference's native kernel bit for bit (the golden-vector tests check it);
    # here against an untrimmed walk of the same rays
    rng = np.random.default_rng(3)
    flat = data.ravel(order="F").copy()
    flat.flags.writeable = False
    src = np.array([-60.0, 41.0, 33.0])
    pix = np.column_stack([np.full(500, 140.0), rng.uniform(-10, 90, 500), rng.uniform(-10, 90, 500)])
    e_trim = backend_cuda.siddon_raysum(flat, (40, 40, 40), (2.0,) * 3, (0.0,) * 3, src, pix)
    backend_cuda._VOL_CACHE.clear()
    e_full = backend_cuda.siddon_raysum(flat.copy(), (40, 40, 40), (2.0,) * 3, (0.0,) * 3, src, pix)
    np.testing.assert_array_equal(e_trim, e_full)


def test_box_touching_faces_and_parallel_rays(cuda_device):
    """Occupied box on a volume face, and axis-parallel rays grazing / missing it."""
    from paper_2208_12737_b200 import _lib
    data = np.zeros((8, 6, 5))
    data[0:3, 2:6, 1:4] = np.arange(36).reshape(3, 4, 3) + 1.0
    tv, fv = _pair(data, (1.0, 2.0, 1.5), cuda_device, torch.float64)
    assert tv.occupied == ((0, 2, 1), (3, 6, 4))
    src = torch.tensor([-5.0, 4.0, 3.0], dtype=torch.float64, device=cuda_device)
    # rays along x at y on / inside / outside the box face y = 4.0 (index 2), z interior
    ys = [3.9, 4.0, 4.1, 8.0, 11.99, 12.0, 12.5]
    pix = torch.tensor([[20.0, y, 3.0] for y in ys] + [[20.0, 5.0, z] for z in (1.5, 6.0, 0.5)],
                       dtype=torch.float64, device=cuda_device)
    srcs = [torch.tensor([-5.0, y, 3.0], dtype=torch.float64, device=cuda_device) for y in ys]
    lib = _lib.load()
    outs = []
    for vol in (tv, fv):
        res = []
        for i in range(pix.shape[0]):
            s = srcs[i] if i < len(ys) else torch.tensor([-5.0, 5.0, float(pix[i, 2])],
                                                          dtype=torch.float64, device=cuda_device)
            o = torch.empty(1, dtype=torch.float64, device=cuda_device)
            _lib.check(lib.drr_raysum(vol.flat.data_ptr(), vol.vol_dtype, vol.grid, s.data_ptr(),
                                      pix[i:i + 1].contiguous().data_ptr(), 1, o.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
            res.append(float(o[0]))
        outs.append(res)
    np.testing.assert_array_equal(outs[0], outs[1])
