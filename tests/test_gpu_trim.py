"""Exact empty-space trimming: the occupied box (drr_volume_bounds; GridDev
tlo / thi) and the 10-direction hull (drr_volume_hull; hull_trim).  The
walks skip the exactly-zero margins of the volume and of each ray, and every
output must be bit-identical to the reference's whole-volume walk -- images,
ray Jacobians, re-walk gradients, fused loss gradients, explicit-ray
energies -- at C2 scale (the chest phantom's air margins), on a ball in its
bounding cube (C5's shape), on scattered blobs, for a single split pose, and
on volumes whose occupied box touches or misses the faces; the box against
numpy (NaN counts as occupied, -0.0 as empty)."""

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


def test_hull_matches_numpy(cuda_device):
    from paper_2208_12737_b200 import DeviceVolume
    from paper_2208_12737_b200.renderer import volume_bounds
    rng = np.random.default_rng(3)
    v = np.zeros((23, 17, 11))
    idx = (rng.integers(0, 23, 9), rng.integers(0, 17, 9), rng.integers(0, 11, 9))
    v[idx] = rng.random(9) + 0.5
    v[22, 0, 10] = np.nan
    dv = DeviceVolume(v, 1.0, device=cuda_device, trim=False)
    box, hull = volume_bounds(dv.flat, dv.grid, dv.vol_dtype, hull=True)
    dirs = np.array([[1, 1, 0], [1, -1, 0], [1, 0, 1], [1, 0, -1], [0, 1, 1], [0, 1, -1],
                     [1, 1, 1], [1, 1, -1], [1, -1, 1], [-1, 1, 1],
                     [2, 1, 0], [1, 2, 0], [2, -1, 0], [1, -2, 0]])
    occ = np.argwhere(~(v == 0))
    dots = occ @ dirs.T
    assert hull == (tuple(int(x) for x in dots.min(0)), tuple(int(x) for x in dots.max(0)))
    assert box == _np_bounds(v)


def _pair(data, spacing, dev, dtype=torch.float32):
    from paper_2208_12737_b200 import DeviceVolume
    a = DeviceVolume(data, spacing, device=dev, dtype=dtype)
    b = DeviceVolume(data, spacing, device=dev, dtype=dtype, trim=False)
    return a, b


@pytest.mark.parametrize("kind", ["ball", "blobs"])
def test_trim_bitwise_air_inside_box(cuda_device, kind):
    """Shapes with air inside their bounding box (and rays that miss it)."""
    from paper_2208_12737_b200 import (Detector, backward_frames, count_steps, pose_frames,
                                       render_frames, render_frames_jac, synthetic)
    from paper_2208_12737_b200.registration import loss_and_gradient
    n = 64
    if kind == "ball":
        data = synthetic.make_phantom("sphere", n, 1.0) + 3.0 * synthetic.make_phantom(
            "off_center_cube", n, 1.0)
    else:
        rng = np.random.default_rng(9)
        data = np.zeros((n, n, n))
        for _ in range(7):
            c = rng.integers(8, n - 8, 3)
            data[c[0] - 4:c[0] + 4, c[1] - 3:c[1] + 5, c[2] - 5:c[2] + 2] = rng.random() + 0.5
    tv, fv = _pair(data, 1.0, cuda_device)
    from paper_2208_12737_b200 import DeviceVolume
    bv = DeviceVolume(data, 1.0, device=cuda_device, trim="box")
    det = Detector(96, 80, 1.4, ray_split=1)
    eta = torch.tensor(synthetic.sample_poses((120.0, 0.7, 1.1, 0.2, 0, 0, 0),
                                              synthetic.NARROW_HALF_WIDTHS, 6, seed=5),
                       device=cuda_device)
    fr = pose_frames(eta, tv.center).detach()
    ib, jb = render_frames_jac(fv, det, fr)
    for vol in (tv, bv):
        ia, ja = render_frames_jac(vol, det, fr)
        torch.testing.assert_close(ia, ib, rtol=0, atol=0)
        torch.testing.assert_close(ja, jb, rtol=0, atol=0)
    assert count_steps(tv, det, fr).sum() < count_steps(bv, det, fr).sum()
    g = torch.randn((6, 96, 80), device=cuda_device)
    torch.testing.assert_close(backward_frames(tv, det, fr, g), backward_frames(fv, det, fr, g),
                               rtol=0, atol=0)
    fixed = render_frames(fv, det, fr[:1])[0]
    for mode in ("fused", "jac"):
        va, ga = loss_and_gradient(tv, det, eta, fixed, mode=mode)
        vb, gb = loss_and_gradient(fv, det, eta, fixed, mode=mode)
        torch.testing.assert_close(va, vb, rtol=0, atol=0)
        torch.testing.assert_close(ga, gb, rtol=0, atol=0)


def test_trim_sources_inside_volume(cuda_device):
    """A source inside the volume but outside the occupied box (clip entry):
    images stay bitwise; the gradient sums may switch to the derived-axis form
    of the walk when the trimmed start is a plane crossing instead of the clip
    (1e-13)."""
    from paper_2208_12737_b200 import backend_cuda, synthetic
    data = synthetic.blob_phantom(48, 1.0)
    flat = data.ravel(order="F").copy()
    flat.flags.writeable = False
    rng = np.random.default_rng(12)
    src = np.array([3.0, 4.0, 2.5])  # inside the volume, in its air corner
    pix = rng.uniform(-20, 70, (800, 3))
    backend_cuda._VOL_CACHE.clear()
    e_t, s_t, p_t = backend_cuda.ray_endpoint_grad(flat, (48,) * 3, (1.0,) * 3, (0.0,) * 3, src, pix)
    w = flat.copy()  # writeable: uploaded per call; walked untrimmed here
    orig = backend_cuda._bounds
    backend_cuda._bounds = lambda vol, dims: (((0, 0, 0), tuple(int(n) for n in dims)), None)
    try:
        e_f, s_f, p_f = backend_cuda.ray_endpoint_grad(w, (48,) * 3, (1.0,) * 3, (0.0,) * 3, src,
                                                       pix)
    finally:
        backend_cuda._bounds = orig
    np.testing.assert_array_equal(e_t, e_f)
    for a, b in ((s_t, s_f), (p_t, p_f)):
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-13 * np.abs(b).max())


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


@pytest.mark.parametrize("seed", range(6))
def test_trim_randomised_bitwise(cuda_device, seed):
    """Random sparse volumes (a few boxes of random density, some touching the
    faces), random spacings and origins, random poses -- including sources
    inside the volume and rays that graze or miss the occupied hull: images
    and one-thread-per-ray Jacobians of the trimmed walk equal the
    whole-volume walk's bit for bit (sources inside the volume: images
    bitwise, Jacobians to 1e-13 -- the derived-axis form may differ)."""
    from paper_2208_12737_b200 import DeviceVolume, Detector, pose_frames, render_frames_jac
    rng = np.random.default_rng(100 + seed)
    dims = tuple(int(x) for x in rng.integers(12, 40, 3))
    data = np.zeros(dims)
    for _ in range(int(rng.integers(1, 5))):
        lo = [int(rng.integers(0, n - 2)) for n in dims]
        hi = [int(rng.integers(l + 1, n + 1)) for l, n in zip(lo, dims)]
        data[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = rng.random() * 3 + 0.1
    sp = tuple(float(x) for x in rng.uniform(0.5, 2.5, 3))
    origin = tuple(float(x) for x in rng.uniform(-20, 20, 3))
    tv = DeviceVolume(data, sp, origin, device=cuda_device)
    fv = DeviceVolume(data, sp, origin, device=cuda_device, trim=False)
    det = Detector(27, 23, float(rng.uniform(1.0, 4.0)), ray_split=1)
    ext = np.array(dims) * np.array(sp)
    rho = float(rng.uniform(0.3, 1.5)) * float(np.linalg.norm(ext))  # some sources inside
    eta = np.column_stack([np.full(5, rho), rng.uniform(0, 2 * np.pi, 5), rng.uniform(0.2, 2.9, 5),
                           rng.uniform(-1, 1, 5), rng.uniform(-5, 5, (5, 3))])
    fr = pose_frames(torch.tensor(eta, device=cuda_device), tv.center).detach()
    ia, ja = render_frames_jac(tv, det, fr, out_dtype=torch.float64)
    ib, jb = render_frames_jac(fv, det, fr, out_dtype=torch.float64)
    torch.testing.assert_close(ia, ib, rtol=0, atol=0)
    scale = jb.abs().max().clamp_min(1e-300)
    assert bool(((ja - jb).abs() <= 1e-13 * scale).all())
    src = fr[:, :3].cpu().numpy()
    lo_b, hi_b = np.array(origin), np.array(origin) + ext
    outside = ~np.all((src >= lo_b) & (src <= hi_b), axis=1)
    for i in np.nonzero(outside)[0]:  # sources outside the volume: the walk semantics are the same
        n = 27 * 23
        torch.testing.assert_close(ja[:, i * n:(i + 1) * n], jb[:, i * n:(i + 1) * n], rtol=0, atol=0)
