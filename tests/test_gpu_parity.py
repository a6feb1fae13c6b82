"""GPU parity: the CUDA path against the reference's golden outputs and the
C oracle (oracle/siddon_oracle.c, itself pinned to the reference by
tests/test_oracle.py).  Bars (BASELINE.json north_star / SURVEY 8(d)):
images per-pixel relative error <= 1e-4 (we assert bit-identity where the
inputs are identical), pose gradients <= 1e-3 relative with the SURVEY floor.
"""

import math

import numpy as np
import pytest
import torch

from conftest import kernel_case, slab_chord_length
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _backend():
    from paper_2208_12737_b200 import backend_cuda
    return backend_cuda


def grad_close(g, ref, rtol=1e-3):
    """|g - ref| <= rtol * max(|ref|, 1e-3 * ||ref||) per component."""
    g, ref = np.asarray(g), np.asarray(ref)
    floor = 1e-3 * np.linalg.norm(ref)
    return np.all(np.abs(g - ref) <= rtol * np.maximum(np.abs(ref), floor)), \
        np.max(np.abs(g - ref) / np.maximum(np.abs(ref), floor))


# ------------------------------------------------------------ kernel protocol
def test_kernel_cases_bitwise(golden, cuda_device):
    """64 random volumes x 8 rays (axis-parallel, corner, face rays included):
    the cuda backend reproduces the reference native backend bit for bit."""
    be = _backend()
    for c in range(int(golden["k_count"])):
        k = kernel_case(golden, c)
        args = (k["flat"], k["dims"], k["spacing"], k["origin"], k["source"], k["pixels"])
        e = be.siddon_raysum(*args)
        np.testing.assert_array_equal(e, k["energy"], err_msg=f"case {c}")
        ej = be.jacobs_raysum(*args)
        scale = max(1.0, float(np.abs(k["energy_jacobs"]).max()))
        np.testing.assert_allclose(ej, k["energy_jacobs"], atol=1e-9 * scale, rtol=0)
        e2, de = be.siddon_raysum_grad(k["flat"], k["dims"], k["spacing"], k["origin"],
                                       k["source"], k["d_source"], k["pixels"], k["d_pixels"])
        np.testing.assert_array_equal(e2, e)
        dscale = max(1.0, float(np.abs(k["d_energy"]).max()))
        np.testing.assert_allclose(de, k["d_energy"], atol=1e-9 * dscale, rtol=0,
                                   err_msg=f"case {c}")


def test_known_answers(golden, cuda_device):
    be = _backend()
    expect = [1.0, math.sqrt(3.0), 0.0, 0.0, 1.0, None]
    for i in range(int(golden["ka_count"])):
        e = be.siddon_raysum(np.ones(1), (1, 1, 1), (1.0,) * 3, (0.0,) * 3,
                             golden[f"ka{i}_source"], golden[f"ka{i}_pixel"])
        np.testing.assert_array_equal(e, golden[f"ka{i}_energy"])
        if expect[i] is not None:
            assert e[0] == pytest.approx(expect[i], abs=1e-12)


def test_uniform_chord_law(cuda_device):
    """test_raytrace.py:102-112: uniform density x slab chord, 1e-10 relative."""
    be = _backend()
    dims, spacing, origin = (8, 10, 12), (1.0, 1.5, 0.75), (-3.0, 1.0, 0.5)
    flat = np.full(int(np.prod(dims)), 2.5)
    rng = np.random.default_rng(7)
    src = rng.uniform(-40, -20, size=3)
    pix = rng.uniform([0, -5, -5], [40, 25, 25], size=(50, 3))
    e = be.siddon_raysum(flat, dims, spacing, origin, src, pix)
    lo = np.asarray(origin)
    hi = lo + np.asarray(dims) * np.asarray(spacing)
    for k in range(50):
        assert e[k] == pytest.approx(2.5 * slab_chord_length(src, pix[k], lo, hi),
                                     rel=1e-10, abs=1e-12)


def test_nan_and_density_scaling(cuda_device):
    be = _backend()
    data = np.ones((2, 2, 2))
    data[0, 1, 1] = np.nan
    flat = data.ravel(order="F")
    hit = be.siddon_raysum(flat, (2, 2, 2), (1.0,) * 3, (0.0,) * 3, [-1.0, 1.5, 1.5], [[3.0, 1.5, 1.5]])
    clean = be.siddon_raysum(flat, (2, 2, 2), (1.0,) * 3, (0.0,) * 3, [-1.0, 0.5, 0.5], [[3.0, 0.5, 0.5]])
    assert math.isnan(hit[0]) and clean[0] == pytest.approx(2.0)
    from paper_2208_12737_b200 import synthetic
    vol = synthetic.make_phantom("sphere", 8, 1.0)
    src = np.array([-5.0, 4.2, 3.9])
    pix = np.array([[12.0, 4.0, 4.1], [12.0, 2.0, 6.0]])
    e1 = be.siddon_raysum(vol.ravel(order="F"), (8,) * 3, (1.0,) * 3, (0.0,) * 3, src, pix)
    e2 = be.siddon_raysum(2.0 * vol.ravel(order="F"), (8,) * 3, (1.0,) * 3, (0.0,) * 3, src, pix)
    np.testing.assert_array_equal(e2, 2.0 * e1)


def test_random_rays_vs_oracle_bitwise(cuda_device):
    """Wider random sweep than the fixtures: cuda backend == C oracle bitwise,
    f64 volumes, including rays built to hit exact ties (integer lattice)."""
    be = _backend()
    rng = np.random.default_rng(11)
    for trial in range(40):
        dims = tuple(int(x) for x in rng.integers(1, 24, 3))
        spacing = rng.uniform(0.3, 3.0, 3) if trial % 2 else np.ones(3)
        origin = rng.uniform(-5, 5, 3) if trial % 3 else np.zeros(3)
        flat = rng.uniform(0, 4, int(np.prod(dims)))
        span = float(max(np.asarray(dims) * spacing))
        lo = origin
        hi = origin + np.asarray(dims) * spacing
        src = rng.uniform(lo - 3 * span, hi + 3 * span)
        if trial % 4 == 0:
            src = np.round(src)
        pix = rng.uniform(lo - 0.5 * span, hi + 0.5 * span, size=(256, 3))
        if trial % 4 == 0:
            pix = np.round(pix)
        pix[0] = 2 * hi - src  # through the far corner region
        e = be.siddon_raysum(flat, dims, spacing, origin, src, pix)
        ref = O.raysum(flat, dims, spacing, origin, src, pix)
        np.testing.assert_array_equal(e, ref, err_msg=f"trial {trial}")
        _, gs, gp = be.ray_endpoint_grad(flat, dims, spacing, origin, src, pix)
        _, rs, rp = O.raysum_endpoint_grad(flat, dims, spacing, origin, src, pix)
        sc = max(1.0, np.abs(rs).max(), np.abs(rp).max())
        np.testing.assert_allclose(gs, rs, atol=1e-10 * sc, rtol=0)
        np.testing.assert_allclose(gp, rp, atol=1e-10 * sc, rtol=0)


# ------------------------------------------------------------ pose / module path
def _vol_from_golden(golden, prefix):
    from paper_2208_12737_b200 import DeviceVolume
    return DeviceVolume.from_flat(golden[prefix + "flat"], golden[prefix + "dims"],
                                  golden[prefix + "spacing"], golden[prefix + "origin"],
                                  dtype=torch.float64)


def test_pose_renders_bitwise(golden, cuda_device):
    """Frames from the oracle's pose_frame -> drr_forward (f64 out) equals the
    reference render() bit for bit, for axis-aligned, oblique, shifted and
    corner-heavy poses (test_raytrace.py:128-137)."""
    from paper_2208_12737_b200 import Detector, render_frames
    vol = _vol_from_golden(golden, "ps_")
    det = Detector(21, 21, 4.0, ray_split=1)
    frames = np.stack([O.pose_frame(eta, golden["ps_center"]) for eta in golden["ps_poses"]])
    img = render_frames(vol, det, torch.tensor(frames, device=cuda_device),
                        out_dtype=torch.float64).cpu().numpy()
    np.testing.assert_array_equal(img, golden["ps_images"])
    # the same through the fp32 product layout (sphere densities are 0/1, exact in fp32)
    vol32 = type(vol).from_flat(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                                golden["ps_origin"])
    img32 = render_frames(vol32, det, torch.tensor(frames, device=cuda_device)).cpu().numpy()
    np.testing.assert_array_equal(img32, golden["ps_images"].astype(np.float32))


def test_module_forward_and_gradient(golden, cuda_device):
    """DRR(volume, spacing, sdr, height, delx) + neg-ZNCC: value and 7-gradient
    against the reference's loss_and_gradient (gradients.py:61-69)."""
    from paper_2208_12737_b200 import DRR
    from paper_2208_12737_b200.metrics import neg_zncc
    dims = tuple(int(n) for n in golden["ps_dims"])
    data = golden["ps_flat"].reshape(dims[::-1]).transpose(2, 1, 0)
    fixed = torch.tensor(golden["ps_fixed"], device=cuda_device)
    for i, eta in enumerate(golden["ps_poses"]):
        if not np.isfinite(golden["ps_values"][i]):
            continue
        drr = DRR(data, 2.0, sdr=float(eta[0]), height=21, delx=4.0, device=cuda_device)
        rot = torch.tensor(eta[1:4], device=cuda_device, requires_grad=True)
        tra = torch.tensor(eta[4:7], device=cuda_device, requires_grad=True)
        sdr = torch.tensor(float(eta[0]), device=cuda_device, dtype=torch.float64,
                           requires_grad=True)
        img = drr(rot, tra, sdr=sdr)
        ref_img = golden["ps_images"][i]
        rel = np.abs(img.detach().cpu().numpy() - ref_img) / np.maximum(
            np.abs(ref_img), 1e-3 * np.abs(ref_img).max())
        assert rel.max() <= 1e-4
        loss = neg_zncc(img, fixed)
        loss.backward()
        assert float(loss) == pytest.approx(golden["ps_values"][i], abs=1e-6)
        g = np.concatenate([[float(sdr.grad)], rot.grad.cpu().numpy(), tra.grad.cpu().numpy()])
        ok, err = grad_close(g, golden["ps_grads"][i])
        assert ok, (i, err, g, golden["ps_grads"][i])


def test_gimbal_pose_rejected(cuda_device):
    from paper_2208_12737_b200 import DRR, GradientUndefinedError, synthetic
    drr = DRR(synthetic.make_phantom("sphere", 16, 2.0), 2.0, 100.0, 21, 4.0, device=cuda_device)
    rot = torch.tensor([0.3, 0.0, 0.0], device=cuda_device, requires_grad=True)
    with pytest.raises(GradientUndefinedError):
        drr(rot, torch.zeros(3, device=cuda_device))
    with torch.no_grad():  # the forward path alone does not reject it
        drr(rot, torch.zeros(3, device=cuda_device))


def test_c1_config(golden, cuda_device):
    """SURVEY 8(d) C1 (128^3 sphere, 100^2): image bit-identical, used-step
    count equal, gradient of neg-ZNCC within tolerance."""
    from paper_2208_12737_b200 import DRR, count_steps, synthetic, pose_frames
    from paper_2208_12737_b200.metrics import neg_zncc
    vol = synthetic.make_phantom("sphere", 128, 1.0)
    import hashlib
    assert hashlib.sha256(vol.ravel(order="F").tobytes()).hexdigest() == str(golden["c1_sha"])
    drr = DRR(vol, 1.0, sdr=300.0, height=100, delx=2.56, device=cuda_device, ray_split=1)
    eta = golden["c1_pose"]
    frame = torch.tensor(O.pose_frame(eta, drr.isocenter), device=cuda_device)[None]
    from paper_2208_12737_b200 import render_frames
    img = render_frames(drr.volume, drr.detector, frame, out_dtype=torch.float64)
    np.testing.assert_array_equal(img[0].cpu().numpy(), golden["c1_image"])
    steps = count_steps(drr.volume, drr.detector, frame, full=True)
    assert int(steps.sum()) == int(golden["c1_steps"])
    rot = torch.tensor(eta[1:4], device=cuda_device, requires_grad=True)
    tra = torch.tensor(eta[4:7], device=cuda_device, requires_grad=True)
    loss = neg_zncc(drr(rot, tra), torch.tensor(golden["c1_fixed"], device=cuda_device))
    loss.backward()
    g = np.concatenate([rot.grad.cpu().numpy(), tra.grad.cpu().numpy()])
    ok, err = grad_close(g, golden["c1_grad"][1:])
    assert ok, (err, g, golden["c1_grad"][1:])


def test_blob_and_corner_diagonal(golden, cuda_device):
    """Acceptance phantoms: shifted oblique pose and the odd-grid corner-to-
    corner diagonal (every crossing tied three ways), bit-identical."""
    from paper_2208_12737_b200 import DeviceVolume, Detector, render_frames, synthetic
    blob = synthetic.blob_phantom(64, 4.0)
    import hashlib
    assert hashlib.sha256(blob.ravel(order="F").tobytes()).hexdigest() == str(golden["blob_sha"])
    vol = DeviceVolume(blob, 4.0, dtype=torch.float64)
    det = Detector(100, 100, 4.0, ray_split=1)
    for key in ("shifted", "truth"):
        f = torch.tensor(O.pose_frame(golden[f"blob_{key}_pose"], vol.center), device=cuda_device)[None]
        img = render_frames(vol, det, f, out_dtype=torch.float64)[0].cpu().numpy()
        np.testing.assert_array_equal(img, golden[f"blob_{key}"])
    uni = DeviceVolume(synthetic.make_phantom("uniform", 64, 4.0), 4.0, dtype=torch.float64)
    f = torch.tensor(O.pose_frame(golden["uni_diag_pose"], uni.center), device=cuda_device)[None]
    img = render_frames(uni, Detector(101, 101, 4.0, ray_split=1), f, out_dtype=torch.float64)[0].cpu().numpy()
    np.testing.assert_array_equal(img, golden["uni_diag101"])


def test_backward_vs_oracle_and_determinism(golden, cuda_device):
    """drr_backward's 12 frame gradients vs the oracle's reverse-mode render
    backward; two runs are bit-identical (fixed-order reduction, no atomics)."""
    from paper_2208_12737_b200 import Detector, backward_frames
    vol = _vol_from_golden(golden, "ps_")
    det = Detector(21, 21, 4.0, ray_split=1)
    rng = np.random.default_rng(3)
    for eta in golden["ps_poses"]:
        frame = O.pose_frame(eta, golden["ps_center"])
        g_img = rng.normal(size=(21, 21))
        _, ref = O.render_backward(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                                   golden["ps_origin"], frame, 21, 21, 4.0, 4.0, g_img)
        ft = torch.tensor(frame, device=cuda_device)[None]
        gt = torch.tensor(g_img, device=cuda_device)[None]
        got = backward_frames(vol, det, ft, gt).cpu().numpy()[0]
        again = backward_frames(vol, det, ft, gt).cpu().numpy()[0]
        np.testing.assert_array_equal(got, again)
        sc = np.abs(ref).max()
        np.testing.assert_allclose(got, ref, atol=1e-10 * sc, rtol=0)


def test_batched_equals_single(golden, cuda_device):
    from paper_2208_12737_b200 import Detector, render_frames
    vol = _vol_from_golden(golden, "ps_")
    det = Detector(21, 17, 4.0, 3.0, ray_split=1)
    frames = torch.tensor(np.stack([O.pose_frame(e, golden["ps_center"]) for e in golden["ps_poses"]]),
                          device=cuda_device)
    batch = render_frames(vol, det, frames, out_dtype=torch.float64)
    for b in range(frames.shape[0]):
        one = render_frames(vol, det, frames[b:b + 1], out_dtype=torch.float64)
        assert torch.equal(one[0], batch[b])
        ref = O.render(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                       golden["ps_origin"], frames[b].cpu().numpy(), 21, 17, 4.0, 3.0)
        np.testing.assert_array_equal(one[0].cpu().numpy(), ref)


def test_chest_c2_vs_oracle(cuda_device):
    """C2 (512 x 512 x 133 chest @ 0.703/2.5 mm, 200^2 @ 3.6 mm, oblique pose):
    the fp32 product path against the oracle fed the same fp32 densities."""
    from paper_2208_12737_b200 import DRR, backward_frames, render_frames, synthetic
    vol = synthetic.chest_phantom()
    spacing = (0.703125, 0.703125, 2.5)
    drr = DRR(vol, spacing, sdr=300.0, height=200, delx=3.6, device=cuda_device, ray_split=1)
    eta = np.array([300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0])
    frame = O.pose_frame(eta, drr.isocenter)
    ft = torch.tensor(frame, device=cuda_device)[None]
    img = render_frames(drr.volume, drr.detector, ft, out_dtype=torch.float64)[0].cpu().numpy()
    flat = vol.astype(np.float64).ravel(order="F")
    ref = O.render(flat, vol.shape, spacing, (0, 0, 0), frame, 200, 200, 3.6, 3.6)
    np.testing.assert_array_equal(img, ref)
    g_img = np.random.default_rng(0).normal(size=(200, 200))
    got = backward_frames(drr.volume, drr.detector, ft,
                          torch.tensor(g_img, device=cuda_device)[None]).cpu().numpy()[0]
    _, refg = O.render_backward(flat, vol.shape, spacing, (0, 0, 0), frame, 200, 200, 3.6, 3.6, g_img)
    np.testing.assert_allclose(got, refg, atol=1e-9 * np.abs(refg).max(), rtol=0)


def test_fd_gradient_check(cuda_device):
    """Central finite differences (gradients.py:72-120 steps) of the GPU loss
    agree with the GPU gradient on a smooth pose."""
    from paper_2208_12737_b200 import DRR, synthetic
    from paper_2208_12737_b200.metrics import neg_zncc
    vol = synthetic.make_phantom("sphere", 32, 2.0) + 0.2 * np.random.default_rng(3).random((32,) * 3)
    drr = DRR(vol.astype(np.float32), 2.0, sdr=150.0, height=48, delx=2.0, device=cuda_device)
    fixed = drr(torch.tensor([0.45, 1.25, 0.12], device=cuda_device),
                torch.tensor([2.0, -1.0, 0.5], device=cuda_device)).detach()
    x0 = np.array([0.4, 1.3, 0.1, 0.0, 0.0, 0.0])
    x = torch.tensor(x0, device=cuda_device, requires_grad=True)
    loss = neg_zncc(drr(x[:3], x[3:]), fixed)
    loss.backward()
    g = x.grad.cpu().numpy()
    steps = np.array([1e-5, 1e-5, 1e-5, 1e-3, 1e-3, 1e-3])
    fd = np.zeros(6)
    with torch.no_grad():
        for i in range(6):
            xp, xm = x0.copy(), x0.copy()
            xp[i] += steps[i]
            xm[i] -= steps[i]
            lp = float(neg_zncc(drr(torch.tensor(xp[:3], device=cuda_device), torch.tensor(xp[3:], device=cuda_device)), fixed))
            lm = float(neg_zncc(drr(torch.tensor(xm[:3], device=cuda_device), torch.tensor(xm[3:], device=cuda_device)), fixed))
            fd[i] = (lp - lm) / (2 * steps[i])
    # fp32 images limit FD resolution; FD is reported, the bar is loose
    np.testing.assert_allclose(g, fd, rtol=2e-2, atol=2e-3 * np.abs(g).max())


@pytest.mark.parametrize("split", [2, 4, 8])
def test_ray_split_matches_single_thread(split, cuda_device):
    """Rays cut across K threads at dominant-axis crossings:
    same used-step counts exactly, images within 1e-13 relative (summation
    order only), frame gradients within 1e-11 -- on the C2 chest at an
    oblique pose and at AP (ties between x/y crossings), and on the
    corner-diagonal uniform phantom where every crossing ties three ways."""
    from paper_2208_12737_b200 import (DeviceVolume, Detector, backward_frames, count_steps,
                                       render_frames, synthetic)
    cases = []
    chest = DeviceVolume(synthetic.chest_phantom(), (0.703125, 0.703125, 2.5))
    cases.append((chest, 200, 3.6, [300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0]))
    cases.append((chest, 200, 3.6, [300.0, np.pi / 2, np.pi / 2, 0.0, 0.0, 0.0, 0.0]))
    uni = DeviceVolume(synthetic.make_phantom("uniform", 64, 4.0), 4.0)
    cases.append((uni, 101, 4.0, [400.0, np.pi / 4, np.arccos(1 / np.sqrt(3)), 0, 0, 0, 0]))
    rng = np.random.default_rng(1)
    for vol, n, pitch, eta in cases:
        f = torch.tensor(O.pose_frame(np.array(eta), vol.center), device=cuda_device)[None]
        d1, dk = Detector(n, n, pitch, ray_split=1), Detector(n, n, pitch, ray_split=split)
        assert torch.equal(count_steps(vol, d1, f), count_steps(vol, dk, f))
        a = render_frames(vol, d1, f, out_dtype=torch.float64)
        b = render_frames(vol, dk, f, out_dtype=torch.float64)
        np.testing.assert_allclose(b.cpu().numpy(), a.cpu().numpy(), rtol=1e-13, atol=1e-12)
        g = torch.tensor(rng.normal(size=(1, n, n)), device=cuda_device)
        ga = backward_frames(vol, d1, f, g).cpu().numpy()
        gb = backward_frames(vol, dk, f, g).cpu().numpy()
        np.testing.assert_allclose(gb, ga, rtol=0, atol=1e-11 * np.abs(ga).max())


@pytest.mark.parametrize("split", [1, 2, 8])
def test_forward_jac_matches_forward_and_rewalk(split, golden, cuda_device):
    """drr_forward_jac + drr_backward_jac (one CT walk per ray, gradient by
    contracting the stored ray Jacobians) against drr_forward (image: bitwise)
    and the fused re-walk drr_backward (frame gradients: bitwise at K = 1, the
    same fixed reduction order), and against the oracle's reverse-mode render
    backward on the C2 chest and the golden sphere poses."""
    from paper_2208_12737_b200 import (DeviceVolume, Detector, backward_frames,
                                       backward_from_jac, render_frames, render_frames_jac,
                                       synthetic)
    rng = np.random.default_rng(7)
    vol = _vol_from_golden(golden, "ps_")
    det = Detector(21, 21, 4.0, ray_split=split)
    frames = torch.tensor(np.stack([O.pose_frame(e, golden["ps_center"]) for e in golden["ps_poses"]]),
                          device=cuda_device)
    g_img = rng.normal(size=(frames.shape[0], 21, 21))
    img, jac = render_frames_jac(vol, det, frames, out_dtype=torch.float64)
    assert torch.equal(img, render_frames(vol, det, frames, out_dtype=torch.float64))
    gt = torch.tensor(g_img, device=cuda_device)
    got = backward_from_jac(det, jac, gt).cpu().numpy()
    again = backward_from_jac(det, jac, gt).cpu().numpy()
    np.testing.assert_array_equal(got, again)
    rewalk = backward_frames(vol, det, frames, gt).cpu().numpy()
    if split == 1:
        np.testing.assert_array_equal(got, rewalk)
    for b, eta in enumerate(golden["ps_poses"]):
        frame = O.pose_frame(eta, golden["ps_center"])
        _, ref = O.render_backward(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                                   golden["ps_origin"], frame, 21, 21, 4.0, 4.0, g_img[b])
        np.testing.assert_allclose(got[b], ref, atol=1e-10 * np.abs(ref).max(), rtol=0)
    # C2 chest, fp32 product layout, oblique pose
    chest = synthetic.chest_phantom()
    spacing = (0.703125, 0.703125, 2.5)
    cv = DeviceVolume(chest, spacing)
    cdet = Detector(200, 200, 3.6, ray_split=split)
    eta = np.array([300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0])
    frame = O.pose_frame(eta, cv.center)
    ft = torch.tensor(frame, device=cuda_device)[None]
    img, jac = render_frames_jac(cv, cdet, ft, out_dtype=torch.float64)
    flat = chest.astype(np.float64).ravel(order="F")
    ref_img = O.render(flat, chest.shape, spacing, (0, 0, 0), frame, 200, 200, 3.6, 3.6)
    if split == 1:
        np.testing.assert_array_equal(img[0].cpu().numpy(), ref_img)
    else:
        np.testing.assert_allclose(img[0].cpu().numpy(), ref_img, rtol=1e-13, atol=1e-12)
    g2 = rng.normal(size=(200, 200))
    got = backward_from_jac(cdet, jac, torch.tensor(g2, device=cuda_device)[None]).cpu().numpy()[0]
    _, refg = O.render_backward(flat, chest.shape, spacing, (0, 0, 0), frame, 200, 200, 3.6, 3.6, g2)
    np.testing.assert_allclose(got, refg, atol=1e-9 * np.abs(refg).max(), rtol=0)


def test_module_uses_one_walk_and_rewalk_fallback(golden, cuda_device, monkeypatch):
    """The nn.Module's autograd path: with a gradient requested it runs the
    one-walk forward + Jacobian contraction; above the Jacobian memory budget
    it re-walks in backward.  Both give the same pose gradient."""
    from paper_2208_12737_b200 import DRR, renderer
    from paper_2208_12737_b200.metrics import neg_zncc
    dims = tuple(int(n) for n in golden["ps_dims"])
    data = golden["ps_flat"].reshape(dims[::-1]).transpose(2, 1, 0)
    fixed = torch.tensor(golden["ps_fixed"], device=cuda_device)
    eta = golden["ps_poses"][1]
    drr = DRR(data, 2.0, sdr=float(eta[0]), height=21, delx=4.0, device=cuda_device)

    def grad():
        rot = torch.tensor(eta[1:4], device=cuda_device, requires_grad=True)
        tra = torch.tensor(eta[4:7], device=cuda_device, requires_grad=True)
        neg_zncc(drr(rot, tra), fixed).backward()
        return torch.cat([rot.grad, tra.grad]).cpu().numpy()

    one_walk = grad()
    monkeypatch.setattr(renderer, "JAC_BUDGET_BYTES", 0)
    rewalk = grad()
    np.testing.assert_allclose(one_walk, rewalk, rtol=1e-12, atol=1e-15)


def test_pose_batches_beyond_one_launch(golden, cuda_device, monkeypatch):
    """Batches larger than one launch's pose limit are split into launches;
    rays are independent, so images, step counts and gradients are unchanged."""
    from paper_2208_12737_b200 import (Detector, backward_frames, count_steps, render_frames,
                                       renderer)
    vol = _vol_from_golden(golden, "ps_")
    det = Detector(21, 21, 4.0, ray_split=1)
    frames = torch.tensor(np.stack([O.pose_frame(e, golden["ps_center"]) for e in golden["ps_poses"]]),
                          device=cuda_device)
    g = torch.randn((frames.shape[0], 21, 21), device=cuda_device, dtype=torch.float64)
    whole = (render_frames(vol, det, frames), count_steps(vol, det, frames),
             backward_frames(vol, det, frames, g))
    from paper_2208_12737_b200.registration import loss_and_gradient
    eta = torch.tensor(golden["ps_poses"], device=cuda_device)
    fixed = torch.rand((eta.shape[0], 21, 21), device=cuda_device)
    whole_lg = loss_and_gradient(vol, det, eta, fixed)
    monkeypatch.setattr(renderer, "MAX_POSES_PER_LAUNCH", 2)
    split = (render_frames(vol, det, frames), count_steps(vol, det, frames),
             backward_frames(vol, det, frames, g))
    for a, b in zip(whole, split):
        assert torch.equal(a, b)
    for a, b in zip(whole_lg, loss_and_gradient(vol, det, eta, fixed)):
        assert torch.equal(a, b)


def test_clip_entry_and_exit_gradients(cuda_device):
    """Rays that start inside the volume (clip entry: the 3-axis gradient
    walk) and rays that end inside it (clip exit: the derived-axis walk with
    its clip terms), energies bitwise and endpoint gradients to 1e-10 against
    the C oracle."""
    be = _backend()
    rng = np.random.default_rng(23)
    for trial in range(24):
        dims = tuple(int(x) for x in rng.integers(2, 20, 3))
        spacing = rng.uniform(0.5, 2.5, 3)
        origin = rng.uniform(-3, 3, 3)
        flat = rng.uniform(0, 4, int(np.prod(dims)))
        lo = origin
        hi = origin + np.asarray(dims) * spacing
        span = float(max(hi - lo))
        if trial % 2:
            src = rng.uniform(lo, hi)                       # source inside
            pix = rng.uniform(lo - span, hi + span, size=(128, 3))
        else:
            src = rng.uniform(lo - 3 * span, hi + 3 * span)  # pixel inside
            pix = rng.uniform(lo, hi, size=(128, 3))
        e = be.siddon_raysum(flat, dims, spacing, origin, src, pix)
        np.testing.assert_array_equal(e, O.raysum(flat, dims, spacing, origin, src, pix))
        _, gs, gp = be.ray_endpoint_grad(flat, dims, spacing, origin, src, pix)
        _, rs, rp = O.raysum_endpoint_grad(flat, dims, spacing, origin, src, pix)
        sc = max(1.0, np.abs(rs).max(), np.abs(rp).max())
        np.testing.assert_allclose(gs, rs, atol=1e-10 * sc, rtol=0, err_msg=f"trial {trial}")
        np.testing.assert_allclose(gp, rp, atol=1e-10 * sc, rtol=0, err_msg=f"trial {trial}")


def test_subnormal_direction_rays(cuda_device):
    """Rays with a direction component of |d| <= 1e-20 (Ray::safe: IEEE
    division for their crossing parameters, the v4 walk) against the oracle,
    energies bitwise and endpoint gradients to 1e-10."""
    be = _backend()
    rng = np.random.default_rng(29)
    dims = (9, 7, 5)
    spacing = np.array([1.5, 1.0, 2.0])
    origin = np.array([-3.0, 1.0, 0.5])
    flat = rng.uniform(0, 4, int(np.prod(dims)))
    hi = origin + np.asarray(dims) * spacing
    src = np.array([origin[0] + 4.1, origin[1] - 20.0, origin[2] + 3.3])
    pix = []
    for tiny in (1e-21, -3e-22, 5e-300, 1e-30):
        for ax in (0, 2):
            p = np.array([src[0], hi[1] + 20.0, src[2]])
            p[ax] += tiny
            pix.append(p)
    pix = np.array(pix)
    e = be.siddon_raysum(flat, dims, spacing, origin, src, pix)
    np.testing.assert_array_equal(e, O.raysum(flat, dims, spacing, origin, src, pix))
    assert np.all(e > 0)
    _, gs, gp = be.ray_endpoint_grad(flat, dims, spacing, origin, src, pix)
    _, rs, rp = O.raysum_endpoint_grad(flat, dims, spacing, origin, src, pix)
    sc = max(1.0, np.abs(rs).max(), np.abs(rp).max())
    np.testing.assert_allclose(gs, rs, atol=1e-10 * sc, rtol=0)
    np.testing.assert_allclose(gp, rp, atol=1e-10 * sc, rtol=0)


def test_pose_group_order_is_invisible(cuda_device):
    """The CTA order interleaves poses in groups of ~16K CTAs (drr_kernels.cu
    pose_group): 40 poses on a 320x200 detector (550 tiles per pose) run as
    groups of 29 + 11.  Images, ray Jacobians and frame gradients equal those
    of one-pose launches bitwise; the forward-only kernel agrees too."""
    from paper_2208_12737_b200 import (DeviceVolume, Detector, backward_from_jac, pose_frames,
                                       render_frames, render_frames_jac, synthetic)
    rng = np.random.default_rng(3)
    vol = DeviceVolume(rng.uniform(0, 2, (40, 36, 30)).astype(np.float32), (1.5, 1.7, 2.0),
                       device=cuda_device)
    B, H, W = 40, 200, 320
    det = Detector(H, W, 0.6, ray_split=1)
    poses = synthetic.sample_poses((300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0),
                                   synthetic.NARROW_HALF_WIDTHS, B, seed=1)
    frames = pose_frames(torch.tensor(poses, device=cuda_device), vol.center).detach()
    g = torch.randn((B, H, W), device=cuda_device)
    img, jac = render_frames_jac(vol, det, frames)
    gf = backward_from_jac(det, jac, g)
    assert torch.equal(render_frames(vol, det, frames), img)
    assert float((img > 0).float().mean()) > 0.2  # the rays do cross the volume
    jac = jac.view(6, B, H * W)
    for b in range(B):
        i1, j1 = render_frames_jac(vol, det, frames[b:b + 1].contiguous())
        assert torch.equal(i1[0], img[b])
        assert torch.equal(j1.view(6, H * W), jac[:, b])
        assert torch.equal(backward_from_jac(det, j1, g[b:b + 1].contiguous())[0], gf[b])


def test_raysum_tangents_epilogue_matches_endpoint_contraction(golden, cuda_device):
    """drr_raysum_tangents (the contraction in the walk's epilogue) equals the
    reverse-mode endpoint derivatives contracted on the host, for the golden
    kernel cases; empty ray bundles return empty arrays."""
    be = _backend()
    for c in range(0, int(golden["k_count"]), 7):
        k = kernel_case(golden, c)
        e, de = be.siddon_raysum_grad(k["flat"], k["dims"], k["spacing"], k["origin"],
                                      k["source"], k["d_source"], k["pixels"], k["d_pixels"])
        e2, gs, gp = be.ray_endpoint_grad(k["flat"], k["dims"], k["spacing"], k["origin"],
                                          k["source"], k["pixels"])
        np.testing.assert_array_equal(e, e2)
        dpix = np.asarray(k["d_pixels"]).reshape(len(e), 3, -1)
        ref = gs @ np.asarray(k["d_source"]) + np.einsum("na,nat->nt", gp, dpix)
        scale = max(1.0, float(np.abs(ref).max()))
        np.testing.assert_allclose(de, ref, rtol=0, atol=1e-13 * scale)
    e, de = be.siddon_raysum_grad(k["flat"], k["dims"], k["spacing"], k["origin"], k["source"],
                                  k["d_source"], np.zeros((0, 3)), np.zeros((0, 3, 7)))
    assert e.shape == (0,) and de.shape == (0, 7)
