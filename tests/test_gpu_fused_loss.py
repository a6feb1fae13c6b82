"""The fused loss-gradient walk (drr_forward_loss_grad) and the two-pass loss.

* float64 volume and images against the C oracle (the reference's arithmetic:
  render, loss_value_and_pixel_grad, render_backward, the frame Jacobian):
  values to 1e-12, gradients to 1e-9 relative -- neg-ZNCC and L2, one shared
  fixed image and one per pose;
* against the stored-Jacobian path (drr_forward_jac + drr_backward_jac) fed
  the same float64 pixel gradient: dL/dframe to 1e-10 relative (the affine
  split c0 sum J + c1 sum aJ + c2 sum bJ may cancel; this bounds it);
* batch invariance: a pose's result does not depend on the batch around it;
* the loss edge cases of metrics.py:26-31: bright images with little
  structure (the two-pass moments keep their digits), exact and inexact
  constants (sigma == 0 -> status 1, NaN), L2 of identical images (0, zero
  gradient).
"""

import math

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DIMS = (26, 22, 18)
SP = (1.5, 1.75, 2.0)
H, W = 23, 19


def _volume():
    rng = np.random.default_rng(11)
    from paper_2208_12737_b200 import synthetic
    v = synthetic.blob_phantom(26, 1.0)[:, :22, :18] + 0.1 * rng.random(DIMS)
    return v


def _poses(n, seed=2):
    rng = np.random.default_rng(seed)
    return np.column_stack([np.full(n, 80.0), rng.uniform(0.3, 2.8, n), rng.uniform(0.5, 2.6, n),
                            rng.uniform(-0.5, 0.5, n), rng.uniform(-3, 3, (n, 3))])


def _run(vol, det, eta, fixed, kind, img_dtype, stride):
    from paper_2208_12737_b200 import _lib, pose_frames
    lib = _lib.load()
    dev = vol.device
    B = eta.shape[0]
    et = torch.tensor(eta, device=dev)
    fr = pose_frames(et, vol.center).detach()
    img = torch.empty((B, det.height, det.width), dtype=img_dtype, device=dev)
    val = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.zeros(B, dtype=torch.int32, device=dev)
    gf = torch.empty((B, 12), dtype=torch.float64, device=dev)
    ge = torch.empty((B, 7), dtype=torch.float64, device=dev)
    ws_bytes = lib.drr_loss_grad_workspace_size(B, det.c)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    fx = torch.as_tensor(fixed, device=dev, dtype=img_dtype).contiguous()
    _lib.check(lib.drr_forward_loss_grad(
        vol.flat.data_ptr(), vol.vol_dtype, vol.grid, fr.data_ptr(), et.data_ptr(), B, det.c,
        fx.data_ptr(), stride, kind, img.data_ptr(), 1 if img_dtype == torch.float64 else 0,
        val.data_ptr(), st.data_ptr(), gf.data_ptr(), ge.data_ptr(), ws.data_ptr(), ws_bytes,
        torch.cuda.current_stream(dev).cuda_stream))
    return fr, img, val, st, gf, ge


def _l2_value_and_grad(a, b):
    d = a - b
    v = float(np.linalg.norm(d.ravel()))
    return v, (np.zeros_like(d) if v == 0.0 else d / v)


@pytest.mark.parametrize("kind", ["neg_zncc", "l2"])
@pytest.mark.parametrize("shared", [True, False])
def test_fused_f64_vs_oracle(cuda_device, kind, shared):
    from paper_2208_12737_b200 import Detector, DeviceVolume, _lib
    v = _volume()
    vol = DeviceVolume(v, SP, device=cuda_device, dtype=torch.float64)
    det = Detector(H, W, 2.5, 2.25, ray_split=1)  # one thread per ray: the oracle's sum order
    eta = _poses(5)
    flat = v.ravel(order="F")
    center = vol.center
    truth = np.array([80.0, 1.2, 1.4, 0.1, 1.0, -1.0, 0.5])
    fixed_one = O.render(flat, DIMS, SP, (0, 0, 0), O.pose_frame(truth, center), H, W, 2.5, 2.25)
    if shared:
        fixed, stride = fixed_one, 0
    else:
        fixed = np.stack([fixed_one * (1.0 + 0.1 * i) + i for i in range(5)])
        stride = H * W
    code = _lib.DRR_LOSS_NEG_ZNCC if kind == "neg_zncc" else _lib.DRR_LOSS_L2
    fr, img, val, st, gf, ge = _run(vol, det, eta, fixed, code, torch.float64, stride)
    assert int(st.sum()) == 0
    for i in range(5):
        frame = fr[i].cpu().numpy()
        ref_img = O.render(flat, DIMS, SP, (0, 0, 0), frame, H, W, 2.5, 2.25)
        np.testing.assert_array_equal(img[i].cpu().numpy(), ref_img)
        fi = fixed if shared else fixed[i]
        if kind == "neg_zncc":
            rv, pg = O.neg_zncc_value_and_grad(ref_img, fi)
        else:
            rv, pg = _l2_value_and_grad(ref_img, fi)
        assert float(val[i]) == pytest.approx(rv, abs=1e-12, rel=1e-12)
        _, rgf = O.render_backward(flat, DIMS, SP, (0, 0, 0), frame, H, W, 2.5, 2.25, pg)
        scale = np.abs(rgf).max()
        np.testing.assert_allclose(gf[i].cpu().numpy(), rgf, rtol=0, atol=1e-9 * scale)
        rge = rgf @ O.frame_jacobian(eta[i], center)
        np.testing.assert_allclose(ge[i].cpu().numpy(), rge, rtol=0, atol=1e-9 * np.abs(rge).max())


def test_fused_matches_stored_jacobian(cuda_device):
    """Same float64 pixel gradient through the stored-Jacobian contraction."""
    from paper_2208_12737_b200 import (Detector, DeviceVolume, _lib, backward_from_jac,
                                       render_frames_jac)
    v = _volume()
    vol = DeviceVolume(v, SP, device=cuda_device, dtype=torch.float64)
    det = Detector(H, W, 2.5, 2.25, ray_split=1)
    eta = _poses(6, seed=5)
    fixed = np.random.default_rng(3).random((H, W)) * 30.0
    fr, img, val, st, gf, ge = _run(vol, det, eta, fixed, _lib.DRR_LOSS_NEG_ZNCC,
                                    torch.float64, 0)
    img2, jac = render_frames_jac(vol, det, fr, out_dtype=torch.float64)
    torch.testing.assert_close(img2, img, rtol=0, atol=0)
    pg = np.stack([O.neg_zncc_value_and_grad(img[i].cpu().numpy(), fixed)[1] for i in range(6)])
    gf2 = backward_from_jac(det, jac, torch.tensor(pg, device=cuda_device)).cpu().numpy()
    scale = np.abs(gf2).max(axis=1, keepdims=True)
    assert np.all(np.abs(gf.cpu().numpy() - gf2) <= 1e-10 * scale)


def test_fused_batch_invariance(cuda_device):
    """A pose's image, value and gradient do not depend on the batch around it
    (one thread per ray; the CTA partials are per pose)."""
    from paper_2208_12737_b200 import Detector, DeviceVolume, _lib
    v = _volume()
    vol = DeviceVolume(v, SP, device=cuda_device)
    det = Detector(H, W, 2.5, 2.25, ray_split=1)
    eta = _poses(7, seed=8)
    fixed = np.random.default_rng(4).random((H, W)).astype(np.float32) * 20.0
    full = _run(vol, det, eta, fixed, _lib.DRR_LOSS_NEG_ZNCC, torch.float32, 0)
    for i in (0, 3, 6):
        one = _run(vol, det, eta[i:i + 1], fixed, _lib.DRR_LOSS_NEG_ZNCC, torch.float32, 0)
        for a, b in zip(full[1:], one[1:]):
            np.testing.assert_array_equal(a[i].cpu().numpy(), b[0].cpu().numpy())


def _loss(img, fixed, kind, dtype, dev):
    from paper_2208_12737_b200 import _lib
    lib = _lib.load()
    a = torch.tensor(img, dtype=dtype, device=dev)[None]
    b = torch.tensor(fixed, dtype=dtype, device=dev)
    val = torch.empty(1, dtype=torch.float64, device=dev)
    g = torch.empty(a.shape, dtype=torch.float32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.drr_image_loss(a.data_ptr(), b.data_ptr(), 1 if dtype == torch.float64 else 0,
                                  0, 1, a.numel(), kind, val.data_ptr(), g.data_ptr(),
                                  st.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    return float(val[0]), g[0].cpu().numpy(), int(st[0])


def test_loss_two_pass_bright_low_variance(cuda_device):
    """mean 1e4, sigma 1e-3: the one-pass E[x^2] - mu^2 would lose ~8 digits;
    the two-pass moments match the reference's centred arithmetic."""
    from paper_2208_12737_b200 import _lib
    rng = np.random.default_rng(21)
    a = 1.0e4 + 1e-3 * rng.standard_normal((200, 200))
    b = 3.0e3 + 1e-3 * (0.6 * (a - 1.0e4) / 1e-3 + 0.8 * rng.standard_normal((200, 200)))
    v, g, st = _loss(a, b, _lib.DRR_LOSS_NEG_ZNCC, torch.float64, cuda_device)
    rv, rg = O.neg_zncc_value_and_grad(a, b)
    assert st == 0
    assert v == pytest.approx(rv, abs=1e-9)
    np.testing.assert_allclose(g, rg, rtol=1e-5, atol=1e-6 * np.abs(rg).max())


@pytest.mark.parametrize("c", [1.0, 0.1, 1.0 / 3.0, 1234.5678])
def test_loss_constant_images_are_undefined(cuda_device, c):
    """metrics.py:29-30: a constant image has sigma 0 -> MetricUndefinedError
    (status 1, NaN value and gradient); for an inexact constant whose mean
    rounds, the reference's sigma can come out as rounding noise instead --
    the kernel decides from the pixels (all equal), the defined answer."""
    from paper_2208_12737_b200 import _lib
    rng = np.random.default_rng(1)
    fixed = rng.random((50, 40))
    for dtype in (torch.float32, torch.float64):
        v, g, st = _loss(np.full((50, 40), c), fixed, _lib.DRR_LOSS_NEG_ZNCC, dtype, cuda_device)
        assert st == 1 and math.isnan(v) and np.isnan(g).all()
        v, g, st = _loss(fixed, np.full((50, 40), c), _lib.DRR_LOSS_NEG_ZNCC, dtype, cuda_device)
        assert st == 1 and math.isnan(v)


def test_loss_l2_identical_images(cuda_device):
    from paper_2208_12737_b200 import _lib
    a = np.random.default_rng(2).random((30, 30))
    v, g, st = _loss(a, a, _lib.DRR_LOSS_L2, torch.float64, cuda_device)
    assert v == 0.0 and st == 0 and not g.any()


def test_api_loss_and_gradient_fused_f64(golden, cuda_device):
    """api.loss_and_gradient (one drr_forward_loss_grad call, float64) against
    the reference's golden loss_and_gradient records: values to 1e-12."""
    from paper_2208_12737_b200 import api
    vol = api.Volume(tuple(golden["ps_dims"]), tuple(golden["ps_spacing"]),
                     tuple(golden["ps_origin"]),
                     np.asarray(golden["ps_flat"]).reshape(tuple(golden["ps_dims"]), order="F"))
    spec = api.DetectorSpec.for_volume(vol, 21, 21, (4.0, 4.0))
    for i, eta in enumerate(golden["ps_poses"]):
        if not np.isfinite(golden["ps_values"][i]):
            continue
        rec = api.loss_and_gradient(vol, api.PoseParameters.from_vector(eta), spec,
                                    golden["ps_fixed"])
        assert rec.value == pytest.approx(golden["ps_values"][i], abs=1e-12)
        ref = golden["ps_grads"][i]
        np.testing.assert_allclose(rec.grad, ref, rtol=0, atol=1e-9 * np.abs(ref).max())


def test_loss_and_gradient_chains_agree(cuda_device):
    """registration.loss_and_gradient's two chains (stored Jacobian vs fused
    walk) on float32 images: identical images and values, gradients within
    the float32 rounding of the stored chain's pixel gradient."""
    from paper_2208_12737_b200 import Detector, DeviceVolume
    from paper_2208_12737_b200.registration import _Buffers, loss_and_gradient
    v = _volume()
    vol = DeviceVolume(v, SP, device=cuda_device)
    det = Detector(H, W, 2.5, 2.25)
    eta = torch.tensor(_poses(6, seed=13), device=cuda_device)
    fixed = np.random.default_rng(6).random((H, W)).astype(np.float32) * 20.0
    bj = _Buffers(vol, det, 6, mode="jac")
    bf = _Buffers(vol, det, 6, mode="fused")
    assert _Buffers(vol, det, 6).mode == "jac"
    assert _Buffers(vol, det, 6, image_dtype=torch.float64).mode == "fused"
    vj, gj = loss_and_gradient(vol, det, eta, fixed, buffers=bj)
    vf, gf = loss_and_gradient(vol, det, eta, fixed, buffers=bf)
    torch.testing.assert_close(bj.img, bf.img, rtol=0, atol=0)
    torch.testing.assert_close(vj, vf, rtol=0, atol=0)
    scale = gf.abs().max(dim=1, keepdim=True).values
    assert bool(((gj - gf).abs() <= 1e-5 * scale).all()), (gj, gf)


@pytest.mark.parametrize("kind", ["neg_zncc", "l2"])
def test_loss_grad_jac_vs_oracle(cuda_device, kind):
    """drr_loss_grad_jac (loss + float64 pixel gradient + Jacobian contraction
    + pose gradient, one cluster launch per image) after drr_forward_jac:
    values to 1e-12, dL/dframe and dL/deta to 1e-9 of the oracle, per-pose
    fixed images and a shared one."""
    from paper_2208_12737_b200 import Detector, DeviceVolume, _lib, pose_frames, render_frames_jac
    v = _volume()
    vol = DeviceVolume(v, SP, device=cuda_device, dtype=torch.float64)
    det = Detector(H, W, 2.5, 2.25, ray_split=1)
    eta = _poses(4, seed=17)
    et = torch.tensor(eta, device=cuda_device)
    fr = pose_frames(et, vol.center).detach()
    img, jac = render_frames_jac(vol, det, fr, out_dtype=torch.float64)
    flat = v.ravel(order="F")
    rng = np.random.default_rng(9)
    code = _lib.DRR_LOSS_NEG_ZNCC if kind == "neg_zncc" else _lib.DRR_LOSS_L2
    for fixed, stride in ((rng.random((H, W)) * 30.0, 0), (rng.random((4, H, W)) * 30.0, H * W)):
        fx = torch.tensor(fixed, device=cuda_device)
        val = torch.empty(4, dtype=torch.float64, device=cuda_device)
        gf = torch.empty((4, 12), dtype=torch.float64, device=cuda_device)
        ge = torch.empty((4, 7), dtype=torch.float64, device=cuda_device)
        st = torch.zeros(4, dtype=torch.int32, device=cuda_device)
        _lib.check(_lib.load().drr_loss_grad_jac(
            jac.data_ptr(), img.data_ptr(), fx.data_ptr(), 1, stride, 4, det.c, code,
            val.data_ptr(), st.data_ptr(), gf.data_ptr(), et.data_ptr(), ge.data_ptr(),
            torch.cuda.current_stream().cuda_stream))
        for i in range(4):
            fi = fixed if stride == 0 else fixed[i]
            ref_img = O.render(flat, DIMS, SP, (0, 0, 0), fr[i].cpu().numpy(), H, W, 2.5, 2.25)
            rv, pg = (O.neg_zncc_value_and_grad(ref_img, fi) if kind == "neg_zncc"
                      else _l2_value_and_grad(ref_img, fi))
            assert float(val[i]) == pytest.approx(rv, abs=1e-12, rel=1e-12)
            _, rgf = O.render_backward(flat, DIMS, SP, (0, 0, 0), fr[i].cpu().numpy(), H, W, 2.5,
                                       2.25, pg)
            np.testing.assert_allclose(gf[i].cpu().numpy(), rgf, rtol=0,
                                       atol=1e-9 * np.abs(rgf).max())
            rge = rgf @ O.frame_jacobian(eta[i], vol.center)
            np.testing.assert_allclose(ge[i].cpu().numpy(), rge, rtol=0,
                                       atol=1e-9 * np.abs(rge).max())


@pytest.mark.parametrize("img_f64", [False, True])
@pytest.mark.parametrize("hw", [(37, 29), (90, 90)])
def test_loss_grad_jac_tma_path_matches_register_path(cuda_device, img_f64, hw):
    """A batch large enough for drr_loss_grad_jac's TMA-staged contraction
    (the Jacobian streamed through shared memory by bulk copies) gives the
    bits of one-image calls, which take the register-staged path.  37 x 29
    (an odd batch of odd images): every tile falls back to direct loads;
    90 x 90: 1013 pixels per CTA, so even ranks stream three full tiles by
    TMA and load the odd last one directly, odd ranks start unaligned."""
    from paper_2208_12737_b200 import Detector, DeviceVolume, _lib, pose_frames, render_frames_jac
    vol = DeviceVolume(_volume(), SP, device=cuda_device)
    Hh, Ww = hw
    det = Detector(Hh, Ww, 3.0 * 29 / Ww, 2.5 * 37 / Hh, ray_split=1)  # the same field
    B = 2 * torch.cuda.get_device_properties(cuda_device).multi_processor_count + 3
    et = torch.tensor(_poses(B, seed=21), device=cuda_device)
    fr = pose_frames(et, vol.center).detach()
    dt = torch.float64 if img_f64 else torch.float32
    img, jac = render_frames_jac(vol, det, fr, out_dtype=dt)
    fixed = torch.rand((B, Hh, Ww), device=cuda_device, dtype=dt)
    npix = Hh * Ww
    lib = _lib.load()

    def run(j, im, fx, n):
        val = torch.empty(n, dtype=torch.float64, device=cuda_device)
        gf = torch.empty((n, 12), dtype=torch.float64, device=cuda_device)
        _lib.check(lib.drr_loss_grad_jac(j.data_ptr(), im.data_ptr(), fx.data_ptr(), int(img_f64),
                                         npix, n, det.c, _lib.DRR_LOSS_NEG_ZNCC, val.data_ptr(),
                                         None, gf.data_ptr(), None, None,
                                         torch.cuda.current_stream().cuda_stream))
        return val, gf
    val, gf = run(jac, img, fixed, B)
    for p in range(0, B, 7):
        v1, g1 = run(jac[:, p * npix:(p + 1) * npix].contiguous(), img[p:p + 1].contiguous(),
                     fixed[p:p + 1].contiguous(), 1)
        assert torch.equal(v1[0], val[p]) and torch.equal(g1[0], gf[p]), p
