"""BASELINE.json configs C4 and C5 as parity cases.

* C4: the C2 chest volume, 1024 narrow poses (seed 0), 256^2 detector at
  2.8125 mm, forward only.  The batch is the multi-GPU unit of work: its pose
  blocks render bit-identically alone or inside the full batch (the pose-shard
  partition has no exchange step), poses match the C oracle bit for bit, and
  the used voxel-steps per DRR match SURVEY 8(d)'s measured 35.7-38.9 M.
* C5: a 512^3 volume at 0.703125 mm (sphere + 3x off-centre cube + noise),
  1024^2 detector at 0.703125 mm, forward + backward: sampled rays against the
  oracle, the one-walk gradient against the re-walk, and the module path above
  the Jacobian memory budget (64 poses at 1024^2 would hold 3.2 GB).
"""

import math

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

C2_SPACING = (0.703125, 0.703125, 2.5)
TRUTH = (300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)


def test_c4_batched_generation(cuda_device):
    from paper_2208_12737_b200 import (DeviceVolume, Detector, count_steps, pose_frames,
                                       render_frames, synthetic)
    chest = synthetic.chest_phantom()
    vol = DeviceVolume(chest, C2_SPACING)
    det = Detector(256, 256, 2.8125)
    poses = synthetic.sample_poses(TRUTH, synthetic.NARROW_HALF_WIDTHS, 1024, seed=0)
    frames = pose_frames(torch.tensor(poses, device=cuda_device), vol.center).detach()
    full = render_frames(vol, det, frames)
    assert full.shape == (1024, 256, 256) and torch.isfinite(full).all()
    # pose shards (two "ranks" and an uneven third) render identically alone
    for lo, hi in ((0, 512), (512, 1024), (100, 357)):
        part = render_frames(vol, det, frames[lo:hi].contiguous())
        assert torch.equal(part, full[lo:hi]), (lo, hi)
    # used voxel-steps per DRR (38.7 M mean, 520-723 steps/ray)
    steps = count_steps(vol, det, frames[:64].contiguous(), full=True).double()
    per_drr = float(steps.sum()) / 64
    assert 30e6 < per_drr < 45e6, per_drr
    # first and last pose against the oracle (fp32 densities fed as f64), one
    # thread per ray (a 2-pose batch would otherwise split rays across lanes)
    flat = chest.astype(np.float64).ravel(order="F")
    det1 = Detector(256, 256, 2.8125, ray_split=1)
    img64 = render_frames(vol, det1, frames[[0, 1023]].contiguous(), out_dtype=torch.float64)
    assert torch.equal(img64.float(), full[[0, 1023]])
    for i, b in enumerate((0, 1023)):
        ref = O.render(flat, chest.shape, C2_SPACING, (0, 0, 0), frames[b].cpu().numpy(),
                       256, 256, 2.8125, 2.8125)
        np.testing.assert_array_equal(img64[i].cpu().numpy(), ref)


def _c5_volume(n=512, spacing=0.703125):
    from paper_2208_12737_b200 import synthetic
    vol = synthetic.make_phantom("sphere", n, spacing) + \
        synthetic.make_phantom("off_center_cube", n, spacing, 3.0)
    rng = np.random.default_rng(5)
    vol = vol + 0.01 * rng.standard_normal(vol.shape) * (vol > 0)
    return np.clip(vol, 0.0, None).astype(np.float32)


def test_c5_large_case(cuda_device):
    from paper_2208_12737_b200 import (DRR, DeviceVolume, Detector, backward_frames,
                                       backward_from_jac, pose_frames, render_frames,
                                       render_frames_jac, renderer)
    from paper_2208_12737_b200.metrics import neg_zncc
    data = _c5_volume()
    vol = DeviceVolume(data, 0.703125)
    det = Detector(1024, 1024, 0.703125)
    eta = np.array([[300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0],
                    [300.0, 0.9, 1.1, 0.2, 3.0, -2.0, 1.0]])
    frames = pose_frames(torch.tensor(eta, device=cuda_device), vol.center).detach()
    img64 = render_frames(vol, det, frames, out_dtype=torch.float64)
    img, jac = render_frames_jac(vol, det, frames, out_dtype=torch.float64)
    assert torch.equal(img, img64)
    # 4096 sampled pixels of each pose against the oracle's explicit-ray walk
    flat = data.astype(np.float64).ravel(order="F")
    rng = np.random.default_rng(11)
    for b in range(2):
        f = frames[b].cpu().numpy()
        pix = O.detector_grid(f, 1024, 1024, 0.703125, 0.703125)
        hh = rng.integers(0, 1024, 4096)
        ww = rng.integers(0, 1024, 4096)
        ref = O.raysum(flat, data.shape, (0.703125,) * 3, (0, 0, 0), f[:3], pix[hh, ww])
        np.testing.assert_array_equal(img64[b].cpu().numpy()[hh, ww], ref)
    # one walk + contraction == fused re-walk (same fixed reduction order)
    g = torch.randn((2, 1024, 1024), device=cuda_device, dtype=torch.float32)
    np.testing.assert_array_equal(backward_from_jac(det, jac, g).cpu().numpy(),
                                  backward_frames(vol, det, frames, g).cpu().numpy())
    # module path above the Jacobian budget re-walks in backward; same gradient
    drr = DRR(data, 0.703125, sdr=300.0, height=1024, delx=0.703125, device=cuda_device)
    fixed = img[:1].float()

    def grad():
        rot = torch.tensor(eta[1, 1:4], device=cuda_device, requires_grad=True)
        tra = torch.tensor(eta[1, 4:7], device=cuda_device, requires_grad=True)
        neg_zncc(drr(rot, tra), fixed[0]).backward()
        return torch.cat([rot.grad, tra.grad]).cpu().numpy()

    one_walk = grad()
    budget = renderer.JAC_BUDGET_BYTES
    try:
        renderer.JAC_BUDGET_BYTES = 0
        rewalk = grad()
    finally:
        renderer.JAC_BUDGET_BYTES = budget
    np.testing.assert_allclose(one_walk, rewalk, rtol=1e-12, atol=1e-15)
    # C5's 64-pose batch (3.2 GB of Jacobian) stays on the stored-Jacobian chain
    assert renderer.jac_bytes(det, 64) <= budget
