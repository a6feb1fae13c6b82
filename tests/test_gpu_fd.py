"""Finite differences "reported alongside" (north star):
fd.finite_difference_gradient / detect_fd_boundaries / fd_report on the GPU,
held to the reference's own bars (test_gradients.py:119-165):

* central FD agrees with the exact gradient to 1e-5 relative on every
  component whose stencil is kink-free, for 12 random poses (any disagreement
  must be explained by a detected boundary);
* the FD error shrinks with the step (1e-6 steps: 1e-4 relative);
* a deliberately huge step is detected as crossing a boundary;
* the boundary detector agrees with the reference's own detect_fd_boundaries
  (oracle/_ref, python_ref.ray_structure hashing) on the same poses.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TRUTH = np.array([100.0, 0.3, 1.2, 0.1, 0.0, 0.0, 0.0])


@pytest.fixture(scope="module")
def setup(cuda_device):
    from paper_2208_12737_b200 import Detector, DeviceVolume, _lib, synthetic
    from paper_2208_12737_b200.fd import _frames
    data = synthetic.make_phantom("sphere", 16, 2.0)
    vol = DeviceVolume(data, 2.0, device=cuda_device, dtype=torch.float64)
    det = Detector(21, 21, 4.0, ray_split=1)
    fr = _frames(vol, TRUTH[None])
    img = torch.empty((1, 21, 21), dtype=torch.float64, device=cuda_device)
    _lib.check(_lib.load().drr_forward(vol.flat.data_ptr(), vol.vol_dtype, vol.grid,
                                       fr.data_ptr(), 1, det.c, img.data_ptr(), 1,
                                       torch.cuda.current_stream().cuda_stream))
    return data, vol, det, img[0].cpu().numpy()


def test_random_poses_match_fd_or_boundary(setup):
    from paper_2208_12737_b200.fd import fd_report
    _, vol, det, fixed = setup
    rng = np.random.default_rng(11)
    worst = 0.0
    for _ in range(12):
        while True:
            eta = TRUTH + rng.uniform(-1, 1, 7) * np.array([0, 0.4, 0.4, 0.3, 8.0, 8.0, 8.0])
            if abs(math.sin(eta[2])) > 0.1:
                break
        rep = fd_report(vol, det, eta, fixed)
        assert not rep["unexplained"], rep
        if rep["max_rel_kink_free"] is not None:
            worst = max(worst, rep["max_rel_kink_free"])
    assert worst < 1e-5


def test_fd_error_shrinks_with_step(setup):
    from paper_2208_12737_b200.fd import finite_difference_gradient
    from paper_2208_12737_b200.registration import loss_and_gradient
    _, vol, det, fixed = setup
    eta = np.array([100.0, 0.35, 1.15, 0.12, 1.0, -2.0, 0.5])
    _, g = loss_and_gradient(vol, det, eta[None], fixed, image_dtype=torch.float64)
    fd = finite_difference_gradient(vol, det, eta, fixed, steps=np.full(7, 1e-6))
    np.testing.assert_allclose(fd, g[0].cpu().numpy(), rtol=1e-4, atol=1e-10)


def test_large_step_crosses_boundary(setup):
    from paper_2208_12737_b200.fd import detect_fd_boundaries
    _, vol, det, _ = setup
    eta = np.array([100.0, 0.35, 1.15, 0.12, 1.0, -2.0, 0.5])
    assert detect_fd_boundaries(vol, det, eta, steps=np.full(7, 2.0)).any()


def test_boundaries_agree_with_reference(setup):
    from oracle.oracle import reference_module
    from paper_2208_12737_b200.fd import detect_fd_boundaries
    dt = reference_module()
    if dt is None:
        pytest.skip("oracle/_ref not built")
    data, vol, det, _ = setup
    rvol = dt.Volume((16, 16, 16), (2.0, 2.0, 2.0), (0.0, 0.0, 0.0), data)
    spec = dt.DetectorSpec.for_volume(rvol, 21, 21, (4.0, 4.0))
    rng = np.random.default_rng(5)
    for steps in (dt.default_fd_steps(), np.full(7, 0.05), np.full(7, 2.0)):
        for _ in range(3):
            eta = TRUTH + rng.uniform(-1, 1, 7) * np.array([0, 0.4, 0.4, 0.3, 8.0, 8.0, 8.0])
            ref = dt.detect_fd_boundaries(rvol, dt.PoseParameters.from_vector(eta), spec,
                                          steps=steps)
            got = detect_fd_boundaries(vol, det, eta, steps=steps)
            np.testing.assert_array_equal(got, ref, err_msg=f"eta={eta} steps={steps}")
