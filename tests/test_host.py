"""Host-side logic on CPU: pose -> frame geometry and its autograd Jacobian,
device losses, synthetic inputs, validation.  (The CUDA compute is covered by
the -m gpu tests.)"""

import math

import numpy as np
import pytest
import torch

from oracle import oracle as O


def test_pose_frames_bitwise_vs_oracle():
    from paper_2208_12737_b200.geometry import pose_frames
    rng = np.random.default_rng(0)
    eta = np.column_stack([rng.uniform(50, 500, 20), rng.uniform(-3, 3, (20, 3)),
                           rng.uniform(-20, 20, (20, 3))])
    iso = (12.5, -3.0, 100.25)
    f = pose_frames(torch.tensor(eta), iso).numpy()
    for i in range(20):
        np.testing.assert_array_equal(f[i], O.pose_frame(eta[i], iso))


def test_pose_frames_autograd_jacobian():
    """torch autograd through pose_frames equals the reference's tangent
    geometry (geometry.py:120-149 duals), so dL/dframe -> dL/dpose is exact."""
    from paper_2208_12737_b200.geometry import pose_frames
    eta = np.array([300.0, 0.4, 1.3, 0.1, 2.0, -1.0, 0.5])
    J = torch.autograd.functional.jacobian(
        lambda e: pose_frames(e[None], (1.0, 2.0, 3.0))[0], torch.tensor(eta))
    np.testing.assert_allclose(J.numpy(), O.frame_jacobian(eta, (1.0, 2.0, 3.0)), atol=1e-13)


def test_reference_tangents_equal_autograd():
    """Live cross-check with the reference's dual numbers when importable."""
    dt = O.reference_module()
    if dt is None:
        pytest.skip("reference not built here")
    from paper_2208_12737_b200.geometry import pose_frames
    pose = dt.PoseParameters(120.0, 0.7, 1.1, -0.3, (1.0, 2.0, -3.0))
    spec = dt.DetectorSpec(5, 4, (1.5, 2.0), (1.0, 2.0, 3.0))
    rays, d_source, d_pixels = dt.detector_grid_with_tangents(pose, spec)
    J = torch.autograd.functional.jacobian(
        lambda e: pose_frames(e[None], spec.isocenter)[0], torch.tensor(pose.to_vector())).numpy()
    np.testing.assert_allclose(J[0:3], d_source, atol=1e-13)
    a_h = (np.arange(5) - 2.0) * 2.0
    a_w = (np.arange(4) - 1.5) * 1.5
    dp = J[3:6][None, None] + a_h[:, None, None, None] * J[6:9][None, None] + \
        a_w[None, :, None, None] * J[9:12][None, None]
    np.testing.assert_allclose(dp, d_pixels, atol=1e-12)


def test_neg_zncc_value_and_pixel_grad():
    from paper_2208_12737_b200.metrics import neg_zncc, l2
    rng = np.random.default_rng(1)
    a = rng.random((13, 17))
    b = rng.random((13, 17)) + 0.3 * a
    ta = torch.tensor(a, requires_grad=True)
    v = neg_zncc(ta, torch.tensor(b))
    v.backward()
    rv, rg = O.neg_zncc_value_and_grad(a, b)
    assert float(v) == pytest.approx(rv, abs=1e-14)
    np.testing.assert_allclose(ta.grad.numpy(), rg, atol=1e-15)
    assert float(neg_zncc(torch.tensor(a), torch.tensor(a))) == pytest.approx(-1.0, abs=1e-12)
    assert float(l2(torch.tensor(a), torch.tensor(b))) == pytest.approx(np.linalg.norm(a - b))


def test_phantoms_match_reference_when_available():
    dt = O.reference_module()
    if dt is None:
        pytest.skip("reference not built here")
    from paper_2208_12737_b200 import synthetic
    for kind in ("uniform", "sphere", "off_center_cube", "single_voxel"):
        for dims, sp in (((9, 7, 5), (1.0, 2.0, 0.5)), (16, 2.0)):
            ref = dt.make_phantom(kind, dims, sp, 2.5).data
            np.testing.assert_array_equal(synthetic.make_phantom(kind, dims, sp, 2.5), ref)


def test_sample_poses_match_reference_when_available():
    dt = O.reference_module()
    if dt is None:
        pytest.skip("reference not built here")
    from paper_2208_12737_b200 import synthetic
    from drrtrace.registration import default_half_widths, sample_initializations
    truth = dt.PoseParameters(300.0, math.pi / 2, math.pi / 2, 0.0)
    ref = np.array([p.to_vector() for p in sample_initializations(truth, default_half_widths(), 16, 0)])
    np.testing.assert_array_equal(
        synthetic.sample_poses(truth.to_vector(), synthetic.NARROW_HALF_WIDTHS, 16, 0), ref)


def test_chest_phantom_shape_and_values():
    from paper_2208_12737_b200 import synthetic
    v = synthetic.chest_phantom((64, 64, 5))
    assert v.shape == (64, 64, 5) and v.dtype == np.float32
    assert v.min() >= 0 and v.max() > 1.9
    assert (v[:, :, 0] == 0).sum() > 0  # air outside the body


def test_module_validation_errors():
    from paper_2208_12737_b200 import DeviceVolume, Detector, InvalidArgumentError
    with pytest.raises(InvalidArgumentError):
        Detector(0, 10, 1.0)
    with pytest.raises(InvalidArgumentError):
        Detector(10, 10, -1.0)
    with pytest.raises(InvalidArgumentError):
        DeviceVolume(np.zeros((4, 4)), 1.0, device="cpu")
    with pytest.raises(InvalidArgumentError):
        DeviceVolume(np.zeros((4, 4, 4)), (1.0, 0.0, 1.0), device="cpu")


def test_device_volume_needs_cuda():
    """No CPU fallback: the layout pass is drr_volume_pack on the device (its
    x-fastest parity is tests/test_gpu_volume_pack.py), so a CPU device fails
    loudly instead of silently packing on the host."""
    from paper_2208_12737_b200 import DeviceVolume, InvalidArgumentError
    data = np.arange(2 * 3 * 4, dtype=np.float64).reshape(2, 3, 4)
    with pytest.raises(InvalidArgumentError):
        DeviceVolume(data, 1.0, device="cpu", dtype=torch.float64)
    with pytest.raises(InvalidArgumentError):
        DeviceVolume.from_flat(data.ravel(order="F"), (2, 3, 4), 1.0, device="cpu")


def test_gimbal_guard_host():
    from paper_2208_12737_b200.geometry import check_gimbal, check_pose_vectors
    from paper_2208_12737_b200 import GradientUndefinedError, InvalidArgumentError
    with pytest.raises(GradientUndefinedError):
        check_gimbal(torch.tensor([[100.0, 0.3, 0.0, 0, 0, 0, 0]]))
    check_gimbal(torch.tensor([[100.0, 0.3, 1e-3, 0, 0, 0, 0]]))
    with pytest.raises(InvalidArgumentError):
        check_pose_vectors(torch.tensor([[-1.0, 0.3, 1.0, 0, 0, 0, 0]]))
    with pytest.raises(InvalidArgumentError):
        check_pose_vectors(torch.tensor([[1.0, float("nan"), 1.0, 0, 0, 0, 0]]))


def test_api_types_mirror_reference():
    """api.Volume / PoseParameters / DetectorSpec / Image validate like the
    reference's dataclasses (volume.py:24-83, geometry.py:32-97,
    raytrace.py:29-47) and carry the same values; reference objects are
    accepted where ours are (same field names)."""
    import numpy as np
    import pytest
    from paper_2208_12737_b200 import api
    from paper_2208_12737_b200.errors import InvalidArgumentError
    bad = [lambda m: m.PoseParameters(0.0, 0.1, 1.0),
           lambda m: m.PoseParameters(100.0, float("nan"), 1.0),
           lambda m: m.DetectorSpec(0, 3),
           lambda m: m.DetectorSpec(3, 3, (0.0, 1.0)),
           lambda m: m.Volume((2, 2, 2), (1, -1, 1), (0, 0, 0), np.zeros(8)),
           lambda m: m.Volume((2, 2, 2), (1, 1, 1), (0, 0, 0), np.zeros(7)),
           lambda m: m.Image(np.zeros(3))]
    for make in bad:
        with pytest.raises(InvalidArgumentError):
            make(api)
    v = api.Volume((3, 4, 5), (1.0, 2.0, 0.5), (1.0, -2.0, 0.0), np.arange(60.0))
    p = api.PoseParameters.from_vector([300.0, 0.4, 1.3, 0.1, 1.0, 2.0, 3.0])
    s = api.DetectorSpec.for_volume(v, 7, 9, 2.5)
    dt = O.reference_module()
    if dt is None:
        return
    for make in bad:
        with pytest.raises(dt.errors.InvalidArgumentError if hasattr(dt, "errors") else Exception):
            make(dt)
    rv = dt.Volume((3, 4, 5), (1.0, 2.0, 0.5), (1.0, -2.0, 0.0), np.arange(60.0))
    assert v.center == rv.center and np.array_equal(v.flat_data(), rv.flat_data())
    assert np.array_equal(p.to_vector(), dt.PoseParameters.from_vector(p.to_vector()).to_vector())
    rs = dt.DetectorSpec.for_volume(rv, 7, 9, 2.5)
    assert (s.height, s.width, s.pixel_pitch, s.isocenter) == \
        (rs.height, rs.width, rs.pixel_pitch, rs.isocenter)
