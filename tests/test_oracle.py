"""Pin the C oracle (oracle/siddon_oracle.c) to the reference before trusting
it: every golden vector in tests/golden/reference_golden.npz was produced by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import kernel_case, slab_chord_length
from oracle import oracle as O


def test_kernel_cases_bitwise(golden):
    """Random volumes (dims 1..7) x rays incl. axis-parallel, corner and face
    shots (test_kernel_properties.py:19-41): energies and forward-mode tangents
    bit-identical to the reference's native kernels (_native.pyx:140-282)."""
    for c in range(int(golden["k_count"])):
        k = kernel_case(golden, c)
        e = O.raysum(k["flat"], k["dims"], k["spacing"], k["origin"], k["source"], k["pixels"])
        np.testing.assert_array_equal(e, k["energy"], err_msg=f"case {c}")
        e2, de = O.raysum_grad(k["flat"], k["dims"], k["spacing"], k["origin"], k["source"],
                               k["d_source"], k["pixels"], k["d_pixels"])
        np.testing.assert_array_equal(e2, k["energy"])
        np.testing.assert_array_equal(de, k["d_energy"], err_msg=f"case {c}")
        # python backend agrees within 1e-9 (test_kernel_properties.py:44-63)
        scale = max(1.0, float(np.abs(e).max()))
        np.testing.assert_allclose(k["energy_python"], e, atol=1e-9 * scale, rtol=0)


def test_reverse_mode_equals_forward_mode(golden):
    """The reverse-mode endpoint gradients the GPU backward computes, contracted
    with the tangents, reproduce the reference's forward-mode d_energy."""
    for c in range(int(golden["k_count"])):
        k = kernel_case(golden, c)
        e, dEds, dEdp = O.raysum_endpoint_grad(k["flat"], k["dims"], k["spacing"], k["origin"],
                                               k["source"], k["pixels"])
        np.testing.assert_array_equal(e, k["energy"])
        de = dEds @ k["d_source"] + np.einsum("na,nat->nt", dEdp, k["d_pixels"])
        scale = max(1.0, float(np.abs(k["d_energy"]).max()))
        np.testing.assert_allclose(de, k["d_energy"], atol=1e-10 * scale, rtol=0)


def test_known_answers(golden):
    expect = [1.0, np.sqrt(3.0), 0.0, 0.0, 1.0]
    for i in range(int(golden["ka_count"])):
        e = O.raysum(np.ones(1), (1, 1, 1), (1.0,) * 3, (0.0,) * 3,
                     golden[f"ka{i}_source"], golden[f"ka{i}_pixel"])
        np.testing.assert_array_equal(e, golden[f"ka{i}_energy"])
        if i < len(expect):
            assert e[0] == pytest.approx(expect[i], abs=1e-12)


def test_uniform_chord_law():
    dims, spacing, origin = (8, 10, 12), (1.0, 1.5, 0.75), (-3.0, 1.0, 0.5)
    rng = np.random.default_rng(7)
    src = rng.uniform(-40, -20, size=3)
    pix = rng.uniform([0, -5, -5], [40, 25, 25], size=(50, 3))
    e = O.raysum(np.full(int(np.prod(dims)), 2.5), dims, spacing, origin, src, pix)
    lo = np.asarray(origin)
    hi = lo + np.asarray(dims) * np.asarray(spacing)
    for k in range(50):
        assert e[k] == pytest.approx(2.5 * slab_chord_length(src, pix[k], lo, hi), rel=1e-10, abs=1e-12)


def test_pose_frames_and_renders(golden):
    """orc_pose_frame + orc_detector_grid + orc_render reproduce the
    reference's detector_grid (geometry.py:166-175) and render() bitwise."""
    for i, eta in enumerate(golden["ps_poses"]):
        f = O.pose_frame(eta, golden["ps_center"])
        np.testing.assert_array_equal(f[:3], golden["ps_sources"][i])
        pix = O.detector_grid(f, 21, 21, 4.0, 4.0)
        np.testing.assert_array_equal(pix, golden["ps_pixels"][i])
        img = O.render(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                       golden["ps_origin"], f, 21, 21, 4.0, 4.0)
        np.testing.assert_array_equal(img, golden["ps_images"][i])


def test_loss_and_gradient(golden):
    """neg-ZNCC value (bitwise) and the reverse-mode pose gradient vs the
    reference's forward-mode loss_and_gradient (gradients.py:61-69)."""
    for i, eta in enumerate(golden["ps_poses"]):
        if not np.isfinite(golden["ps_values"][i]):
            continue
        f = O.pose_frame(eta, golden["ps_center"])
        img = O.render(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                       golden["ps_origin"], f, 21, 21, 4.0, 4.0)
        val, pg = O.neg_zncc_value_and_grad(img, golden["ps_fixed"])
        assert val == golden["ps_values"][i]
        _, gf = O.render_backward(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                                  golden["ps_origin"], f, 21, 21, 4.0, 4.0, pg)
        g = gf @ O.frame_jacobian(eta, golden["ps_center"])
        ref = golden["ps_grads"][i]
        np.testing.assert_allclose(g, ref, atol=1e-11 * np.abs(ref).max(), rtol=0)


def test_c1_and_blob(golden):
    from paper_2208_12737_b200 import synthetic
    vol = synthetic.make_phantom("sphere", 128, 1.0)
    flat = vol.ravel(order="F")
    assert hashlib.sha256(flat.tobytes()).hexdigest() == str(golden["c1_sha"])
    center = (64.0, 64.0, 64.0)
    f = O.pose_frame(golden["c1_pose"], center)
    img, steps = O.render(flat, (128,) * 3, (1.0,) * 3, (0.0,) * 3, f, 100, 100, 2.56, 2.56,
                          with_steps=True)
    np.testing.assert_array_equal(img, golden["c1_image"])
    assert int(steps.sum()) == int(golden["c1_steps"])
    val, pg = O.neg_zncc_value_and_grad(img, golden["c1_fixed"])
    assert val == float(golden["c1_value"])
    _, gf = O.render_backward(flat, (128,) * 3, (1.0,) * 3, (0.0,) * 3, f, 100, 100, 2.56, 2.56, pg)
    g = gf @ O.frame_jacobian(golden["c1_pose"], center)
    np.testing.assert_allclose(g, golden["c1_grad"], atol=1e-10 * np.abs(golden["c1_grad"]).max(), rtol=0)
    blob = synthetic.blob_phantom(64, 4.0)
    assert hashlib.sha256(blob.ravel(order="F").tobytes()).hexdigest() == str(golden["blob_sha"])
    for key in ("shifted", "truth"):
        f = O.pose_frame(golden[f"blob_{key}_pose"], (128.0,) * 3)
        img = O.render(blob.ravel(order="F"), (64,) * 3, (4.0,) * 3, (0.0,) * 3, f, 100, 100, 4.0, 4.0)
        np.testing.assert_array_equal(img, golden[f"blob_{key}"])


def test_frame_jacobian_matches_fd():
    eta = np.array([300.0, 0.4, 1.3, 0.1, 2.0, -1.0, 0.5])
    J = O.frame_jacobian(eta, (1.0, 2.0, 3.0))
    fd = np.zeros_like(J)
    for i in range(7):
        h = 1e-6
        ep, em = eta.copy(), eta.copy()
        ep[i] += h
        em[i] -= h
        fd[:, i] = (O.pose_frame(ep, (1.0, 2.0, 3.0)) - O.pose_frame(em, (1.0, 2.0, 3.0))) / (2 * h)
    np.testing.assert_allclose(J, fd, atol=1e-6)


def test_live_reference_when_available():
    """In the build container the reference itself is importable: spot-check
    the oracle against a fresh reference render (skipped on the GPU box)."""
    dt = O.reference_module()
    if dt is None:
        pytest.skip("reference not built here")
    vol = dt.make_phantom("sphere", 24, 1.5)
    spec = dt.DetectorSpec.for_volume(vol, 33, 27, (2.0, 2.5))
    pose = dt.PoseParameters(80.0, 2.1, 0.9, -0.7, (1.5, -2.0, 0.25))
    ref = dt.render(vol, pose, spec).values
    f = O.pose_frame(pose.to_vector(), vol.center)
    img = O.render(vol.flat_data(), vol.dims, vol.spacing, vol.plane_origin, f, 33, 27, 2.0, 2.5)
    np.testing.assert_array_equal(img, ref)
