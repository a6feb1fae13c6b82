"""Batched loss landscape (registration.loss_landscape) vs the reference's
(registration.py:159-203) golden sweeps; device volume ingest renders
identically."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_landscape_matches_reference(golden, cuda_device):
    from paper_2208_12737_b200 import DeviceVolume, Detector
    from paper_2208_12737_b200.registration import loss_landscape
    vol = DeviceVolume.from_flat(golden["ps_flat"], golden["ps_dims"], golden["ps_spacing"],
                                 golden["ps_origin"], device=cuda_device)
    det = Detector(21, 21, 4.0)
    g1 = loss_landscape(vol, det, golden["ls_truth"], axes=("theta",), samples=11)
    np.testing.assert_allclose(g1.coords[0], golden["ls1_coords"], rtol=0, atol=0)
    np.testing.assert_allclose(g1.losses, golden["ls1_losses"], atol=1e-5)
    g2 = loss_landscape(vol, det, golden["ls_truth"], axes=("phi", "bx"), samples=(5, 7),
                        half_widths=(0.4, 150.0), chunk=8)
    ref = golden["ls2_losses"]
    assert np.array_equal(np.isinf(g2.losses), np.isinf(ref))
    fin = np.isfinite(ref)
    np.testing.assert_allclose(g2.losses[fin], ref[fin], atol=1e-4)
    # convexity near the optimum (acceptance criterion 5 shape): truth is the minimum
    assert np.argmin(g1.losses) == 5


def test_dvol_ingest_renders_identically(tmp_path, cuda_device):
    from paper_2208_12737_b200 import DeviceVolume, Detector, render_frames, synthetic
    from paper_2208_12737_b200.volume_io import load_dvol, save_dvol
    from oracle import oracle as O
    data = synthetic.blob_phantom(32, 4.0)
    a = DeviceVolume(data, 4.0, device=cuda_device)
    p = tmp_path / "blob.dvol"
    save_dvol(DeviceVolume(data, 4.0, device=cuda_device, dtype=torch.float64), p)
    b = load_dvol(p, device=cuda_device)
    f = torch.tensor(O.pose_frame(np.array([300.0, 0.4, 1.3, 0.1, 2, -1, 0.5]), a.center),
                     device=cuda_device)[None]
    det = Detector(64, 64, 2.0)
    assert torch.equal(render_frames(a, det, f), render_frames(b, det, f))
