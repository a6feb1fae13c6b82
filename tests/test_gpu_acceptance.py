"""The reference's acceptance criteria that concern this path, on the GPU
(pkg/tests/test_acceptance.py), with the reference's own
fixtures: blob64 (64^3 sphere + 3x off-centre cube @ 4 mm), TRUTH =
(rho 400, theta 0.4, phi 1.3, gamma 0.1), a 100^2 detector at 4 mm.

* criterion 6 (test_acceptance.py:185-203): 50 wide-range initialisations
  (seed 0) registered against the TRUTH render: >= 35 converge, mean
  iterations of converged runs <= 150 -- here as ONE batched, graph-captured
  registration of all 50;
* criterion 7 (test_acceptance.py:206-233): render time non-decreasing in
  detector size, 200^2 at most 8x 100^2, gradient render < 10x primal.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

RHO = 400.0
TRUTH = (RHO, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0)
WIDE_HALF_WIDTHS = (0.0, math.radians(60.0), math.radians(60.0), math.radians(60.0),
                    30.0, 30.0, 30.0)  # registration.py:34-38


@pytest.fixture(scope="module")
def blob(cuda_device):
    from paper_2208_12737_b200 import DeviceVolume, synthetic
    return DeviceVolume(synthetic.blob_phantom(64, 4.0), 4.0, device=cuda_device)


def test_criterion_6_registration_population(blob, cuda_device):
    from paper_2208_12737_b200 import Detector, pose_frames, render_frames, synthetic
    from paper_2208_12737_b200.registration import OptimizerConfig, register_batch
    det = Detector(100, 100, 4.0)
    f = pose_frames(torch.tensor([TRUTH], dtype=torch.float64, device=cuda_device), blob.center).detach()
    fixed = render_frames(blob, det, f)[0]
    inits = synthetic.sample_poses(TRUTH, WIDE_HALF_WIDTHS, 50, seed=0)
    cfg = OptimizerConfig()
    traces = register_batch(fixed, blob, inits, det, cfg, use_graph=True)
    converged = [t for t in traces if t.converged]
    for t in traces:
        assert t.converged == (t.final_loss < cfg.converged_threshold)
    mean_iters = float(np.mean([t.iterations_used for t in converged]))
    assert len(converged) >= 35, len(converged)
    assert mean_iters <= 150.0, mean_iters


def test_criterion_7_performance_scaling(blob, cuda_device):
    from paper_2208_12737_b200 import (Detector, backward_from_jac, pose_frames, render_frames,
                                       render_frames_jac)
    f = pose_frames(torch.tensor([TRUTH], dtype=torch.float64, device=cuda_device), blob.center).detach()

    def timed(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    times = {}
    for size in (100, 200, 300):
        det = Detector(size, size, 400.0 / size)
        times[size] = timed(lambda: render_frames(blob, det, f))
    assert times[100] <= times[200] * 1.05 and times[200] <= times[300] * 1.05, times
    assert times[200] <= 8.0 * times[100], times
    det = Detector(100, 100, 4.0)
    g = torch.ones((1, 100, 100), device=cuda_device)
    grad_t = timed(lambda: backward_from_jac(det, render_frames_jac(blob, det, f)[1], g))
    assert grad_t < 10.0 * times[100], (grad_t, times[100])
