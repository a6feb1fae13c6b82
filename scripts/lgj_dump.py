"""Dump the stored-Jacobian chain's per-pose loss and gradient (C2 volume:
256 and 32 poses at 200^2, 300 poses at 77 x 53 -- both contraction paths of
k_loss_grad_jac) to an .npz, for
bitwise A/B of library variants run in separate processes
(DRR_B200_LIB=... python scripts/lgj_dump.py out.npz)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_12737_b200 import DeviceVolume, Detector, synthetic  # noqa: E402
from paper_2208_12737_b200.registration import loss_and_gradient  # noqa: E402

dev = torch.device("cuda")
truth = (300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)
out = {}
vol = DeviceVolume(synthetic.chest_phantom(), (0.703125, 0.703125, 2.5), device=dev)
for name, det, n in (("c2", Detector(200, 200, 3.6), 256), ("c2_small", Detector(200, 200, 3.6), 32),
                     ("odd", Detector(77, 53, 7.0), 300)):
    eta = torch.tensor(synthetic.sample_poses(truth, synthetic.NARROW_HALF_WIDTHS, n, seed=1),
                       device=dev)
    fixed = torch.rand((det.height, det.width), device=dev, generator=torch.Generator(dev).manual_seed(3))
    v, g = loss_and_gradient(vol, det, eta, fixed, mode="jac")
    out[name + "_v"], out[name + "_g"] = v.cpu().numpy(), g.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
