"""C5 (512^3 ball + cube, 1024^2, 64 poses) loss_and_gradient: the stored-Jacobian
chain vs the fused walk, device time (A/B for registration._Buffers' auto rule)."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2208_12737_b200 import DeviceVolume, Detector, synthetic  # noqa: E402
from paper_2208_12737_b200.registration import _Buffers, loss_and_gradient  # noqa: E402

dev = torch.device("cuda")
vol = DeviceVolume(bench.c5_volume(dev), 0.703125, device=dev)
det = Detector(1024, 1024, 0.703125)
truth = (300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)
eta = torch.tensor(synthetic.sample_poses(truth, synthetic.NARROW_HALF_WIDTHS, 64, seed=0),
                   device=dev)
fixed = torch.rand((1024, 1024), device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
out = {}
for mode in ("jac", "fused"):
    buf = _Buffers(vol, det, 64, mode=mode)
    ts = []
    for i in range(5):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        loss_and_gradient(vol, det, eta, fixed, buffers=buf)
        b.record()
        b.synchronize()
        if i >= 1:
            ts.append(a.elapsed_time(b))
    out[mode] = float(np.median(ts))
    del buf
    torch.cuda.empty_cache()
print(json.dumps(out))
