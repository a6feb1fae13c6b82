"""Single-pose timings of the one-walk step kernels per ray split K (C2 volume, 200^2; C1)."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_12737_b200 import (DeviceVolume, Detector, backward_from_jac, pose_frames,  # noqa: E402
                                   render_frames, render_frames_jac, synthetic)

dev = torch.device("cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def timed(fn, n=20):
    ts = []
    for i in range(n + 3):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


vol = DeviceVolume(synthetic.chest_phantom(), (0.703125, 0.703125, 2.5), device=dev)
f = pose_frames(torch.tensor([[300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0]], dtype=torch.float64, device=dev),
                vol.center).detach()
v1 = DeviceVolume(synthetic.make_phantom("sphere", 128, 1.0), 1.0, device=dev)
f1 = pose_frames(torch.tensor([[300.0, 0.4, 1.3, 0.1, 0.0, 0.0, 0.0]], dtype=torch.float64, device=dev), v1.center).detach()
g = torch.randn((1, 200, 200), device=dev)
res = {}
for K in (0, 1, 2, 4, 8):
    det = Detector(200, 200, 3.6, ray_split=K)
    hold = {}

    def step():
        hold["i"], hold["j"] = render_frames_jac(vol, det, f)
        backward_from_jac(det, hold["j"], g)
    d1 = Detector(100, 100, 2.56, ray_split=K)
    res[K] = {"c2_fwd_jac_bwd_ms": timed(step), "c2_fwd_ms": timed(lambda: render_frames(vol, det, f)),
              "c1_fwd_ms": timed(lambda: render_frames(v1, d1, f1))}
print(json.dumps(res))
