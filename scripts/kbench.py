"""Kernel micro-benchmark for iteration (not the driver bench): times
k_forward / k_backward on C2 (chest 512x512x133, 200^2) for a pose batch and a
single pose, CUDA events, L2 flushed between launches."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_12737_b200 import DRR, backward_frames, count_steps, pose_frames, render_frames, synthetic

dev = torch.device("cuda")
vol = synthetic.chest_phantom()
drr = DRR(vol, (0.703125, 0.703125, 2.5), 300.0, 200, 3.6, device=dev, strict=False)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
res = {}
truth = (300.0, math.pi / 2, math.pi / 2, 0, 0, 0, 0)
for B in [int(x) for x in (sys.argv[1:] or ["32", "1"])]:
    poses = synthetic.sample_poses(truth, synthetic.NARROW_HALF_WIDTHS, B, seed=0)
    frames = pose_frames(torch.tensor(poses, device=dev), drr.isocenter)
    S = float(count_steps(drr.volume, drr.detector, frames).double().sum())
    g = torch.randn((B, 200, 200), device=dev)
    tf, tb = [], []
    for i in range(12):
        flush.fill_(1)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); render_frames(drr.volume, drr.detector, frames); b.record(); b.synchronize()
        flush.fill_(1)
        c, d = torch.cuda.Event(True), torch.cuda.Event(True)
        c.record(); backward_frames(drr.volume, drr.detector, frames, g); d.record(); d.synchronize()
        if i >= 2:
            tf.append(a.elapsed_time(b)); tb.append(c.elapsed_time(d))
    f, bw = float(np.median(tf)), float(np.median(tb))
    res[B] = {"fwd_ms": f, "bwd_ms": bw, "steps_per_drr": S / B,
              "fwd_gsteps_s": S / f / 1e6, "bwd_gsteps_s": S / bw / 1e6,
              "fwd_bwd_drr_s": B / ((f + bw) / 1e3)}
print(json.dumps(res))
