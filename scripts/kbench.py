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
from paper_2208_12737_b200 import (DRR, backward_frames, backward_from_jac, count_steps, pose_frames,
                                   render_frames, render_frames_jac, synthetic)

dev = torch.device("cuda")
vol = synthetic.chest_phantom()
drr = DRR(vol, (0.703125, 0.703125, 2.5), 300.0, 200, 3.6, device=dev, strict=False)
if os.environ.get("DRR_KBENCH_TRIM"):  # A/B of the trimming modes: "none", "box", "hull"
    from paper_2208_12737_b200 import DeviceVolume
    mode = {"hull": True, "box": "box", "none": False}[os.environ["DRR_KBENCH_TRIM"]]
    drr.volume = DeviceVolume(vol, (0.703125, 0.703125, 2.5), device=dev, trim=mode)
if os.environ.get("DRR_KBENCH_F64"):  # the CT held as float64 (same values)
    from paper_2208_12737_b200 import DeviceVolume
    drr.volume = DeviceVolume(vol, (0.703125, 0.703125, 2.5), device=dev, dtype=torch.float64)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
res = {}
truth = (300.0, math.pi / 2, math.pi / 2, 0, 0, 0, 0)
for B in [int(x) for x in (sys.argv[1:] or ["32", "1"])]:
    poses = synthetic.sample_poses(truth, synthetic.NARROW_HALF_WIDTHS, B, seed=0)
    frames = pose_frames(torch.tensor(poses, device=dev), drr.isocenter)
    S = float(count_steps(drr.volume, drr.detector, frames).double().sum())
    g = torch.randn((B, 200, 200), device=dev)
    from paper_2208_12737_b200 import _lib
    from paper_2208_12737_b200.registration import _Buffers
    lib = _lib.load()
    lb = _Buffers(drr.volume, drr.detector, B, mode="fused")
    et = torch.tensor(poses, device=dev)
    fixed = torch.rand((200, 200), device=dev)

    def fused():
        _lib.check(lib.drr_forward_loss_grad(
            drr.volume.flat.data_ptr(), 0, drr.volume.grid, frames.data_ptr(), et.data_ptr(), B,
            drr.detector.c, fixed.data_ptr(), 0, 0, lb.img.data_ptr(), 0, lb.value.data_ptr(),
            lb.status.data_ptr(), lb.grad_frames.data_ptr(), lb.grad_eta.data_ptr(),
            lb.ws.data_ptr(), lb.ws_bytes, torch.cuda.current_stream().cuda_stream))
    fns = {"fl": fused,
           "fwd": lambda: render_frames(drr.volume, drr.detector, frames),
           "bwd": lambda: backward_frames(drr.volume, drr.detector, frames, g),
           "fj": lambda: hold.update(zip(("img", 0), render_frames_jac(drr.volume, drr.detector,
                                                                        frames))),
           "bj": lambda: backward_from_jac(drr.detector, hold[0], g),
           "lgj": lambda: _lib.check(lib.drr_loss_grad_jac(
               hold[0].data_ptr(), hold["img"].data_ptr(), fixed.data_ptr(), 0, 0, B,
               drr.detector.c, _lib.DRR_LOSS_NEG_ZNCC, lb.value.data_ptr(), None,
               lb.grad_frames.data_ptr(), None, None, torch.cuda.current_stream().cuda_stream))}
    hold = {}
    t = {k: [] for k in fns}
    for i in range(12):
        for k, fn in fns.items():
            flush.fill_(1)
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); fn(); b.record(); b.synchronize()
            if i >= 2:
                t[k].append(a.elapsed_time(b))
    m = {k: float(np.median(v)) for k, v in t.items()}
    res[B] = {"fused_loss_ms": m["fl"], "fwd_ms": m["fwd"], "bwd_ms": m["bwd"], "fwd_jac_ms": m["fj"], "bwd_jac_ms": m["bj"],
              "loss_grad_jac_ms": m["lgj"], "steps_per_drr": S / B,
              "fwd_gsteps_s": S / m["fwd"] / 1e6, "fwd_jac_gsteps_s": S / m["fj"] / 1e6,
              "rewalk_drr_s": B / ((m["fwd"] + m["bwd"]) / 1e3),
              "one_walk_drr_s": B / ((m["fj"] + m["bj"]) / 1e3)}
print(json.dumps(res))
