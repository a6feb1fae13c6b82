"""C3: slice-to-volume registration, 250 momentum-GD steps of
neg-ZNCC fwd+bwd on the 512x512x133 chest volume (200^2 @ 3.6 mm), fixed DRR
at truth (300, pi/2, pi/2, 0), pose0 = first narrow sample (seed 0), threshold
-1.1 so every step runs.  The whole loop is one CUDA graph; reports ms/step
for 1 registration and for a batched population."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_12737_b200 import DRR, synthetic
from paper_2208_12737_b200.registration import OptimizerConfig, RegistrationEngine

dev = torch.device("cuda")
truth = (300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)
drr = DRR(synthetic.chest_phantom(), (0.703125, 0.703125, 2.5), 300.0, 200, 3.6, device=dev,
          strict=False)
with torch.no_grad():
    fixed = drr(torch.tensor(truth[1:4], device=dev), torch.tensor(truth[4:], device=dev))
cfg = OptimizerConfig(converged_threshold=-1.1)
out = {}
for B in [int(x) for x in (sys.argv[1:] or ["1", "64"])]:
    poses = synthetic.sample_poses(truth, synthetic.NARROW_HALF_WIDTHS, B, seed=0)
    eng = RegistrationEngine(drr.volume, drr.detector, fixed, B, cfg)
    eng.reset(poses)
    eng.run(use_graph=True)  # capture + first replay
    times = []
    for _ in range(3):
        eng.reset(poses)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        eng.run(use_graph=True)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
    tr = eng.traces()
    ms = float(np.median(times))
    out[B] = {"ms_total": ms, "ms_per_step": ms / (cfg.max_iters + 1),
              "registrations_per_s": B / (ms / 1e3),
              "fwd_bwd_drr_s": B * (cfg.max_iters + 1) / (ms / 1e3),
              "final_loss_median": float(np.median([t.final_loss for t in tr])),
              "first_loss_median": float(np.median([t.losses[0] for t in tr]))}
print(json.dumps(out))
