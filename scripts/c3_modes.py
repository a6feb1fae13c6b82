"""C3 (250-step registration on the C2 volume, one pose, whole loop one CUDA
graph): ms per step with the stored-Jacobian iteration (4 launches: frames,
forward_jac, loss_grad_jac, register_update) vs the three-launch
drr_register_step iteration.  Last run: 0.0880 vs 0.0854 ms."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_12737_b200 import DRR, synthetic  # noqa: E402
from paper_2208_12737_b200.registration import OptimizerConfig, RegistrationEngine  # noqa: E402

dev = torch.device("cuda")
truth = (300.0, math.pi / 2, math.pi / 2, 0.0, 0.0, 0.0, 0.0)
drr = DRR(synthetic.chest_phantom(), (0.703125, 0.703125, 2.5), 300.0, 200, 3.6, device=dev)
with torch.no_grad():
    fixed = drr(torch.tensor(truth[1:4], dtype=torch.float64, device=dev),
                torch.tensor(truth[4:7], dtype=torch.float64, device=dev))
p0 = synthetic.sample_poses(truth, synthetic.NARROW_HALF_WIDTHS, 1, seed=0)
cfg = OptimizerConfig(converged_threshold=-1.1)
out = {}
for mode in ("jac", "fused"):
    eng = RegistrationEngine(drr.volume, drr.detector, fixed, 1, cfg, mode=mode)
    ts = []
    for i in range(6):
        eng.reset(p0)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        eng.run(use_graph=True)
        b.record()
        b.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    out[mode] = {"ms_per_step": float(np.median(ts)) / (cfg.max_iters + 1),
                 "final_loss": eng.traces()[0].final_loss}
print(json.dumps(out))
