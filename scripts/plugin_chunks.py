"""Per-chunk cost of the cuda backend's siddon_raysum_grad at C2 (one pose's
40 000 rays in the reference's 2048-ray chunks, or as one call): wall time per
call and the kernel's own device time.  Measurement script."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2208_12737_b200 import backend_cuda as B, synthetic  # noqa: E402
from paper_2208_12737_b200.geometry import pose_frames  # noqa: E402

dims, sp = (512, 512, 133), (0.703125, 0.703125, 2.5)
flat = synthetic.chest_phantom(dims).astype(np.float64).ravel(order="F")
flat.flags.writeable = False
center = tuple(0.5 * n * s for n, s in zip(dims, sp))
f = pose_frames(torch.tensor([[300.0, 0.4, 1.3, 0.1, 0, 0, 0]], dtype=torch.float64), center)[0].numpy()
H = W = 200
ah = (np.arange(H) - (H - 1) / 2) * 3.6
aw = (np.arange(W) - (W - 1) / 2) * 3.6
pix = (f[3:6][None, None] + ah[:, None, None] * f[6:9] + aw[None, :, None] * f[9:12]).reshape(-1, 3)
src = f[:3]
rng = np.random.default_rng(0)
dsrc = rng.standard_normal((3, 7))
dpix = rng.standard_normal((pix.shape[0], 3, 7))
out = {}
for chunk in (2048, 16384, 40000):
    B.siddon_raysum_grad(flat, dims, sp, (0, 0, 0), src, dsrc, pix[:chunk], dpix[:chunk])
    t = []
    for _ in range(5):
        t0 = time.perf_counter()
        for s in range(0, pix.shape[0], chunk):
            B.siddon_raysum_grad(flat, dims, sp, (0, 0, 0), src, dsrc, pix[s:s + chunk],
                                 dpix[s:s + chunk])
        t.append(time.perf_counter() - t0)
    out[f"grad_chunk{chunk}_ms_per_40k"] = 1e3 * float(np.median(t))
    # kernel only, one chunk (events around the launch the backend makes)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    orig = B._lib.load().drr_raysum_tangents
    times = []

    class Timed:
        def __call__(self, *a):
            ev[0].record()
            rc = orig(*a)
            ev[1].record()
            return rc
    lib = B._lib.load()
    lib.drr_raysum_tangents = Timed()
    for _ in range(5):
        B.siddon_raysum_grad(flat, dims, sp, (0, 0, 0), src, dsrc, pix[:chunk], dpix[:chunk])
        times.append(ev[0].elapsed_time(ev[1]))
    lib.drr_raysum_tangents = orig
    out[f"grad_chunk{chunk}_kernel_ms"] = float(np.median(times))
print(json.dumps(out))
