"""Time the reference's own dispatcher on the "cuda" backend at C2.

The unmodified reference (oracle/_ref: drrtrace) with INTEGRATION.md section
2's patch applied by tests/ref_suite/drr_cuda_backend_plugin.py:
``render_with_gradient(volume, pose, spec, backend=...)`` (gradients.py:45-58)
-> ``ray_energies_with_tangents`` (raytrace.py:108-129, chunks of 2048 rays)
-> ``backend.siddon_raysum_grad``, for backend "cuda" and "native", on the C2
chest volume (200^2 detector, one pose), plus ``render`` (ray_energies,
chunks of 16384).  Measurement script (test infrastructure), not the product.
    PYTHONPATH=oracle/_ref:.:tests/ref_suite python scripts/plugin_c2.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (os.path.join(ROOT, "oracle", "_ref"), ROOT, os.path.join(ROOT, "tests", "ref_suite")):
    sys.path.insert(0, p)
import drr_cuda_backend_plugin  # noqa: F401,E402  (the patch)
import drrtrace as dt  # noqa: E402
import torch  # noqa: E402

from paper_2208_12737_b200 import synthetic  # noqa: E402

vol = dt.Volume((512, 512, 133), (0.703125, 0.703125, 2.5), (0.0, 0.0, 0.0),
                synthetic.chest_phantom().astype(np.float64))
spec = dt.DetectorSpec.for_volume(vol, 200, 200, (3.6, 3.6))
pose = dt.PoseParameters(300.0, 0.4, 1.3, 0.1)
out = {"workload": "C2 chest 512x512x133, 200x200 @3.6 mm, pose (300, 0.4, 1.3, 0.1): the "
                   "reference's render / render_with_gradient through its own dispatcher"}
res = {}
for backend in ("cuda", "native"):
    for name, fn in (("render", dt.render), ("render_with_gradient", dt.render_with_gradient)):
        reps = 5 if backend == "cuda" else 1
        fn(vol, pose, spec, backend=backend)  # warm (uploads + caches the volume on cuda)
        torch.cuda.synchronize()
        t = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = fn(vol, pose, spec, backend=backend)
            t.append(time.perf_counter() - t0)
        res[(backend, name)] = r
        out[f"{backend}_{name}_ms"] = 1e3 * float(np.median(t))
# the reference's own host work inside those calls (pixel grids and their
# tangents, gradients.py / geometry.py): the floor any backend sits on
for name, fn in (("detector_grid", lambda: dt.detector_grid(pose, spec)),
                 ("detector_grid_with_tangents", lambda: dt.detector_grid_with_tangents(pose, spec))):
    t = []
    for _ in range(5):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    out[f"host_{name}_ms"] = 1e3 * float(np.median(t))
img_c, img_n = res[("cuda", "render")].values, res[("native", "render")].values
out["render_bitwise_equal"] = bool(np.array_equal(img_c, img_n))
gc, gn = res[("cuda", "render_with_gradient")], res[("native", "render_with_gradient")]
out["rwg_image_bitwise_equal"] = bool(np.array_equal(gc[0].values, gn[0].values))
out["rwg_d_image_max_abs_diff"] = float(np.abs(gc[1] - gn[1]).max())
out["rwg_d_image_max_abs"] = float(np.abs(gn[1]).max())
print(json.dumps(out))
