"""C1 / C4 / C5 timings alone (bench.other_configs) for A/B iteration; prints one JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2208_12737_b200 import DeviceVolume, synthetic  # noqa: E402

dev = torch.device("cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def timed(fn, n, warm):
    out = []
    for i in range(n + warm):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        if i >= warm:
            out.append(e0.elapsed_time(e1))
    return out


vol = DeviceVolume(synthetic.chest_phantom(bench.DIMS), bench.SPACING, device=dev)
res = bench.other_configs(dev, vol, timed, flush)
print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "workload"} for k, v in res.items()}))
