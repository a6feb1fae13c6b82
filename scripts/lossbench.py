import os
import sys

import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2208_12737_b200 import _lib
dev = torch.device("cuda")
for B in (1, 32):
    m = torch.rand((B, 200, 200), device=dev); f = torch.rand((200, 200), device=dev)
    val = torch.empty(B, dtype=torch.float64, device=dev); g = torch.empty_like(m)
    lib = _lib.load()
    def run():
        _lib.check(lib.drr_image_loss(m.data_ptr(), f.data_ptr(), 0, 0, B, 40000, _lib.DRR_LOSS_NEG_ZNCC, val.data_ptr(), g.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
    for _ in range(5): run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(100): run()
    b.record(); b.synchronize()
    print(B, a.elapsed_time(b) / 100 * 1000, "us per call")
