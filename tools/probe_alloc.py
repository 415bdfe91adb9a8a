"""Time Forest.reserve / torch allocation patterns on the GPU box."""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16310_b200 as ow  # noqa: E402

dom = ow.Aabb((0, 0, 0), (1, 1, 1))
for it in range(6):
    f = ow.init_root_grid(dom, (16, 16, 16), capacity=32768)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f.reserve(121632)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x = [torch.empty(121632 * 2, dtype=torch.int32, device="cuda") for _ in range(7)]
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"reserve {1e3 * (t1 - t0):.3f} ms   7x empty {1e3 * (t2 - t1):.3f} ms")
    del x
