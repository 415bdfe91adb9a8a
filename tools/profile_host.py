"""cProfile of the host side of one bench step (GPU box helper).

    python tools/profile_host.py [C2] [steps]
"""

import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])


def step():
    geom = ow.geometry.stl_records_to_coords(rec, n)
    f = ow.init_root_grid(dom, (cfg["root"],) * dim, capacity=32 * cfg["root"] ** dim)
    ow.refine_near_wall(f, geom, params)
    ow.build_lattice_links(f, geom, None, cfg["lattice"])


for _ in range(3):
    step()
torch.cuda.synchronize()

# log slow torch.empty calls (size, caller) during a few steps
import time as _t  # noqa: E402
import traceback  # noqa: E402

_orig_empty = torch.empty
slow = []


def _timed_empty(*a, **k):
    t0 = _t.perf_counter()
    r = _orig_empty(*a, **k)
    dt = _t.perf_counter() - t0
    if dt > 50e-6:
        fr = traceback.extract_stack(limit=3)[0]
        slow.append((round(dt * 1e6), tuple(r.shape), str(r.dtype), f"{os.path.basename(fr.filename)}:{fr.lineno}"))
    return r


torch.empty = _timed_empty
for _ in range(5):
    step()
torch.cuda.synchronize()
torch.empty = _orig_empty
for s in slow:
    print("slow empty", s)
m0 = torch.cuda.memory_stats()
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    step()
torch.cuda.synchronize()
pr.disable()
m1 = torch.cuda.memory_stats()
for k in ("num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams"):
    print(k, m1.get(k, 0) - m0.get(k, 0))
import time  # noqa: E402

sizes = [(32768, torch.int16), (32768, torch.int32), (121632, torch.int32), (4435968, torch.int32),
         (191360 * 19, torch.float32), (24806, torch.int32), (69312, torch.int32)]
for nel, dt in sizes:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        x = torch.empty(nel, dtype=dt, device="cuda")
        del x
    t1 = time.perf_counter()
    print(f"empty({nel}, {dt}) {1e6 * (t1 - t0) / 100:.1f} us")
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
