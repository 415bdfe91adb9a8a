"""cProfile of GridPlan.run(host=True, defer=True) in steady state (GPU box
helper): where the Python time around the native call goes.
    python tools/profile_run_py.py [C2]"""

import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = bench.CONFIGS[name]
data = bench.make_input(cfg)
n = int.from_bytes(data[80:84], "little")
rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
dim = cfg["dim"]
dom = ow.Aabb(np.zeros(dim), np.ones(dim))
params = ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"])
plans = [pipeline.GridPlan(dom, (cfg["root"],) * dim, params, cfg["lattice"], reuse_outputs=True, stage_times=False)
         for _ in range(2)]
for k in range(6):
    plans[k % 2].run(rec, n, host=True, defer=True).wait()
pr = cProfile.Profile()
pr.enable()
for k in range(200):
    g = plans[k % 2].run(rec, n, host=True, defer=True)
    g.wait()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
