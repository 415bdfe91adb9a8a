"""Bin-density sweep of BASELINE.json's C3 configuration (bunny-scale bumpy
sphere, 69 936 triangles, 16^3 root, d = 0.05, 4 levels) over the paper's B
values, writing the reference's sweep CSV (GPU box helper).

    python tools/sweep_c3.py [out.csv]
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2502_16310_b200 as ow  # noqa: E402
from paper_2502_16310_b200 import report  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep_c3.csv"
cfg = bench.CONFIGS["C3"]
geom = ow.import_stl_bytes(bench.make_input(cfg))
dom = ow.Aabb(np.zeros(3), np.ones(3))
bs = [1, 2, 4, 6, 7, 8, 9, 10, 12, 14, 16]
report.sweep(geom, dom, (16, 16, 16), cfg["d"], cfg["levels"], bs, verbose=False)  # warm-up pass
rows = report.sweep(geom, dom, (16, 16, 16), cfg["d"], cfg["levels"], bs, out_csv=out)
print(open(out).read())
