"""Diagnostics: per-phase cycles of the resident kernel (G-phase, L-phase, grid barrier) on a shape,
plus sweep time with phases switched off (barrier-only = the synchronisation floor)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="8500")
ap.add_argument("--iters", type=int, default=2000)
ap.add_argument("--max-ctas", type=int, default=0)
a = ap.parse_args()
f = fg.make_feeder(a.shape)
for skip, label in ((0, "full sweep"), (2, "sync only (no update work)")):
    h = Lopf.setup(f, kernel=2, diag_profile=True, diag_skip=skip, max_ctas=a.max_ctas).bind("cuda")
    for _ in range(2):
        h.reset()
        r = h.run(a.iters)
    pr = h.get_profile()
    us = 1e3 * r.solve_ms / a.iters
    cyc = pr[:, 0:2] / np.maximum(pr[:, 3:4], 1)
    print(f"{label:26s} G={h.sizes.grid:3d} {us:7.3f} us/sweep (instrumented) | cycles/sweep [work, publish+wait] "
          f"mean {cyc.mean(0).round(0)} max {cyc.max(0).round(0)}", flush=True)
