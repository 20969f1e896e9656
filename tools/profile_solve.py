"""Profiling driver: set up one feeder, bind, run `--solves` solves of the chosen kernel.
Used under ncu (`-k regex:admm_ -s <warmup launches> -c 1`); prints the result of each solve."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="8500")
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--iters", type=int, default=0, help="fixed sweeps per launch (0 = solve to tolerance)")
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()
h = Lopf.setup(fg.make_feeder(a.shape), kernel=a.kernel, precision=a.precision).bind("cuda")
for i in range(a.solves):
    h.reset()
    r = h.run(a.iters, test=False) if a.iters else h.solve()
    print(f"solve {i}: kernel={h.sizes.kernel} grid={h.sizes.grid} K={r.iters} ms={r.solve_ms:.3f} "
          f"us/sweep={1e3 * r.solve_ms / max(r.iters, 1):.3f}", flush=True)
