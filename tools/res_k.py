"""Resident kernel: event time for several K at one diag setting -> per-sweep slope and fixed overhead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

f = fg.make_feeder(sys.argv[1])
skip = int(sys.argv[2])
h = Lopf.setup(f, kernel=2, diag_skip=skip).bind("cuda")
for _ in range(3):
    h.reset(); h.run(3000)
res = {}
for K in (100, 1000, 10000):
    best = 1e9
    for _ in range(3):
        h.reset()
        best = min(best, h.run(K).solve_ms)
    res[K] = best
slope = (res[10000] - res[1000]) / 9000 * 1e3
print(f"{sys.argv[1]} skip={skip}: ms {res}  slope {slope:.3f} us/sweep  fixed {res[1000] - slope * 1000 / 1e3:.3f} ms", flush=True)
