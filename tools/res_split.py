"""Resident kernel on the 8500 shape: us/sweep with and without the update work (diag_skip=2 keeps only
the exchange / flags / reducer protocol).  Usage: python tools/res_split.py [shape]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

f = fg.make_feeder(sys.argv[1] if len(sys.argv) > 1 else "8500")
for skip in [int(a) for a in sys.argv[2:]] or (0, 2, 4, 6):
    h = Lopf.setup(f, kernel=2, diag_skip=skip).bind("cuda")
    best = 1e9
    for _ in range(4):
        h.reset()
        r = h.run(3000)
        best = min(best, 1e3 * r.solve_ms / 3000)
    print(f"skip={skip}: G={h.sizes.grid} {best:.3f} us/sweep", flush=True)
    h.destroy()
