"""Per-warp event timeline of one CTA (G/2) over sweeps 500-502 of the resident kernel, from the
LOPF_RES_TIMELINE diagnostics build (set LOPF_LIB).  Events: 0 loop top, 1 work/decision done,
2 warp sums stored, 3 after [A], 4 flag published (warp 0), 5 neighbour flags seen, 6 after fence, 7 after [B]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

h = Lopf.setup(fg.make_feeder(sys.argv[1] if len(sys.argv) > 1 else "8500"), kernel=2, diag_profile=True).bind("cuda")
h.run(600)
h.reset()
h.run(600)
pr = h.get_profile().reshape(-1)
W = h.sizes.block // 32
ev = pr[: 3 * W * 8].reshape(3, W, 8).astype(np.int64)
for sw in range(3):
    e = ev[sw]
    t0 = e[:, 0][e[:, 0] > 0].min()
    print(f"sweep {500 + sw}: (cycles from the earliest loop top)")
    for w in range(W):
        row = ["%6d" % (x - t0) if x > 0 else "     -" for x in e[w]]
        print(f"  warp {w:2d}: " + " ".join(row))
