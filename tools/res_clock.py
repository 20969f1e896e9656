"""Resident kernel: in-kernel cycles per sweep (diag profile) vs event-timed us per sweep -> implied SM clock."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

f = fg.make_feeder(sys.argv[1] if len(sys.argv) > 1 else "8500")
K = 3000
for skip in [int(a) for a in sys.argv[2:]] or (0, 134):
    h = Lopf.setup(f, kernel=2, diag_skip=skip, diag_profile=True).bind("cuda")
    h.reset()
    r = h.run(K)
    pr = h.get_profile()
    cyc = (pr[:, 0] + pr[:, 1]) / np.maximum(pr[:, 3], 1)
    us = 1e3 * r.solve_ms / K
    print(f"skip={skip}: {us:.3f} us/sweep, in-kernel {cyc.mean():.0f} cycles/sweep (work {np.mean(pr[:,0]/np.maximum(pr[:,3],1)):.0f}, "
          f"protocol {np.mean(pr[:,1]/np.maximum(pr[:,3],1)):.0f}) -> {cyc.mean() / us / 1e3:.2f} GHz", flush=True)
    h.destroy()
