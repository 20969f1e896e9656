"""Debug: which copies are wrong after K sweeps (single launch vs 3 launches)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
import oracle  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

f = fg.make_feeder("123")
p = oracle.build_problem(f)
h = Lopf.setup(f, kernel=2).bind("cuda")
for K in (20, 50, 100, 300, 1000):
    r = oracle.run_k(p, K)
    for mode in ("single", "split"):
        h.reset()
        if mode == "single":
            h.run(K)
        else:
            h.run(1); h.run(K // 3); h.run(K - 1 - K // 3)
        x, xl, lam = h.get_state()
        el = np.abs(xl - r.x_loc)
        bad = np.nonzero(el > 1e-9 * max(1, np.abs(r.x_loc).max()))[0]
        gl = sorted(set(int(p.dec.copy_global[j]) for j in bad))
        print(f"K={K:5d} {mode:6s}: max xl err {el.max():.3e}, bad copies {len(bad)}, globals {gl[:12]} "
              f"nu {[int(p.dec.nu[g]) for g in gl[:12]]} vars {[p.lp.var[g] for g in gl[:4]]}", flush=True)
