"""Stress: repeated fixed-K runs of the resident kernel vs the oracle (catches rare races)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
import oracle  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

shape, reps, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
f = fg.make_feeder(shape)
p = oracle.build_problem(f)
r = oracle.run_k(p, k)
h = Lopf.setup(f, kernel=2).bind("cuda")
bad = 0
for i in range(reps):
    h.reset()
    for part in (1, k // 3, k - 1 - k // 3):
        h.run(part)
    x, xl, lam = h.get_state()
    e = max(np.abs(x - r.x).max(), np.abs(xl - r.x_loc).max(), np.abs(lam - r.lam).max() / max(1, np.abs(r.lam).max()))
    bad += e > 1e-9
print(f"{shape}: {reps} repetitions of K={k} in 3 launches: {bad} outside 1e-9", flush=True)
