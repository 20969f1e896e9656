"""Debug: first sweep of the streaming kernel vs the oracle on a small feeder; prints mismatching copies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import feedergen as fg  # noqa: E402
import oracle  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

f = fg.make_feeder(sys.argv[1] if len(sys.argv) > 1 else "13")
p = oracle.build_problem(f)
h = Lopf.setup(f, kernel=1).bind("cuda")
print("tasks", h.sizes.n_tasks, "slots", h.sizes.n_slots, "grid", h.sizes.grid, "block", h.sizes.block)
for k in (1, 2):
    h.run(1)
    ref = oracle.run_k(p, k)
    x, xl, lam = h.get_state()
    d = h.get_decomposition()
    sub_of_copy = np.repeat(np.arange(len(d.n_s)), d.n_s)
    for name, a, b in (("x", x, ref.x), ("xl", xl, ref.x_loc), ("lam", lam, ref.lam)):
        bad = np.nonzero(np.abs(a - b) > 1e-9 * max(1, np.abs(b).max()))[0]
        print(k, name, "bad", len(bad), "of", len(a))
        for i in bad[:8]:
            extra = f" sub {sub_of_copy[i]} n_s {d.n_s[sub_of_copy[i]]} kind {d.kind[sub_of_copy[i]]}" if name != "x" else ""
            print("   ", i, a[i], b[i], extra)
