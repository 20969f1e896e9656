"""Debug: continued launches (run(k1) then run(k2)) vs the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
import oracle  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "123"
f = fg.make_feeder(shape)
p = oracle.build_problem(f)
h = Lopf.setup(f, kernel=2).bind("cuda")
for seq in ((1, 1), (1, 9), (2, 3), (5, 5), (1, 1, 1, 1)):
    h.reset()
    for k in seq:
        h.run(k)
    x, xl, lam = h.get_state()
    r = oracle.run_k(p, sum(seq))
    ex = np.abs(x - r.x); el = np.abs(xl - r.x_loc)
    i = int(np.argmax(ex)); j = int(np.argmax(el))
    print(f"{seq}: x err {ex.max():.3e} at {i} {p.lp.var[i]} nu={p.dec.nu[i]} | xl err {el.max():.3e} at copy {j} "
          f"global {p.dec.copy_global[j]} nu={p.dec.nu[p.dec.copy_global[j]]}; #bad copies {(el > 1e-12).sum()}", flush=True)
