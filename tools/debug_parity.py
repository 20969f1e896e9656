"""Debug: per-sweep parity of a kernel vs the oracle; reports the worst global/copy."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
import oracle  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "123"
kernel = int(sys.argv[2]) if len(sys.argv) > 2 else 2
f = fg.make_feeder(shape)
p = oracle.build_problem(f)
h = Lopf.setup(f, kernel=kernel).bind("cuda")
print("grid", h.sizes.grid)
for k in (1, 2, 3, 5, 10):
    h.reset()
    h.run(k)
    x, xl, lam = h.get_state()
    r = oracle.run_k(p, k)
    ex = np.abs(x - r.x)
    el = np.abs(xl - r.x_loc)
    em = np.abs(lam - r.lam)
    i = int(np.argmax(ex)); j = int(np.argmax(el))
    print(f"k={k}: x err {ex.max():.3e} at global {i} {p.lp.var[i]} nu={p.dec.nu[i]} | x_loc err {el.max():.3e} at copy {j} "
          f"(global {p.dec.copy_global[j]}) | lam err {em.max():.3e}; #x>1e-12: {(ex > 1e-12).sum()}", flush=True)
