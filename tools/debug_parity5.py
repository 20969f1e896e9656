"""Debug: split sequences with longer second launches."""
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
refs = {}
def ref(k):
    if k not in refs:
        refs[k] = oracle.run_k(p, k)
    return refs[k]
for seq in ([16], [1, 16], [2, 16], [1, 40], [3, 40], [0, 40], [1, 1, 40], [10, 40], [40, 40], [1, 100]):
    fails = 0
    for trial in range(10):
        h.reset()
        for k in seq:
            h.run(k)
        _, xl, _ = h.get_state()
        fails += np.abs(xl - ref(sum(seq)).x_loc).max() > 1e-9
    print(seq, "fails", fails, "/ 10", flush=True)
