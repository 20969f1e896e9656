"""Debug: after which launch of a split sequence does the state go wrong?"""
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
for trial in range(30):
    seq = [1, 2, 5, 3, 7, 1, 1, 4]
    h.reset()
    done = 0
    msg = []
    for k in seq:
        h.run(k)
        done += k
        _, xl, lam = h.get_state()
        e = np.abs(xl - ref(done).x_loc).max()
        msg.append(f"{done}:{e:.0e}")
        if e > 1e-9:
            break
    print(f"trial {trial}: " + " ".join(msg), flush=True)
