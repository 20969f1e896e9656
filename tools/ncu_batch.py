"""Profile target: batch kernel, 4096 scenarios of the 123 shape, launch 2 of 2 (K sweeps each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 64
f = fg.make_feeder("123")
h = Lopf.setup_batch(f, fg.scenario_scales(f, 4096), precision=prec).bind("cuda")
h.run(K)
h.run(K)
torch.cuda.synchronize()
s = h.sizes
print("tasks", s.n_tasks, "slots", s.n_slots, "alg bytes", s.alg_bytes, "grid", s.grid)
