"""Profile target: resident kernel on the 8500 shape, K sweeps (launch 2 of 2 is the one to capture)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
h = Lopf.setup(fg.make_feeder("8500"), kernel=2).bind("cuda")
h.run(K)
h.run(K)
torch.cuda.synchronize()
print("done")
