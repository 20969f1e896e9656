"""Profile target: the 64 x 8500 stitched instance, one warm-up launch then one launch of K sweeps
(streaming kernel).  Usage under ncu: ncu -k admm_stream_kernel --launch-skip 1 -c 1 python tools/ncu_stitched.py [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 64
h = Lopf.setup(fg.make_stitched(64, "8500"), kernel=1, precision=prec).bind("cuda")
h.run(K)
h.run(K)
torch.cuda.synchronize()
print("done", h.sizes.alg_bytes)
