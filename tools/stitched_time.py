"""Config 5 on one GPU: the 64 x 8500 stitched feeder through the streaming kernel.
Prints setup time, us/sweep at fixed K (test off), algorithmic GB/s, and time-to-tolerance.
Usage: python tools/stitched_time.py [n_sub] [K]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

n_sub = int(sys.argv[1]) if len(sys.argv) > 1 else 64
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
t = time.time()
f = fg.make_stitched(n_sub, "8500")
t_gen = time.time() - t
t = time.time()
h = Lopf.setup(f, max_iter=50_000)
t_setup = time.time() - t
h.bind("cuda")
s = h.sizes
out = dict(n_sub=n_sub, gen_s=round(t_gen, 1), setup_s=round(t_setup, 1), S=s.S, n=s.n, n_copies=s.n_copies,
           kernel=s.kernel, grid=s.grid, alg_bytes=s.alg_bytes, device_bytes=s.device_bytes)
h.run(5)
torch.cuda.synchronize()
times = []
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h.run(K)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
ms = min(times)
out.update(K=K, ms=[round(x, 3) for x in times], us_per_sweep=round(1e3 * ms / K, 2),
           alg_gbs=round(s.alg_bytes * K / (ms * 1e-3) / 1e9, 1))
h.reset()
r = h.solve()
out.update(solve_iters=r.iters, solve_outcome=r.outcome, solve_ms=round(r.solve_ms, 2), objective=r.objective)
print(json.dumps(out), flush=True)
