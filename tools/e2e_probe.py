import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, feedergen as fg
from paper_2310_09410_b200 import Lopf
f = fg.make_feeder("8500")
h = Lopf.setup(f).bind("cuda")
s = torch.cuda.Stream()
for _ in range(3): h.reset(); h.solve()
torch.cuda.synchronize()
for it in range(4):
    t0 = time.perf_counter(); h.bind("cuda", stream=s); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    h.solve_async(1000000, True, stream=s); t3 = time.perf_counter()
    r = h.result_get(stream=s); t4 = time.perf_counter()
    x = h.get_x(stream=s); t5 = time.perf_counter()
    print(f"bind call {1e3*(t1-t0):.3f} ms, bind complete {1e3*(t2-t0):.3f}, launch {1e3*(t3-t2):.3f}, solve wait {1e3*(t4-t3):.3f} (kernel {r.solve_ms:.3f}), get_x {1e3*(t5-t4):.3f}")
