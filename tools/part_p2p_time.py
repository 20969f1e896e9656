"""Per-sweep time of the partitioned mode's device-initiated exchange against the plain
streaming kernel on the same feeder: fixed K sweeps (test off), CUDA events, best of 3.
  streaming            lopf_run on the whole feeder (one launch)
  p2p world 1          lopf_part_solve_p2p on a one-rank partition (the protocol with no peer)
  p2p emulated world W lopf_part_emulate: W ranks in one cooperative launch on this GPU (each rank gets
                       148 / W SMs, so this measures protocol cost, not multi-GPU speed-up)
Usage: python tools/part_p2p_time.py [n_sub] [K] [W ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

n_sub = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
worlds = [int(a) for a in sys.argv[3:]] or [2]
f = fg.make_stitched(n_sub, "8500") if n_sub > 1 else fg.make_feeder("8500")


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return 1e3 * best / K


s = Lopf.setup(f, kernel=1).bind("cuda")
s.run(50)
print(f"{f.name}: streaming {timed(lambda: (s.reset(), s.solve_async(K, False))):.2f} us/sweep", flush=True)
h = Lopf.setup_part(f, 0, 1).bind("cuda")
h.reset()
h.part_solve_p2p(50, False)
print(f"{f.name}: p2p world 1 {timed(lambda: (h.reset(), h.part_solve_p2p(K, False))):.2f} us/sweep", flush=True)
for W in worlds:
    own = fg.stitched_bus_owner(f, W) if n_sub > 1 and n_sub % W == 0 else None
    hs = [Lopf.setup_part(f, r, W, bus_owner=own).bind("cuda") for r in range(W)]

    def run():
        for x in hs:
            x.reset()
        Lopf.part_emulate(hs, K, test=False)
    run()
    print(f"{f.name}: p2p emulated world {W} {timed(run):.2f} us/sweep", flush=True)
