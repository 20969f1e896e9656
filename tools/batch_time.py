"""Timing of the batch kernel: fixed K sweeps for n_scen scenarios of the 123-shaped feeder."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

n_scen = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 200
f = fg.make_feeder("123")
t = time.time()
h = Lopf.setup_batch(f, fg.scenario_scales(f, n_scen)).bind("cuda")
print(f"setup+bind {time.time() - t:.2f}s, arena {h.sizes.device_bytes / 1e6:.0f} MB", flush=True)
for _ in range(2):
    h.reset()
    r = h.run(k)
print(f"{n_scen} scenarios x {k} sweeps: {r.solve_ms:.2f} ms -> {1e3 * r.solve_ms / k:.1f} us per batch sweep, "
      f"{n_scen * k / (r.solve_ms / 1e3) / 1e6:.2f} M scenario-sweeps/s", flush=True)
