"""Timing of the batch kernel: fixed K sweeps for n_scen scenarios of the 123-shaped feeder (A/B tool:
LOPF_LIB selects the build).  Prints the median of `reps` launches and the SM clock during the run."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

n_scen = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
shape = sys.argv[4] if len(sys.argv) > 4 else "123"
prec = int(sys.argv[5]) if len(sys.argv) > 5 else 64
f = fg.make_feeder(shape)
t = time.time()
h = Lopf.setup_batch(f, fg.scenario_scales(f, n_scen), precision=prec).bind("cuda")
print(f"setup+bind {time.time() - t:.2f}s, arena {h.sizes.device_bytes / 1e6:.0f} MB, grid {h.sizes.grid} x {h.sizes.block}",
      flush=True)
h.reset()
h.run(k)
ms = []
for _ in range(reps):
    h.reset()
    ms.append(h.run(k).solve_ms)
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"], capture_output=True,
                     text=True).stdout.strip()
ms.sort()
m = ms[len(ms) // 2]
print(f"{os.environ.get('LOPF_LIB', 'current')} p{prec} {n_scen} scenarios x {k} sweeps: {m:.2f} ms (min {ms[0]:.2f}) -> {1e3 * m / k:.1f} us per batch sweep, "
      f"{n_scen * k / (m / 1e3) / 1e6:.2f} M scenario-sweeps/s, sm clock {clk} MHz", flush=True)
