"""us/sweep at fixed K (test off) for the library in $LOPF_LIB (default: in-tree).
Usage: python tools/kern_time.py SHAPE KERNEL K   (SHAPE: 13 | 123 | 8500 | s<N>x<shape>)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

shape, kernel, K = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if shape.startswith("s"):
    n, sub = shape[1:].split("x")
    f = fg.make_stitched(int(n), sub)
else:
    f = fg.make_feeder(shape)
h = Lopf.setup(f, kernel=kernel).bind("cuda")
best = 1e9
for _ in range(4):
    h.reset()
    r = h.run(K)
    best = min(best, 1e3 * r.solve_ms / K)
s = h.sizes
print(f"{os.environ.get('LOPF_LIB', 'current')}: {shape} kernel {s.kernel} grid {s.grid} tasks {s.n_tasks} "
      f"slots {s.n_slots} best {best:.3f} us/sweep alg {s.alg_bytes / best / 1e3:.0f} GB/s", flush=True)
