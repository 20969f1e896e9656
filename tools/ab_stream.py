"""A/B of streaming / batch builds ($LOPF_LIB): us/sweep at fixed K (test off) for
  batch  : 4096 scenarios of the 123 shape (config 4), 100 sweeps
  s8500  : 8500 shape, streaming kernel, fp64 and fp32, 2000 sweeps
  stitch : 16 x 8500 stitched feeder (a quarter of config 5), fp64 and fp32, 200 sweeps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

lib = os.path.basename(os.environ.get("LOPF_LIB", "current"))
which = sys.argv[1:] or ["batch", "s8500", "stitch"]


def best(h, k, reps=3):
    b = 1e9
    for _ in range(reps):
        h.reset()
        r = h.run(k)
        b = min(b, 1e3 * r.solve_ms / k)
    return b


if "batch" in which:
    f = fg.make_feeder("123")
    for prec in (64, 32):
        h = Lopf.setup_batch(f, fg.scenario_scales(f, 4096), precision=prec).bind("cuda")
        print(f"{lib} batch p{prec} tasks={h.sizes.n_tasks}: {best(h, 100, 2):.1f} us/batch-sweep", flush=True)
        h.destroy()
if "s8500" in which:
    f = fg.make_feeder("8500")
    for prec in (64, 32):
        h = Lopf.setup(f, kernel=1, precision=prec).bind("cuda")
        print(f"{lib} s8500 p{prec} tasks={h.sizes.n_tasks}: {best(h, 2000):.2f} us/sweep", flush=True)
        h.destroy()
if "stitch" in which:
    f = fg.make_stitched(16, "8500")
    for prec in (64, 32):
        h = Lopf.setup(f, kernel=1, precision=prec, max_iter=10_000).bind("cuda")
        us = best(h, 200)
        print(f"{lib} stitch16 p{prec} tasks={h.sizes.n_tasks}: {us:.1f} us/sweep "
              f"{h.sizes.alg_bytes / us / 1e3:.0f} GB/s alg", flush=True)
        h.destroy()
