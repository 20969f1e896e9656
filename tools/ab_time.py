"""A/B: us/sweep of the resident kernel for the library in $LOPF_LIB (fixed K, no diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "8500"
mixed = len(sys.argv) > 2 and sys.argv[2] == "mixed"
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 64
h = Lopf.setup(fg.make_feeder(shape), kernel=2, precision=prec)
if mixed:
    h.destroy()
    from paper_2310_09410_b200.lopf import Options  # noqa: F401
    import ctypes as C
    from paper_2310_09410_b200 import lopf as L
    o = L.Options(); L.load_library().lopf_options_default(C.byref(o)); o.kernel = 2; o.reserved[2] = 1
    net, keep = L._network(fg.make_feeder(shape)); hh = C.c_void_p()
    L._check(L.load_library().lopf_setup(C.byref(net), C.byref(o), C.byref(hh)), "setup")
    h = Lopf(hh.value, o)
h.bind("cuda")
best = 1e9
for _ in range(5):
    h.reset()
    r = h.run(3000)
    best = min(best, 1e3 * r.solve_ms / 3000)
print(f"{os.environ.get('LOPF_LIB', 'current')}{' mixed' if mixed else ''}: {shape} p{prec} G={h.sizes.grid} best {best:.3f} us/sweep", flush=True)
