"""A/B of resident-kernel builds: us/sweep at fixed K (test off), best of 5, several shapes.
Usage: python tools/res_ab.py LIB1.so [LIB2.so ...]  (each in a fresh process via LOPF_LIB)"""
import os
import subprocess
import sys

code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import feedergen as fg
from paper_2310_09410_b200 import Lopf
for shape, K in (("8500", 3000), ("123", 3000)):
    h = Lopf.setup(fg.make_feeder(shape), kernel=2).bind("cuda")
    best = 1e9
    for _ in range(5):
        h.reset()
        best = min(best, 1e3 * h.run(K).solve_ms / K)
    print(f"{os.environ['LOPF_LIB']}: {shape} G={h.sizes.grid} {best:.3f} us/sweep", flush=True)
'''
for lib in sys.argv[1:]:
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LOPF_LIB=lib))
