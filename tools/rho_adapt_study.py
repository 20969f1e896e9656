"""Residual balancing (reading F2) vs the paper's fixed rho = 100 on the synthetic feeders, on the
GPU (streaming kernel): iterations to the paper's stopping criterion, the objective and its gap to the LP
optimum (tests/golden/lp_optimum.json).  Writes profiles/r02_rho_adapt.json.  Usage: python tools/rho_adapt_study.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

lp = json.load(open(os.path.join(ROOT, "tests", "golden", "lp_optimum.json")))["configs"]
out = {"_note": "written by tools/rho_adapt_study.py (GPU, streaming kernel, rho0 = 100, eps_rel = 1e-3, mu = 10, "
                "tau = 2)", "runs": []}
for shape in ("13", "123", "8500"):
    f = fg.make_feeder(shape)
    opt = lp[shape]["objective"]
    for every in (0, 1, 10, 100):
        h = Lopf.setup(f, kernel=1, adapt_every=every, max_iter=400_000).bind("cuda")
        r = h.solve()
        rho, n = h.get_rho()
        row = dict(shape=shape, adapt_every=every, outcome=int(r.outcome), iters=int(r.iters), objective=r.objective,
                   gap_vs_lp=(r.objective - opt) / abs(opt), rho_final=rho, rho_changes=n, solve_ms=r.solve_ms)
        print(json.dumps(row), flush=True)
        out["runs"].append(row)
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_rho_adapt.json"), "w"), indent=1)
