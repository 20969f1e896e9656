"""Write tests/golden/oracle_golden.json: the ORACLE's iteration count to (termination),
objective and final residuals for configs 1-3 at the paper's defaults, plus two small
instances of the config-5 stitched family (feedergen.make_stitched: 4 x 13-shaped, 2 x 8500-shaped).
Calls only oracle/ and feedergen (no CUDA path); re-run after any change to either.
Usage: python tests/golden/make_oracle_golden.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import feedergen as fg  # noqa: E402
import oracle  # noqa: E402

out = {"_note": "written by tests/golden/make_oracle_golden.py from oracle/ only", "configs": {}}
CASES = {"13": lambda: fg.make_feeder("13"), "37": lambda: fg.make_feeder("37"), "123": lambda: fg.make_feeder("123"),
         "8500": lambda: fg.make_feeder("8500"), "s4x13": lambda: fg.make_stitched(4, "13"),
         "s2x8500": lambda: fg.make_stitched(2, "8500")}
for shape, make in CASES.items():
    f = make()
    t = time.time()
    p = oracle.build_problem(f, rho=100.0, eps_rel=1e-3)
    r = oracle.solve(p, max_iter=1_000_000)
    out["configs"][shape] = dict(sha256=f.sha256(), S=p.dec.S, n=p.lp.n, m=p.lp.m, n_copies=p.dec.n_copies,
                                 converged=r.converged, iters=r.iters, objective=r.objective, pres=r.pres,
                                 dres=r.dres, eps_prim=r.eps_prim, eps_dual=r.eps_dual,
                                 oracle_seconds=round(time.time() - t, 2))
    print(shape, out["configs"][shape], flush=True)
with open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json"), "w") as fh:
    json.dump(out, fh, indent=1)
