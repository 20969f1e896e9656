"""Write tests/golden/lp_optimum.json: the optimum of the centralized LP (LP_model) of
the synthetic feeders of configs 1-3, by HiGHS on the ORACLE's assembly (oracle.lp_reference.highs), so
bench.py can report how far the paper's stopping criterion leaves the ADMM objective
from the LP optimum.  Calls only oracle/ and feedergen.  Usage: python tests/golden/make_lp_golden.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import feedergen as fg  # noqa: E402
import oracle  # noqa: E402
from oracle.lp_reference import highs  # noqa: E402

out = {"_note": "written by tests/golden/make_lp_golden.py: HiGHS optimum of oracle.assemble_lp", "configs": {}}
for shape in ("13", "123", "8500"):
    f = fg.make_feeder(shape)
    t = time.time()
    _, obj = highs(oracle.assemble_lp(f))
    out["configs"][shape] = dict(sha256=f.sha256(), objective=obj, seconds=round(time.time() - t, 2))
    print(shape, out["configs"][shape], flush=True)
with open(os.path.join(ROOT, "tests", "golden", "lp_optimum.json"), "w") as fh:
    json.dump(out, fh, indent=1)
