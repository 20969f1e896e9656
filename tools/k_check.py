"""K (iterations to tolerance) of the resident kernel for the library in $LOPF_LIB vs the oracle goldens."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

G = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                "oracle_golden.json")))["configs"]
for key in ("13", "123", "8500", "s4x13"):
    f = fg.make_stitched(4, "13") if key == "s4x13" else fg.make_feeder(key)
    r = Lopf.setup(f, kernel=2).bind("cuda").solve()
    print(os.environ.get("LOPF_LIB", "current"), key, r.iters, G[key]["iters"], "OK" if r.iters == G[key]["iters"] else "MISMATCH",
          flush=True)
