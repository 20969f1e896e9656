"""Scenario batches (config 4) through the C-ABI on the GPU: every sampled scenario's iterate after a
fixed K matches the oracle run on that scenario's scaled feeder (1e-9 relative), and its iteration
count to (termination) is bit-exact."""
import numpy as np
import pytest

import feedergen as fg
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def batch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_09410_b200 import Lopf
    f = fg.make_feeder("123")
    K = fg.scenario_scales(f, 40)                  # two groups, the second one partial
    h = Lopf.setup_batch(f, K).bind("cuda")
    return f, K, h


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def test_fixed_k_per_scenario(batch):
    f, K, h = batch
    h.reset()
    h.run(150)
    h.run(50)                                      # continuation across launches
    r = h.get_batch_results()
    assert np.all(r["iters"] == 50) and np.all(r["outcome"] == 2)
    for sc in (0, 13, 31, 32, 39):
        p = oracle.build_problem(fg.scale_loads(f, K[sc]))
        o = oracle.run_k(p, 200)
        x, xl, lam = h.get_state_scen(sc)
        assert _rel(x, o.x) <= TOL and _rel(xl, o.x_loc) <= TOL and _rel(lam, o.lam) <= TOL, sc


def test_solve_to_tolerance_per_scenario(batch):
    f, K, h = batch
    h.reset()
    res = h.solve()
    r = h.get_batch_results()
    assert np.all(r["outcome"] == 0) and res.iters == r["iters"].max()
    for sc in (5, 38):
        p = oracle.build_problem(fg.scale_loads(f, K[sc]))
        o = oracle.solve(p)
        assert int(r["iters"][sc]) == o.iters, (sc, int(r["iters"][sc]), o.iters)
        assert abs(r["objective"][sc] - o.objective) <= 1e-6 * abs(o.objective)
        x, _, _ = h.get_state_scen(sc)
        assert np.all(x >= p.lp.lo) and np.all(x <= p.lp.hi)


def test_full_4096_batch_sampled():
    """BASELINE configs[3] at full size in the bench's launch configuration: 4096 scenarios in one batch
    handle; sampled scenarios (first, middle, last) against the oracle run on that scenario alone --
    iterates after a fixed K (1e-9 relative) and the iteration count to (termination), bit-exact."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_09410_b200 import Lopf
    f = fg.make_feeder("123")
    K = fg.scenario_scales(f, 4096)
    h = Lopf.setup_batch(f, K).bind("cuda")
    h.run(60)
    samples = (0, 2047, 4095)
    probs = {sc: oracle.build_problem(fg.scale_loads(f, K[sc])) for sc in samples}
    for sc in samples:
        o = oracle.run_k(probs[sc], 60)
        x, xl, lam = h.get_state_scen(sc)
        assert _rel(x, o.x) <= TOL and _rel(xl, o.x_loc) <= TOL and _rel(lam, o.lam) <= TOL, sc
    h.reset()
    h.solve()
    r = h.get_batch_results()
    assert np.all(r["outcome"] == 0)
    for sc in (0, 4095):
        o = oracle.solve(probs[sc])
        assert int(r["iters"][sc]) == o.iters, (sc, int(r["iters"][sc]), o.iters)


def test_staged_only_batch():
    """A feeder whose every operator block fits the SMEM stage (max n_s = 10: no kTaskDirect task) runs
    the batch kernel's staged-only instantiation (SRC 2, shared-space operator loads): iterates after a
    fixed K, across two launches, within 1e-9 of the oracle per scenario."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import fixtures as fx
    from paper_2310_09410_b200 import Lopf
    f = fx.chain_1ph(24)
    K = fg.scenario_scales(f, 37)
    h = Lopf.setup_batch(f, K).bind("cuda")
    assert h.sizes.max_ns * (h.sizes.max_ns + 3) // 2 <= 448      # triangle + b-bar fit one stage
    h.run(300)
    h.run(200)
    for sc in (0, 17, 36):
        o = oracle.run_k(oracle.build_problem(fg.scale_loads(f, K[sc])), 500)
        x, xl, lam = h.get_state_scen(sc)
        assert _rel(x, o.x) <= TOL and _rel(xl, o.x_loc) <= TOL and _rel(lam, o.lam) <= TOL, sc
