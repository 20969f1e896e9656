"""Scenario batches (config 4) through the C-ABI on the GPU: every sampled scenario's iterate after a
fixed K matches the oracle run on that scenario's scaled feeder (1e-9 relative), and its iteration
count to (termination) is bit-exact."""
import os

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


def _oracle_solve(args):
    f, k = args
    o = oracle.solve(oracle.build_problem(fg.scale_loads(f, k)))
    return o.iters, o.objective


def test_full_4096_batch_sampled():
    """BASELINE configs[3] at full size in the bench's launch configuration: 4096 scenarios in one batch
    handle.  Iterates after a fixed K (1e-9 relative) on the first / middle / last scenario, and the
    iteration count to (termination) bit-exact and the objective within 1e-6 on 64 sampled scenarios
    (SURVEY §8(c) parity matrix, config 4) -- the oracle runs each sampled scenario alone, in a host
    process pool.  Then the two shards [0, 2048) and [2048, 4096) solved as separate batch handles (the
    scenario sharding of bench.py --config 4 at N = 2) give bit-identical per-scenario K, objective and
    iterate to the full batch: a lane depends on its own scenario only."""
    import multiprocessing as mp
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_09410_b200 import Lopf
    f = fg.make_feeder("123")
    K = fg.scenario_scales(f, 4096)
    h = Lopf.setup_batch(f, K).bind("cuda")
    h.run(60)
    for sc in (0, 2047, 4095):
        o = oracle.run_k(oracle.build_problem(fg.scale_loads(f, K[sc])), 60)
        x, xl, lam = h.get_state_scen(sc)
        assert _rel(x, o.x) <= TOL and _rel(xl, o.x_loc) <= TOL and _rel(lam, o.lam) <= TOL, sc
    h.reset()
    h.solve()
    r = h.get_batch_results()
    assert np.all(r["outcome"] == 0)
    samples = sorted(set(np.random.default_rng(64).choice(4096, 62, replace=False).tolist()) | {0, 4095})
    # spawn, not fork: a fork of this process (CUDA context, BLAS thread pool) can leave the parent's BLAS
    # deadlocked in a later linalg call
    with mp.get_context("spawn").Pool(min(len(samples), max(1, os.cpu_count() or 1))) as pool:
        ref = pool.map(_oracle_solve, [(f, K[sc]) for sc in samples])
    for sc, (k, obj) in zip(samples, ref):
        assert int(r["iters"][sc]) == k, (sc, int(r["iters"][sc]), k)
        assert abs(r["objective"][sc] - obj) <= 1e-6 * abs(obj), sc
    full_x = {sc: h.get_state_scen(sc) for sc in (5, 2047, 2048, 4090)}
    for lo, hi in ((0, 2048), (2048, 4096)):
        hs = Lopf.setup_batch(f, K[lo:hi]).bind("cuda")
        hs.solve()
        rs = hs.get_batch_results()
        assert np.array_equal(rs["iters"], r["iters"][lo:hi]) and np.array_equal(rs["objective"], r["objective"][lo:hi])
        for sc in full_x:
            if lo <= sc < hi:
                for a, b in zip(hs.get_state_scen(sc - lo), full_x[sc]):
                    assert np.array_equal(a, b), sc
        del hs


def test_small_fixture_batch():
    """A 1-phase chain (every subsystem small) through the batch kernel: iterates after a fixed K,
    across two launches, within 1e-9 of the oracle per scenario; a partial last group (37 scenarios)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import fixtures as fx
    from paper_2310_09410_b200 import Lopf
    f = fx.chain_1ph(24)
    K = fg.scenario_scales(f, 37)
    h = Lopf.setup_batch(f, K).bind("cuda")
    h.run(300)
    h.run(200)
    for sc in (0, 17, 36):
        o = oracle.run_k(oracle.build_problem(fg.scale_loads(f, K[sc])), 500)
        x, xl, lam = h.get_state_scen(sc)
        assert _rel(x, o.x) <= TOL and _rel(xl, o.x_loc) <= TOL and _rel(lam, o.lam) <= TOL, sc


def test_batch_handle_rejects_single_problem_state_calls(batch):
    """lopf_set_state / lopf_get_state act on one problem: on a batch handle they are LOPF_E_STATE
    (the per-scenario getters are lopf_get_state_scen)."""
    from paper_2310_09410_b200 import LopfError
    from paper_2310_09410_b200.lopf import STATUS
    f, K, h = batch
    nc = int(h.sizes.n_copies)
    with pytest.raises(LopfError) as e:
        h.set_state(np.zeros(nc), np.zeros(nc))
    assert STATUS[e.value.status] == "LOPF_E_STATE"
    with pytest.raises(LopfError) as e:
        h.get_state()
    assert STATUS[e.value.status] == "LOPF_E_STATE"


@pytest.mark.parametrize("precision", [64, 32])
def test_batch_repeat_bit_identical(precision):
    """Race stress for the team kernel: items are claimed dynamically, so which team and SM
    run an item changes from launch to launch; the team's SMEM hand-overs (d rows, the residual partials by
    bar.arrive / bar.sync) and the L2-parked v must still give the same bits.  512 scenarios, 400 sweeps
    run twice from reset (the second time as 150 + 250 across launches): every scenario's outcome,
    residuals and objective, and the iterate of sampled scenarios, are bit-identical."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_09410_b200 import Lopf
    f = fg.make_feeder("123")
    K = fg.scenario_scales(f, 512, seed=77)
    h = Lopf.setup_batch(f, K, eps_rel=1e-2, precision=precision).bind("cuda")
    h.run(400, test=True)
    r1 = h.get_batch_results()
    s1 = {sc: h.get_state_scen(sc) for sc in (0, 100, 511)}
    h.reset()
    h.run(150, test=True)
    h.run(250, test=True)
    r2 = h.get_batch_results()
    for key in ("outcome", "res", "objective"):
        assert np.array_equal(r1[key], r2[key]), key
    for sc, st in s1.items():
        for a, b in zip(h.get_state_scen(sc), st):
            assert np.array_equal(a, b), sc
