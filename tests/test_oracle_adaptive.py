"""Pins of the residual-balancing oracle (reading F2) against the
fixed-rho oracle (itself pinned in test_oracle_admm.py / test_oracle_physics.py) and the LP optimum:
* adapt_every = 0 and a never-firing rule (mu = inf) are the fixed-rho Algorithm 1 bit for bit;
* a run whose rho changes once at sweep t0 equals the fixed-rho oracle with rho_0 for t0 sweeps, continued
  from that state with rho_1 (lambda is the unscaled multiplier of PAPER.md:284, so nothing is rescaled,
  and Abar_s, bbar_s are rho-free) -- this pins when the change takes effect and that
  nothing else changes with it;
* the change follows the balancing rule on that sweep's residuals (pres, dres of the fixed-rho run);
* at a tight tolerance the adaptive run reaches the LP optimum (HiGHS): rho does not move the fixed point."""
import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from oracle.admm import initial_state, _run


def test_no_adaptation_is_fixed_rho():
    p = oracle.build_problem(fg.make_feeder("13"))
    ref = oracle.solve(p)
    for every, mu in ((0, 10.0), (1, np.inf)):
        r, rho, n = oracle.solve_adaptive(p, every=every, mu=mu)
        assert (r.iters, rho, n) == (ref.iters, 100.0, 0)
        assert np.array_equal(r.x, ref.x) and np.array_equal(r.lam, ref.lam)


def test_single_change_is_a_restart_with_the_new_rho():
    f = fx.four_bus()
    p = oracle.build_problem(f)
    every = 25
    # the first sweep t0 (a multiple of `every`) at which the rule fires, from the fixed-rho trace
    tr = _run(p, *initial_state(p), 2000, False, trace_every=1).trace
    t0 = next(t for t in range(every, 2000, every) if tr[t - 1, 0] > 10 * tr[t - 1, 1] or tr[t - 1, 1] > 10 * tr[t - 1, 0])
    rho1 = 200.0 if tr[t0 - 1, 0] > 10 * tr[t0 - 1, 1] else 50.0
    # adaptive run for t0 + m sweeps (m < t0) with a rule that can fire only once (every = t0)
    m = min(40, t0 - 1)
    r, rho, n = oracle.solve_adaptive(p, every=t0, max_iter=t0 + m, test=False)
    assert n == 1 and rho == rho1
    # composition of two fixed-rho runs
    a = oracle.run_k(p, t0)
    q = oracle.build_problem(f, rho=rho1)
    b = oracle.run_k(q, m, state=(a.x_loc, a.lam))
    assert np.array_equal(r.x_loc, b.x_loc) and np.array_equal(r.lam, b.lam) and np.array_equal(r.x, b.x)


@pytest.mark.parametrize("make", [fx.four_bus, fx.physical, lambda: fx.chain_1ph(4)])
def test_adaptive_reaches_lp_optimum(make):
    from oracle.lp_reference import highs
    f = make()
    lp = oracle.assemble_lp(f)
    _, oh = highs(lp)
    r, rho, n = oracle.solve_adaptive(oracle.build_problem(f, lp=lp, eps_rel=1e-8), every=10, max_iter=2_000_000)
    assert r.converged and n > 0
    assert abs(r.objective - oh) <= 1e-6 * abs(oh)
