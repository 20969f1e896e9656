"""Pins of the oracle closed forms and of Algorithm 1 (§III) against brute force:
KKT solves, grid search, projector identities, hand examples from SPEC.md, invariants, and the
centralized LP optimum by vertex enumeration / HiGHS (SURVEY §8(c) pin table)."""
import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from oracle.admm import initial_state, problem_from_parts
from oracle.lp_reference import highs, kkt_check, vertex_enumeration
from oracle.precompute import InfeasibleSubsystem, precompute, row_rank_reduce


# ---------------------------------------------------------------- precompute (closed_2 operators)
def test_precompute_spec_example():
    # A = [1 1], b = 2 -> Abar = [[-1/2, 1/2], [1/2, -1/2]], bbar = (1, 1)
    Ab, bb = precompute(np.array([[1.0, 1.0]]), np.array([2.0]))
    assert np.allclose(Ab, [[-0.5, 0.5], [0.5, -0.5]], atol=1e-15) and np.allclose(bb, [1, 1], atol=1e-15)
    # A = I -> Abar = 0, bbar = b
    Ab, bb = precompute(np.eye(3), np.array([1.0, 2.0, 3.0]))
    assert np.abs(Ab).max() < 1e-15 and np.allclose(bb, [1, 2, 3])


def _random_subsystem(rng):
    n = int(rng.integers(4, 58))
    m = int(rng.integers(1, min(n - 1, 42) + 1))
    return rng.normal(size=(m, n)), rng.normal(size=m)


def test_projector_identities():
    """A Abar = 0, A bbar = b, Abar^2 = -Abar, Abar = Abar^T, Abar bbar = 0."""
    rng = np.random.default_rng(1)
    for _ in range(100):
        A, b = _random_subsystem(rng)
        Ab, bb = precompute(A, b)
        assert np.abs(A @ Ab).max() < 1e-9
        assert np.abs(A @ bb - b).max() < 1e-9
        assert np.abs(Ab @ Ab + Ab).max() < 1e-9
        assert np.abs(Ab - Ab.T).max() < 1e-9
        assert np.abs(Ab @ bb).max() < 1e-9


def test_local_update_matches_kkt():
    """closed_2 = the solution of the KKT system [rho I A^T; A 0][x; mu] = [-d; b]
    of the equality QP, on 100 random subsystems of Table IV sizes."""
    rng = np.random.default_rng(2)
    rho = 100.0
    for _ in range(100):
        A, b = _random_subsystem(rng)
        m, n = A.shape
        prob = problem_from_parts([A], [b], [list(range(n))], np.zeros(n), -np.inf * np.ones(n),
                                  np.inf * np.ones(n), rho=rho)
        x = rng.normal(size=n)
        lam = rng.normal(size=n)
        xl = prob.local_update(x, lam)
        d = -rho * x - lam
        K = np.block([[rho * np.eye(n), A.T], [A, np.zeros((m, m))]])
        sol = np.linalg.solve(K, np.concatenate([-d, b]))
        assert np.abs(xl - sol[:n]).max() <= 1e-8 * max(1.0, np.abs(sol[:n]).max())


def test_local_update_spec_examples():
    # A = [1 1], b = 2, rho = 1, lambda = 0, B x = (1, 1) -> x_s = (1, 1)
    p = problem_from_parts([np.array([[1.0, 1.0]])], [np.array([2.0])], [[0, 1]], np.zeros(2), -np.inf * np.ones(2),
                           np.inf * np.ones(2), rho=1.0)
    assert np.allclose(p.local_update(np.array([1.0, 1.0]), np.zeros(2)), [1, 1], atol=1e-15)
    # lambda = 0 and A(Bx) = b already -> x_s = Bx
    assert np.allclose(p.local_update(np.array([0.5, 1.5]), np.zeros(2)), [0.5, 1.5], atol=1e-15)
    # m_s = 0 -> x_s = Bx + lambda/rho
    q = problem_from_parts([np.zeros((0, 2))], [np.zeros(0)], [[0, 1]], np.zeros(2), -np.inf * np.ones(2),
                           np.inf * np.ones(2), rho=4.0)
    assert np.allclose(q.local_update(np.array([1.0, 2.0]), np.array([4.0, -8.0])), [2.0, 0.0])


def test_row_rank_reduce():
    A = np.array([[1.0, 2.0, 0.0], [1.0, 2.0, 0.0], [0.0, 1.0, 1.0]])
    Ar, br, keep = row_rank_reduce(A, np.array([1.0, 1.0, 2.0]))
    assert keep == [0, 2]                                          # duplicate removed
    rng = np.random.default_rng(4)
    B = rng.normal(size=(3, 4))
    A = rng.normal(size=(6, 3)) @ B                                # rank 3, 6 x 4
    xs = rng.normal(size=4)
    Ar, br, _ = row_rank_reduce(A, A @ xs)
    assert Ar.shape == (3, 4)
    x_ls = np.linalg.lstsq(Ar, br, rcond=None)[0]
    assert np.abs(A @ x_ls - A @ xs).max() < 1e-8
    with pytest.raises(InfeasibleSubsystem):
        row_rank_reduce(np.array([[1.0, 1.0], [2.0, 2.0]]), np.array([1.0, 3.0]))
    # reduced rows give the same projection as the full set
    Ab1, bb1 = precompute(A, A @ xs)
    Ab2, bb2 = precompute(Ar, br, reduce=False)
    assert np.abs(Ab1 - Ab2).max() < 1e-9 and np.abs(bb1 - bb2).max() < 1e-9


@pytest.mark.parametrize("shape", ["13", "123"])
def test_feeder_subsystems_full_row_rank(shape):
    """The paper's assumption holds for every subsystem of the synthetic shapes."""
    f = fg.make_feeder(shape)
    d = oracle.decompose(f, oracle.assemble_lp(f))
    for s in range(d.S):
        assert np.linalg.matrix_rank(d.A[s]) == d.A[s].shape[0]


# ---------------------------------------------------------------- global update (closed_1, rho restored)
def _scalar_problem(ts, lams, c, lo, hi, rho):
    """One global variable owned by len(ts) single-variable subsystems with no local rows."""
    k = len(ts)
    return problem_from_parts([np.zeros((0, 1))] * k, [np.zeros(0)] * k, [[0]] * k, np.array([c]), np.array([lo]),
                              np.array([hi]), rho=rho)


def test_global_update_spec_examples():
    # c = 0, lambda = 0, one owner at 5 in [0, 10] -> 5; owner at -3 -> 0
    p = _scalar_problem([5.0], [0.0], 0.0, 0.0, 10.0, 100.0)
    assert p.global_update(np.array([5.0]), np.zeros(1))[0] == 5.0
    assert p.global_update(np.array([-3.0]), np.zeros(1))[0] == 0.0


def test_global_update_grid_search():
    """closed_1 with the rho restored (reading C1) = argmin over a dense grid of the 1-D problem
    of PAPER.md:300: (c + sum lam) x + rho/2 sum (x - t_k)^2 on [lo, hi]."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        nu = int(rng.integers(1, 5))
        rho = float(rng.choice([1.0, 10.0, 100.0]))
        t = rng.uniform(-1, 1, size=nu)
        lam = rng.uniform(-50, 50, size=nu)
        c = float(rng.uniform(-2, 2))
        lo, hi = -1.0, 1.0
        p = _scalar_problem(t, lam, c, lo, hi, rho)
        x = p.global_update(t.copy(), lam.copy())[0]
        grid = np.linspace(lo, hi, 2_000_001)
        obj = (c + lam.sum()) * grid + 0.5 * rho * ((grid[:, None] - t[None, :]) ** 2).sum(axis=1)
        assert abs(x - grid[np.argmin(obj)]) <= 2e-6
        assert lo <= x <= hi


def test_global_update_infinite_bounds_are_no_clamp():
    p = _scalar_problem([0.0, 0.0], [0, 0], 0.0, -np.inf, np.inf, 100.0)
    assert p.global_update(np.array([1e6, 3e6]), np.zeros(2))[0] == 2e6


# ---------------------------------------------------------------- dual update and residuals
def test_dual_update_spec():
    # lambda = 0, rho = 100, gap 0.01 on one coordinate -> that lambda becomes 1
    p = problem_from_parts([np.zeros((0, 2))], [np.zeros(0)], [[0, 1]], np.zeros(2), -np.inf * np.ones(2),
                           np.inf * np.ones(2), rho=100.0)
    lam = p.dual_update(np.array([0.5, 0.25]), np.array([0.49, 0.25]), np.zeros(2))
    assert lam[0] == pytest.approx(1.0, abs=1e-12) and lam[1] == 0.0
    # consensus -> unchanged
    assert np.array_equal(p.dual_update(np.array([0.5, 0.25]), np.array([0.5, 0.25]), np.array([3.0, -2.0])), [3, -2])


def test_residuals_spec_example():
    # B = I, x = (1, 0), x_s = (0, 0), prev = (0, 0), rho = 100 -> pres 1, dres 0, eps_prim eps_rel * 1
    p = problem_from_parts([np.zeros((0, 2))], [np.zeros(0)], [[0, 1]], np.zeros(2), -np.inf * np.ones(2),
                           np.inf * np.ones(2), rho=100.0, eps_rel=1e-3)
    pres, dres, ep, ed = p.residuals(np.array([1.0, 0.0]), np.zeros(2), np.zeros(2), np.zeros(2))
    assert (pres, dres, ep, ed) == (1.0, 0.0, 1e-3, 0.0)
    # consensus and stationary -> pres = dres = 0
    pres, dres, _, _ = p.residuals(np.array([0.3, 0.7]), np.array([0.3, 0.7]), np.array([0.3, 0.7]), np.zeros(2))
    assert pres == 0.0 and dres == 0.0


def test_termination_is_a_conjunction():
    """(termination) fires only when BOTH tests pass."""
    f = fx.chain_1ph(3)
    p = oracle.build_problem(f, eps_rel=1e-3)
    r = oracle.solve(p, max_iter=100000, trace_every=1)
    tr = r.trace
    ok = (tr[:, 0] <= tr[:, 2]) & (tr[:, 1] <= tr[:, 3])
    assert r.converged and ok[-1] and not ok[:-1].any()
    assert ((tr[:, 0] <= tr[:, 2]) ^ (tr[:, 1] <= tr[:, 3])).any()    # one test alone passed earlier


def test_max_iter_zero_returns_initial_state():
    p = oracle.build_problem(fx.four_bus())
    xl0, lam0 = initial_state(p)
    r = oracle.run_k(p, 0)
    assert r.iters == 0 and np.array_equal(r.x_loc, xl0) and np.array_equal(r.lam, lam0)


def test_initial_point_rule():
    """lambda = 0; x_s = 1 for voltages, midpoint if bounded, 0 if unbounded."""
    p = oracle.build_problem(fx.four_bus())
    xl, lam = initial_state(p)
    assert not lam.any()
    for k in range(p.nc):
        g = int(p.dec.copy_global[k])
        role = p.lp.var[g][0]
        if role == "w":
            assert xl[k] == 1.0
        elif role in ("pb", "qb", "pd", "qd"):
            assert xl[k] == 0.0
        else:
            assert xl[k] == 0.5 * (p.lp.lo[g] + p.lp.hi[g])


# ---------------------------------------------------------------- invariants along the iteration
def test_iteration_invariants():
    """After every sweep: lo <= x <= hi exactly; A_s x_s = b_s; Abar_s lambda_s = 0 (lambda_s in
    range(A_s^T), a consequence of closed_2 + ADMM-3)."""
    f = fg.make_feeder("13")
    p = oracle.build_problem(f)
    xl, lam = initial_state(p)
    d = p.dec
    for t in range(60):
        x = p.global_update(xl, lam)
        assert np.all(x >= p.lp.lo) and np.all(x <= p.lp.hi)
        xl = p.local_update(x, lam)
        lam = p.dual_update(x, xl, lam)
        for s in range(0, d.S, 3):
            o0, o1 = d.sub_ptr[s], d.sub_ptr[s + 1]
            scale = max(1.0, np.abs(xl[o0:o1]).max())
            assert np.abs(d.A[s] @ xl[o0:o1] - d.b[s]).max() <= 1e-10 * scale
            assert np.abs(p.abar[s] @ lam[o0:o1]).max() <= 1e-10 * max(1.0, np.abs(lam[o0:o1]).max())


# ---------------------------------------------------------------- fixed point = LP optimum
@pytest.mark.parametrize("make", [lambda: fx.chain_1ph(2), lambda: fx.chain_1ph(4), lambda: fx.two_bus_3ph(fg.WYE),
                                  lambda: fx.two_bus_3ph(fg.DELTA), fx.four_bus])
def test_converged_point_is_lp_vertex(make):
    """On tiny feeders the ADMM fixed point equals the unique optimal vertex found by brute-force
    enumeration within 1e-6 (north_star (a)); HiGHS agrees."""
    f = make()
    lp = oracle.assemble_lp(f)
    xv, ov, n_opt = vertex_enumeration(lp)
    assert n_opt == 1                                                  # unique optimum (reading C19)
    _, oh = highs(lp)
    assert abs(ov - oh) <= 1e-9 * max(1.0, abs(ov))
    p = oracle.build_problem(f, eps_rel=1e-10, lp=lp)
    r = oracle.solve(p, max_iter=2_000_000)
    assert r.converged
    assert np.abs(r.x - xv).max() <= 1e-6
    assert abs(r.objective - ov) <= 1e-6 * max(1.0, abs(ov))
    eq, bnd, _ = kkt_check(lp, r.x)
    assert eq <= 1e-7 and bnd == 0.0


def test_s1_and_rho_independence():
    """S = 1 (centralized) and rho in {10, 100, 1000} reach the same optimum
    (Abar, bbar contain no rho)."""
    f = fx.four_bus()
    lp = oracle.assemble_lp(f)
    _, oh = highs(lp)
    for single in (False, True):
        for rho in (10.0, 100.0, 1000.0):
            p = oracle.build_problem(f, rho=rho, eps_rel=1e-9, single=single, lp=lp)
            r = oracle.solve(p, max_iter=3_000_000)
            assert r.converged and abs(r.objective - oh) <= 1e-6 * abs(oh), (single, rho)


def test_default_tolerance_objective_close_to_lp():
    """SPEC.md acceptance 4: at the paper's defaults (rho = 100, eps_rel = 1e-3,
    PAPER.md:494) the 4-bus fixture converges with an objective gap <= 1e-2 and passes kkt_check at
    1e-2.  The 13-shaped feeder is held to 2.5e-2: the relative test of PAPER.md:358-361 bounds the
    residuals, not the gap (observed 1.9% with its 2-phase lateral and shunt conductances)."""
    for make, gap in ((fx.four_bus, 1e-2), (lambda: fg.make_feeder("13"), 2.5e-2)):
        f = make()
        lp = oracle.assemble_lp(f)
        _, oh = highs(lp)
        r = oracle.solve(oracle.build_problem(f, lp=lp))
        assert r.converged
        assert abs(r.objective - oh) <= gap * abs(oh)
        eq, bnd, _ = kkt_check(lp, r.x)
        assert eq <= 1e-2 and bnd == 0.0
