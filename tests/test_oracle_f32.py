"""Pins of the oracle's fp32 variant (oracle/admm_loop.c `oracle_run_f32`; reading F1).

The paper runs its GPU code in single precision and reports that this does not change the convergence
behaviour (Table V lists identical CPU/GPU iteration counts).  The fp32 loop is
pinned against the (already pinned) fp64 loop, never against itself:
  * exactness — on an instance whose every intermediate value is a short dyadic rational (rho = 4,
    nu in {1, 2}, Abar in {0, +-1/2}), binary32 and binary64 arithmetic are both exact, so the fp32
    iterates must equal the fp64 ones bit for bit: a dropped term, a wrong index or a transposed
    operand in the fp32 code breaks equality;
  * forward error — after K sweeps on the 13-bus shape the fp32 iterate stays within the rounding
    bound K * (n_max + nu_max + 4) * 2^-24 (relative to the largest entry) of the fp64 iterate;
  * precision robustness (the paper's Fig. 2 / Table V claim) — fp32 and fp64 reach the
    stopping criterion within +-5% of each other's iteration counts, objectives within 1e-2.
"""
import numpy as np
import pytest

import feedergen as fg
import oracle
from oracle.admm import problem_from_parts

from fixtures import four_bus


def _dyadic_instance():
    # S1: x0 + x1 = 2 (Abar = [[-.5, .5], [.5, -.5]], bbar = (1, 1)); S2: x1 - x2 = 0 (Abar = -.5 * ones)
    A = [np.array([[1.0, 1.0]]), np.array([[1.0, -1.0]])]
    b = [np.array([2.0]), np.array([0.0])]
    cols = [[0, 1], [1, 2]]
    c = [1.0, 0.0, 0.0]
    lo = [-8.0, -8.0, -np.inf]
    hi = [8.0, 8.0, np.inf]
    return problem_from_parts(A, b, cols, c, lo, hi, rho=4.0)


def test_f32_exact_on_dyadic_instance():
    p = _dyadic_instance()
    for a in p.abar:
        assert set(np.unique(np.abs(a))) <= {0.0, 0.5}
    x0 = (np.array([1.5, -2.0, 3.0, 0.25]), np.array([0.5, -1.0, 2.0, 0.75]))   # dyadic start
    for k in (1, 2, 3, 4):
        r64 = oracle.run_k(p, k, state=x0)
        r32 = oracle.run_k_f32(p, k, state=x0)
        # the fp64 run must itself stay dyadic-short for the comparison to be a pin of the fp32 code
        for v in (r64.x, r64.x_loc, r64.lam):
            assert np.all(np.asarray(v, np.float32).astype(np.float64) == v)
        np.testing.assert_array_equal(r32.x, r64.x)
        np.testing.assert_array_equal(r32.x_loc, r64.x_loc)
        np.testing.assert_array_equal(r32.lam, r64.lam)
        assert r32.pres == r64.pres and r32.dres == r64.dres


def test_f32_forward_error_13():
    f = fg.make_feeder("13")
    p = oracle.build_problem(f)
    K = 50
    r64 = oracle.run_k(p, K)
    r32 = oracle.run_k_f32(p, K)
    n_max = int(p.dec.n_s().max())
    nu_max = int(np.diff(p.dec.seg_ptr).max())
    bound = K * (n_max + nu_max + 4) * 2.0 ** -24
    for a, b in ((r32.x, r64.x), (r32.x_loc, r64.x_loc), (r32.lam, r64.lam)):
        err = np.abs(a - b).max() / max(1.0, np.abs(b).max())
        assert err <= bound, (err, bound)
        assert err > 0.0            # the fp32 loop really rounds to binary32


@pytest.mark.parametrize("make", [lambda: four_bus(), lambda: fg.make_feeder("13")], ids=["4bus", "13"])
def test_f32_precision_robustness(make):
    p = oracle.build_problem(make())
    r64 = oracle.solve(p)
    r32 = oracle.solve_f32(p)
    assert r64.converged and r32.converged
    assert abs(r32.iters - r64.iters) <= 0.05 * r64.iters, (r32.iters, r64.iters)
    assert abs(r32.objective - r64.objective) <= 1e-2 * abs(r64.objective)
