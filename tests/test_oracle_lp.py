"""Pins of the oracle LP assembly (§II-A) against hand counts, textbook special cases
and circuit identities — never against a retyped copy of the oracle's own formulas."""
import cmath
import math

import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from oracle.lp import m_matrices


def test_spec_hand_counts():
    # 1 bus + 1-phase wye load + 1-phase gen -> n = 7, m = 6
    lp = oracle.assemble_lp(fx.one_bus_wye())
    assert (lp.n, lp.m) == (7, 6)
    assert sorted(v[0] for v in lp.var) == sorted(["pg", "qg", "w", "pb", "qb", "pd", "qd"])
    # two buses, one 3-phase line, nothing else -> m = 2*2*3 + 3*3 = 21
    lp = oracle.assemble_lp(fx.two_bus_line())
    assert lp.m == 21
    assert lp.n == 6 + 12


def test_m_matrix_spec_examples():
    # r = diag(.1), x = diag(.2) -> Mp = diag(-.2), Mq = diag(-.4)
    Mp, Mq = m_matrices(np.eye(3) * 0.1, np.eye(3) * 0.2)
    assert np.array_equal(Mp, np.diag([-0.2] * 3)) and np.array_equal(Mq, np.diag([-0.4] * 3))
    # r12 = .01, x12 = .02 -> Mp[1,2] = .01 - sqrt(3) .02
    r = np.zeros((3, 3)); x = np.zeros((3, 3))
    r[0, 1], x[0, 1] = 0.01, 0.02
    Mp, _ = m_matrices(r, x)
    assert Mp[0, 1] == pytest.approx(0.01 - math.sqrt(3) * 0.02, abs=1e-16)


def _row_value(lp, row, xvec):
    return sum(v * xvec[j] for j, v in row.coef.items()) - row.rhs


def test_distflow_positive_sequence():
    """Balanced flows through a line with symmetric r, x reduce (5c) to positive-sequence
    DistFlow w_i - w_j = 2 (r1 P + x1 Q), r1 = r_s - r_m (textbook LinDistFlow)."""
    f = fx.two_bus_line()
    lp = oracle.assemble_lp(f)
    P, Q = 0.2, 0.1
    rs, rm, xs, xm = 0.010, 0.004, 0.030, 0.012
    x = np.zeros(lp.n)
    for ph in range(3):
        x[lp.col[("pf", 0, ph)]] = P
        x[lp.col[("qf", 0, ph)]] = Q
        x[lp.col[("w", 1, ph)]] = 1.0
        x[lp.col[("w", 0, ph)]] = 1.0 + 2 * ((rs - rm) * P + (xs - xm) * Q)
    for row in lp.rows:
        if row.role == "volt-drop":
            assert abs(_row_value(lp, row, x)) < 1e-15
    # a single-phase line: w_i - w_j = 2 (r P + x Q) exactly (LinDistFlow)
    f1 = fx.chain_1ph(2)
    lp1 = oracle.assemble_lp(f1)
    r, xx = f1.line_r[0, 0], f1.line_x[0, 0]
    y = np.zeros(lp1.n)
    y[lp1.col[("pf", 0, 0)]], y[lp1.col[("qf", 0, 0)]] = 0.3, -0.2
    y[lp1.col[("w", 1, 0)]] = 0.95
    y[lp1.col[("w", 0, 0)]] = 0.95 + 2 * (r * 0.3 + xx * -0.2)
    vd = [row for row in lp1.rows if row.role == "volt-drop"][0]
    assert abs(_row_value(lp1, vd, y)) < 1e-15


def test_line_losses_lossless_and_charging():
    """(5a)-(5b): zero shunts give p_ij + p_ji = 0; b^s terms give the charging -b^s_i w_i - b^s_j w_j."""
    f = fx.two_bus_3ph(shunts=True)
    lp = oracle.assemble_lp(f)
    rng = np.random.default_rng(0)
    x = rng.normal(size=lp.n)
    for row in lp.rows:
        if row.role == "loss-p":                            # g^s = 0 in the fixture
            ph = row.phase
            assert set(row.coef) == {lp.col[("pf", 0, ph)], lp.col[("pt", 0, ph)]}
        if row.role == "loss-q":
            ph = row.phase
            expect = (x[lp.col[("qf", 0, ph)]] + x[lp.col[("qt", 0, ph)]]
                      + f.line_bs_from[0, ph] * x[lp.col[("w", 0, ph)]] + f.line_bs_to[0, ph] * x[lp.col[("w", 1, ph)]])
            assert _row_value(lp, row, x) == pytest.approx(expect, abs=1e-14)


def test_vdlm_nominal_voltage_and_taylor():
    """VDLM-1/2: at nominal voltage (w = 1) every load type draws a; the
    row is the first-order Taylor expansion of the ZIP law a * V^alpha = a * w^(alpha/2) at w = 1."""
    f = fx.one_bus_wye()
    for alpha in (0.0, 1.0, 2.0):
        g = f.copy()
        g.load_alpha[0, 0] = alpha
        lp = oracle.assemble_lp(g)
        row = [r for r in lp.rows if r.role == "vdlm-1"][0]
        jw, jd = lp.col[("w", 0, 0)], lp.col[("pd", 0, 0)]
        a = g.load_a[0, 0]
        for w in (1.0, 1.01, 0.99):
            # solve the row for p^d
            pd = (row.rhs - row.coef.get(jw, 0.0) * w) / row.coef[jd]
            exact = a * w ** (alpha / 2)
            tol = 1e-15 if w == 1.0 else 2e-4 * a
            assert abs(pd - exact) <= tol


def test_wye_coupling_and_delta_balanced():
    """VDLM-5: p^b = p^d for wye loads.  VDLM-6..10 are exactly the
    balanced-voltage delta->bus power conversion with d-index 1,2,3 = branches ab, bc, ca
    (SURVEY App. A1): computed here from complex circuit quantities, independently of the rows."""
    lp = oracle.assemble_lp(fx.two_bus_3ph(fg.DELTA))
    rng = np.random.default_rng(7)
    a = cmath.exp(2j * math.pi / 3)
    V = {1: 1.0 + 0j, 2: a * a, 3: a}                       # balanced phasors a, b, c
    for trial in range(20):
        Sd = {k: complex(rng.uniform(-1, 1), rng.uniform(-1, 1)) for k in (1, 2, 3)}   # ab, bc, ca
        pairs = {1: (1, 2), 2: (2, 3), 3: (3, 1)}
        Ib = {k: (Sd[k] / (V[p] - V[q])).conjugate() for k, (p, q) in pairs.items()}  # branch currents
        Iph = {1: Ib[1] - Ib[3], 2: Ib[2] - Ib[1], 3: Ib[3] - Ib[2]}                   # KCL at phases
        Sb = {p: V[p] * Iph[p].conjugate() for p in (1, 2, 3)}
        x = np.zeros(lp.n)
        for p in (1, 2, 3):
            x[lp.col[("pd", 0, p - 1)]], x[lp.col[("qd", 0, p - 1)]] = Sd[p].real, Sd[p].imag
            x[lp.col[("pb", 0, p - 1)]], x[lp.col[("qb", 0, p - 1)]] = Sb[p].real, Sb[p].imag
        for row in lp.rows:
            if row.role in ("vdlm-6p", "vdlm-6q", "vdlm-7", "vdlm-8", "vdlm-9", "vdlm-10"):
                assert abs(_row_value(lp, row, x)) < 1e-14, row.role
    lpw = oracle.assemble_lp(fx.two_bus_3ph(fg.WYE))
    roles = [r.role for r in lpw.rows]
    assert roles.count("vdlm-5p") == 3 and roles.count("vdlm-5q") == 3 and "vdlm-7" not in roles


def test_objective_and_bounds():
    """c = 1 on every p^g column; bounds from (2); loads free."""
    f = fx.four_bus()
    lp = oracle.assemble_lp(f)
    for j, (role, comp, ph) in enumerate(lp.var):
        assert lp.c[j] == (1.0 if role == "pg" else 0.0)
        if role in ("pb", "qb", "pd", "qd"):
            assert lp.lo[j] == -np.inf and lp.hi[j] == np.inf
        else:
            assert np.isfinite(lp.lo[j]) and np.isfinite(lp.hi[j]) and lp.lo[j] <= lp.hi[j]
    # variable blocks in PAPER.md:215-221 order: gen, bus, load, line
    blocks = [{"pg": 0, "qg": 0, "w": 1, "pb": 2, "qb": 2, "pd": 2, "qd": 2}.get(r, 3) for r, _, _ in lp.var]
    assert blocks == sorted(blocks)


@pytest.mark.parametrize("shape,exp", [("13", dict(nodes=29, lines=28, leaves=7)),
                                       ("123", dict(nodes=147, lines=146, leaves=43))])
def test_shapes_match_table3(shape, exp):
    """Synthetic shapes reproduce Table III node/line/leaf counts."""
    st = fg.graph_stats(fg.make_feeder(shape))
    for k, v in exp.items():
        assert st[k] == v


def test_lp_feasible_highs():
    """Configs 1-2 and the fixtures are feasible LPs (HiGHS, SURVEY §8(d) 'Feasibility is checked')."""
    from oracle.lp_reference import highs
    for f in (fg.make_feeder("13"), fg.make_feeder("123"), fx.four_bus()):
        _, obj = highs(oracle.assemble_lp(f))
        assert np.isfinite(obj) and obj > 0
