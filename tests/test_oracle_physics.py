"""Pins of the oracle's LP rows and residual terms against things OTHER than the oracle's formulas:

* a physically consistent operating point of a small radial feeder (fixtures.physical) computed by a
  textbook backward/forward sweep — complex power conservation at every bus, pi-model line shunts
  (S = w * conj(y)), the phasor linearisation of the voltage drop w_i - w_j = 2 Re(conj(V_phi) sum_psi
  z_phi,psi conj(S_psi / V_psi)) with balanced unit phasors V = (1, a^2, a) (the LinDist3Flow
  derivation), the first-order Taylor expansion of the ZIP law a * w^(alpha/2) at w = 1, and the
  delta -> bus conversion through branch currents.  Every assembled row (3), (4), (5a)-(5c)
   must vanish there; mutated rows (a flipped shunt sign, flows entered with the
  wrong direction, tau on the wrong side, g^s dropped from (5c), a transposed M) must not;
* hand-computed residual examples (readings C3/C4) whose dres, eps_dual and the
  sqrt(sum ||x_s||^2) branch of eps_prim are nonzero, so a dropped rho or eps_rel fails.
"""
import cmath
import math

import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from oracle.admm import problem_from_parts

A_OP = cmath.exp(2j * math.pi / 3)
V_BAL = np.array([1.0, A_OP * A_OP, A_OP])          # balanced unit phasors of phases a, b, c


def _tree(f):
    """Parent line of every bus and a breadth-first order from the root."""
    par = {}
    kids = {i: [] for i in range(f.n_bus)}
    for e in range(f.n_line):
        par[int(f.line_to[e])] = e
        kids[int(f.line_from[e])].append(e)
    order, q = [], [f.root_bus]
    while q:
        i = q.pop(0)
        order.append(i)
        q.extend(int(f.line_to[e]) for e in kids[i])
    return par, kids, order


def _load_powers(f, l, w):
    """(S_d, S_b) per phase slot of load l at bus voltages w (complex, index 0..2).
    S_d: first-order Taylor of the ZIP law P = a * what^(alpha/2), Q = b * what^(beta/2) at what = 1
    (what = w for wye, 3 w for delta as printed, reading C16).  S_b (drawn from the bus): = S_d for
    wye; for delta, branch phi = ab, bc, ca carries S_d[phi], the branch currents I = conj(S / (V_p - V_q))
    meet the bus phases by KCL and S_b = V conj(I_phase) (balanced unit phasors)."""
    i = int(f.load_bus[l])
    kappa = 3.0 if f.load_conn[l] == fg.DELTA else 1.0
    Sd = np.zeros(3, complex)
    for ph in fg.phase_list(f.load_phases[l]):
        wh = kappa * w[i][ph]
        P = f.load_a[l, ph] * (1.0 + f.load_alpha[l, ph] / 2.0 * (wh - 1.0))
        Q = f.load_b[l, ph] * (1.0 + f.load_beta[l, ph] / 2.0 * (wh - 1.0))
        Sd[ph] = complex(P, Q)
    if f.load_conn[l] == fg.WYE:
        return Sd, Sd.copy()
    pairs = [(0, 1), (1, 2), (2, 0)]
    Ib = [np.conj(Sd[k] / (V_BAL[p] - V_BAL[q])) for k, (p, q) in enumerate(pairs)]
    Iph = [Ib[0] - Ib[2], Ib[1] - Ib[0], Ib[2] - Ib[1]]
    return Sd, np.array([V_BAL[p] * np.conj(Iph[p]) for p in range(3)])


def physical_point(f, w_root=1.0, sweeps=300):
    """Backward/forward sweep power flow of the linearised network.  Returns a dict of values keyed
    like the oracle's variable catalog (role, component, phase)."""
    par, kids, order = _tree(f)
    w = {i: np.where([(int(f.bus_phases[i]) >> p) & 1 for p in range(3)], 1.0, 0.0) for i in range(f.n_bus)}
    w[f.root_bus] = w[f.root_bus] * w_root
    loads_at = {i: [l for l in range(f.n_load) if int(f.load_bus[l]) == i] for i in range(f.n_bus)}
    for _ in range(sweeps):
        Sd, Sb = {}, {}
        for l in range(f.n_load):
            Sd[l], Sb[l] = _load_powers(f, l, w)
        s_ij, s_ji, s_ser = {}, {}, {}
        for j in reversed(order):                                   # backward: complex power conservation
            demand = np.zeros(3, complex)
            for l in loads_at[j]:
                demand += Sb[l]
            demand += w[j] * np.conj(f.bus_gsh[j] + 1j * f.bus_bsh[j])        # bus shunt S = w conj(y)
            for e in kids[j]:
                demand += s_ij[e]                                   # power leaving j into child lines
            if j == f.root_bus:
                gen = demand
                continue
            e = par[j]
            i = int(f.line_from[e])
            y_to = f.line_gs_to[e] + 1j * f.line_bs_to[e]
            y_fr = f.line_gs_from[e] + 1j * f.line_bs_from[e]
            s_ji[e] = -demand                                       # balance at j: s_ji + demand = 0
            s_ser[e] = w[j] * np.conj(y_to) - s_ji[e]               # series flow i -> j (pi model)
            s_ij[e] = s_ser[e] + w[i] * np.conj(y_fr)
        for i in order:                                             # forward: voltage drops
            for e in kids[i]:
                j = int(f.line_to[e])
                pl = fg.phase_list(f.line_phases[e])
                z = f.line_r[e].reshape(3, 3) + 1j * f.line_x[e].reshape(3, 3)
                tau = f.line_tau[e]
                for ph in pl:
                    drop = 2.0 * np.real(np.conj(V_BAL[ph]) * sum(z[ph, ps] * np.conj(s_ser[e][ps] / V_BAL[ps])
                                                                   for ps in pl))
                    if tau[ph] != 1.0:                              # a tap changer: zero impedance, w_i = tau w_j
                        assert not np.any(z), "tap lines of the fixture have no impedance"
                        w[j][ph] = w[i][ph] / tau[ph]
                    else:
                        w[j][ph] = w[i][ph] - drop
    val = {}
    for i in range(f.n_bus):
        for ph in fg.phase_list(f.bus_phases[i]):
            val[("w", i, ph)] = w[i][ph]
    for e in range(f.n_line):
        for ph in fg.phase_list(f.line_phases[e]):
            val[("pf", e, ph)], val[("qf", e, ph)] = s_ij[e][ph].real, s_ij[e][ph].imag
            val[("pt", e, ph)], val[("qt", e, ph)] = s_ji[e][ph].real, s_ji[e][ph].imag
    for l in range(f.n_load):
        for ph in fg.phase_list(f.load_phases[l]):
            val[("pd", l, ph)], val[("qd", l, ph)] = Sd[l][ph].real, Sd[l][ph].imag
            val[("pb", l, ph)], val[("qb", l, ph)] = Sb[l][ph].real, Sb[l][ph].imag
    assert f.n_gen == 1 and int(f.gen_bus[0]) == f.root_bus
    for ph in fg.phase_list(f.gen_phases[0]):
        val[("pg", 0, ph)], val[("qg", 0, ph)] = gen[ph].real, gen[ph].imag
    return val


def _vector(lp, val):
    x = np.zeros(lp.n)
    for j, key in enumerate(lp.var):
        x[j] = val[key]
    return x


def _row_value(row, x):
    return sum(v * x[j] for j, v in row.coef.items()) - row.rhs


FEEDERS = {"physical": fx.physical, "four_bus": fx.four_bus, "two_bus_delta": lambda: fx.two_bus_3ph(fg.DELTA),
           "chain4": lambda: fx.chain_1ph(4)}


@pytest.mark.parametrize("name", sorted(FEEDERS))
def test_rows_vanish_at_physical_point(name):
    """Every row of (3), (4), (5) holds at the physically consistent point (1e-13)."""
    f = FEEDERS[name]()
    lp = oracle.assemble_lp(f)
    x = _vector(lp, physical_point(f))
    roles = set()
    for row in lp.rows:
        assert abs(_row_value(row, x)) <= 1e-13, (row.role, row.owner, row.phase, _row_value(row, x))
        roles.add(row.role)
    if name == "physical":
        assert {"balance-p", "balance-q", "vdlm-1", "vdlm-2", "vdlm-5p", "vdlm-5q", "vdlm-6p", "vdlm-7", "vdlm-10",
                "loss-p", "loss-q", "volt-drop"} <= roles
        assert x[lp.col[("w", 1, 0)]] == pytest.approx(1.0 / 1.02, abs=1e-15)      # the tap, w_i = tau w_j


def _mutations(f, lp):
    """Plausible assembly mistakes, each a function row -> mutated coefficient dict (or None = unchanged)."""
    col = lp.col

    def flip_gsh(row):                         # +g^sh w written as -g^sh w in balance-p
        if row.role != "balance-p":
            return None
        i, ph = row.owner[1], row.phase
        if f.bus_gsh[i, ph] == 0:
            return None
        c = dict(row.coef)
        c[col[("w", i, ph)]] = -c[col[("w", i, ph)]]
        return c

    def flip_bsh(row):                         # -b^sh w written as +b^sh w in balance-q
        if row.role != "balance-q":
            return None
        i, ph = row.owner[1], row.phase
        if f.bus_bsh[i, ph] == 0:
            return None
        c = dict(row.coef)
        c[col[("w", i, ph)]] = -c[col[("w", i, ph)]]
        return c

    def flow_direction(row):                   # at the to-bus, use p_eij (pf) instead of p_eji (pt)
        if row.role not in ("balance-p", "balance-q"):
            return None
        i, ph = row.owner[1], row.phase
        k = row.role[-1]
        c = dict(row.coef)
        changed = False
        for e in range(f.n_line):
            if int(f.line_to[e]) == i and ph in fg.phase_list(f.line_phases[e]):
                c.pop(col[(k + "t", e, ph)])
                c[col[(k + "f", e, ph)]] = 1.0
                changed = True
        return c if changed else None

    def tau_side(row):                         # w_i - tau w_j  ->  tau w_i - w_j
        if row.role != "volt-drop":
            return None
        e, ph = row.owner[1], row.phase
        tau = f.line_tau[e, ph]
        if tau == 1.0:
            return None
        i, j = int(f.line_from[e]), int(f.line_to[e])
        c = dict(row.coef)
        c[col[("w", i, ph)]] = c.get(col[("w", i, ph)], 0.0) + tau - 1.0
        c[col[("w", j, ph)]] = c.get(col[("w", j, ph)], 0.0) + -1.0 + tau
        return c

    def drop_gs_in_vd(row):                    # (5c) with p_eij instead of p_eij - g^s w_i
        if row.role != "volt-drop":
            return None
        e, ph = row.owner[1], row.phase
        if not np.any(f.line_gs_from[e]):
            return None
        Mp, _ = oracle.lp.m_matrices(f.line_r[e], f.line_x[e])
        i = int(f.line_from[e])
        c = dict(row.coef)
        for ps in fg.phase_list(f.line_phases[e]):
            c[col[("w", i, ps)]] = c.get(col[("w", i, ps)], 0.0) + Mp[ph, ps] * f.line_gs_from[e, ps]
        return c

    def m_transposed(row):                     # M^p_{psi,phi} instead of M^p_{phi,psi}
        if row.role != "volt-drop":
            return None
        e, ph = row.owner[1], row.phase
        pl = fg.phase_list(f.line_phases[e])
        if len(pl) < 2:
            return None
        Mp, Mq = oracle.lp.m_matrices(f.line_r[e], f.line_x[e])
        c = dict(row.coef)
        for ps in pl:
            c[col[("pf", e, ps)]] = c.get(col[("pf", e, ps)], 0.0) + Mp[ps, ph] - Mp[ph, ps]
            c[col[("qf", e, ps)]] = c.get(col[("qf", e, ps)], 0.0) + Mq[ps, ph] - Mq[ph, ps]
        return c

    def gs_to_in_loss(row):                    # (5a) with the from-end g^s on both ends
        if row.role != "loss-p":
            return None
        e, ph = row.owner[1], row.phase
        if f.line_gs_from[e, ph] == f.line_gs_to[e, ph]:
            return None
        j = int(f.line_to[e])
        c = dict(row.coef)
        c[col[("w", j, ph)]] = -f.line_gs_from[e, ph]
        return c

    return dict(flip_gsh=flip_gsh, flip_bsh=flip_bsh, flow_direction=flow_direction, tau_side=tau_side,
                drop_gs_in_vd=drop_gs_in_vd, m_transposed=m_transposed, gs_to_in_loss=gs_to_in_loss)


def test_physical_point_rejects_plausible_mistakes():
    """Each mutation of the assembly leaves some row violated by far more than rounding at the
    physical point — so the pin above would catch that mistake in the oracle."""
    f = fx.physical()
    lp = oracle.assemble_lp(f)
    x = _vector(lp, physical_point(f))
    for name, mut in _mutations(f, lp).items():
        worst, hit = 0.0, 0
        for row in lp.rows:
            c = mut(row)
            if c is None:
                continue
            hit += 1
            worst = max(worst, abs(sum(v * x[j] for j, v in c.items()) - row.rhs))
        assert hit > 0, name
        assert worst > 1e-6, (name, worst)


def test_physical_fixture_structure():
    """The 2-phase bus with three incident lines and no load has (m_s, n_s) = (4, 8) — IEEE13 bus 684,
    Table IV's minimum; the g^sh-only pass-through bus owns its w (C11); the leaf with a
    constant-power load owns its w only through g^sh."""
    f = fx.physical()
    lp = oracle.assemble_lp(f)
    d = oracle.decompose(f, lp)
    s684 = [s for s in range(d.S) if d.kind[s] == 0 and d.comp[s] == 3][0]
    assert (len(d.rows[s684]), len(d.cols[s684])) == (4, 8)
    s7 = [s for s in range(d.S) if d.kind[s] == 0 and d.comp[s] == 7][0]
    assert lp.col[("w", 7, 1)] in d.cols[s7]
    s5 = [s for s in range(d.S) if d.leaf_bus[s] == 5][0]
    assert lp.col[("w", 5, 0)] in d.cols[s5]
    g = f.copy()
    g.bus_gsh[7] = 0
    lp2 = oracle.assemble_lp(g)
    d2 = oracle.decompose(g, lp2)
    s7 = [s for s in range(d2.S) if d2.kind[s] == 0 and d2.comp[s] == 7][0]
    assert lp2.col[("w", 7, 1)] not in d2.cols[s7]
    assert (len(d2.rows[s7]), len(d2.cols[s7])) == (2, 4)              # 1-phase pass-through: (2, 4)


def test_physical_lp_optimum_is_admm_fixed_point():
    """The fixture is a feasible LP (HiGHS) and ADMM at tight eps reaches its optimum."""
    from oracle.lp_reference import highs
    f = fx.physical()
    lp = oracle.assemble_lp(f)
    _, oh = highs(lp)
    r = oracle.solve(oracle.build_problem(f, lp=lp, eps_rel=1e-9), max_iter=3_000_000)
    assert r.converged and abs(r.objective - oh) <= 1e-6 * abs(oh)


# ---------------------------------------------------------------- residual terms with nonzero dres / eps_dual
def _two_copy_problem(rho, eps_rel, S=1):
    """Two globals, each copied once by one subsystem with no local rows (B_s = I)."""
    return problem_from_parts([np.zeros((0, 2))], [np.zeros(0)], [[0, 1]], np.zeros(2), -np.inf * np.ones(2),
                              np.inf * np.ones(2), rho=rho, eps_rel=eps_rel)


def test_residuals_nonzero_dual_terms():
    """x = x_s = (0.6, 0.8), previous x_s = (0.59, 0.8), lambda = (3, 4), rho = 100, eps_rel = 1e-3:
    pres = 0; dres = rho * 0.01 = 1; eps_prim = 1e-3 * max(1, 1); eps_dual = 1e-3 * 5
    (PAPER.md:359).  A dropped rho gives dres = 0.01, a dropped eps_rel gives eps_dual = 5."""
    p = _two_copy_problem(100.0, 1e-3)
    pres, dres, ep, ed = p.residuals(np.array([0.6, 0.8]), np.array([0.6, 0.8]), np.array([0.59, 0.8]),
                                     np.array([3.0, 4.0]))
    assert pres == 0.0
    assert dres == pytest.approx(1.0, rel=1e-12)
    assert ep == pytest.approx(1e-3, rel=1e-12)
    assert ed == pytest.approx(5e-3, rel=1e-12)


def test_residuals_local_norm_branch_of_eps_prim():
    """x = 0, x_s = (3, 4): sqrt(sum ||B_s x||^2) = 0 < sqrt(sum ||x_s||^2) = 5, so eps_prim = 5 eps_rel
    (the second argument of the max, PAPER.md:358 with the braces of C3); pres = 5."""
    p = _two_copy_problem(10.0, 1e-2)
    pres, dres, ep, ed = p.residuals(np.zeros(2), np.array([3.0, 4.0]), np.array([3.0, 4.0]), np.zeros(2))
    assert pres == pytest.approx(5.0, rel=1e-15) and dres == 0.0
    assert ep == pytest.approx(0.05, rel=1e-12) and ed == 0.0


def test_residuals_weight_shared_globals_by_nu():
    """One global copied by two subsystems (nu = 2): ||B x||^2 sums over both copies, x = 3 ->
    sqrt(2 * 9) = 3 sqrt 2 (reading C4: sum_s ||B_s x||^2 = sum_i nu_i x_i^2); x_s = (1, 2) ->
    pres = sqrt(4 + 1); lambda = (1, -1) -> eps_dual = eps_rel sqrt 2."""
    p = problem_from_parts([np.zeros((0, 1)), np.zeros((0, 1))], [np.zeros(0)] * 2, [[0], [0]], np.zeros(1),
                           -np.inf * np.ones(1), np.inf * np.ones(1), rho=2.0, eps_rel=1e-3)
    pres, dres, ep, ed = p.residuals(np.array([3.0]), np.array([1.0, 2.0]), np.array([1.0, 1.0]),
                                     np.array([1.0, -1.0]))
    assert pres == pytest.approx(math.sqrt(5.0), rel=1e-15)
    assert dres == pytest.approx(2.0 * 1.0, rel=1e-15)
    assert ep == pytest.approx(1e-3 * 3.0 * math.sqrt(2.0), rel=1e-12)
    assert ed == pytest.approx(1e-3 * math.sqrt(2.0), rel=1e-12)
