"""Oracle LP assembly: the linearized OPF of PAPER.md §II-A as `min c'x, Ax = b, lo <= x <= hi`.

Test infrastructure only (see oracle/__init__.py).  Every row is written out as the
paper prints it; the voltage-dependent load variable w-hat is substituted
(VDLM-3 / VDLM-4), reading C16 of DESIGN.md.

Variable order (PAPER.md:215-221 block order; within a block: component index,
then role, then phase — reading C12):
  gen k:  pg(phases), qg(phases)
  bus i:  w(phases)
  load l: pb, qb, pd, qd (each over phases)
  line e: pf = p_eij, qf = q_eij, pt = p_eji, qt = q_eji (each over phases); i = from, j = to
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from feedergen import Feeder, phase_list

SQ3 = math.sqrt(3.0)


@dataclass
class Row:
    role: str                 # balance-p, balance-q, vdlm-1, vdlm-2, vdlm-5p, vdlm-5q, vdlm-6p, vdlm-6q,
                              # vdlm-7..vdlm-10, loss-p, loss-q, volt-drop
    owner: tuple              # ('bus', i) or ('line', e): the component whose subsystem owns the row (C11)
    phase: int
    coef: dict                # column -> coefficient (exact zeros are never stored)
    rhs: float


@dataclass
class LP:
    n: int
    c: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    var: list                 # var[j] = (role, component, phase)
    col: dict                 # (role, component, phase) -> j
    rows: list = field(default_factory=list)

    @property
    def m(self) -> int:
        return len(self.rows)

    def dense(self):
        A = np.zeros((self.m, self.n))
        b = np.zeros(self.m)
        for r, row in enumerate(self.rows):
            for j, v in row.coef.items():
                A[r, j] += v
            b[r] = row.rhs
        return A, b


def m_matrices(r: np.ndarray, x: np.ndarray):
    """M^p_e and M^q_e exactly as displayed at PAPER.md:180-191 (1-based (phi, psi) -> 0-based)."""
    r = np.asarray(r, dtype=np.float64).reshape(3, 3)
    x = np.asarray(x, dtype=np.float64).reshape(3, 3)
    Mp = np.array([
        [-2 * r[0, 0], r[0, 1] - SQ3 * x[0, 1], r[0, 2] + SQ3 * x[0, 2]],
        [r[1, 0] + SQ3 * x[1, 0], -2 * r[1, 1], r[1, 2] - SQ3 * x[1, 2]],
        [r[2, 0] - SQ3 * x[2, 0], r[2, 1] + SQ3 * x[2, 1], -2 * r[2, 2]],
    ])
    Mq = np.array([
        [-2 * x[0, 0], x[0, 1] + SQ3 * r[0, 1], x[0, 2] - SQ3 * r[0, 2]],
        [x[1, 0] - SQ3 * r[1, 0], -2 * x[1, 1], x[1, 2] + SQ3 * r[1, 2]],
        [x[2, 0] + SQ3 * r[2, 0], x[2, 1] - SQ3 * r[2, 1], -2 * x[2, 2]],
    ])
    return Mp, Mq


def _catalog(f: Feeder):
    var, col = [], {}

    def add(role, comp, ph):
        col[(role, comp, ph)] = len(var)
        var.append((role, comp, ph))

    for k in range(f.n_gen):                          # {pg, qg}_{k in G, phi in P_k}
        for role in ("pg", "qg"):
            for ph in phase_list(f.gen_phases[k]):
                add(role, k, ph)
    for i in range(f.n_bus):                          # {w}_{i in N, phi in P_i}
        for ph in phase_list(f.bus_phases[i]):
            add("w", i, ph)
    for l in range(f.n_load):                         # {pb, qb, pd, qd}_{l, phi in P_l}
        for role in ("pb", "qb", "pd", "qd"):
            for ph in phase_list(f.load_phases[l]):
                add(role, l, ph)
    for e in range(f.n_line):                         # {p_eij, q_eij, p_eji, q_eji}_{e, phi in P_e}
        for role in ("pf", "qf", "pt", "qt"):
            for ph in phase_list(f.line_phases[e]):
                add(role, e, ph)
    return var, col


def assemble_lp(f: Feeder) -> LP:
    """Assemble (LP_model) PAPER.md:206-227 from (2)-(5).

    Bounds (operational): pg, qg, w, and both flow directions of
    every line; load variables are unbounded (+-inf).  Objective:
    c = 1 on every p^g column.
    """
    var, col = _catalog(f)
    n = len(var)
    c = np.zeros(n)
    lo = np.full(n, -np.inf)
    hi = np.full(n, np.inf)
    for j, (role, comp, ph) in enumerate(var):
        if role == "pg":
            c[j] = 1.0
            lo[j], hi[j] = f.gen_pmin[comp, ph], f.gen_pmax[comp, ph]
        elif role == "qg":
            lo[j], hi[j] = f.gen_qmin[comp, ph], f.gen_qmax[comp, ph]
        elif role == "w":
            lo[j], hi[j] = f.bus_wmin[comp, ph], f.bus_wmax[comp, ph]
        elif role in ("pf", "pt"):
            lo[j], hi[j] = f.line_pmin[comp, ph], f.line_pmax[comp, ph]
        elif role in ("qf", "qt"):
            lo[j], hi[j] = f.line_qmin[comp, ph], f.line_qmax[comp, ph]
    lp = LP(n=n, c=c, lo=lo, hi=hi, var=var, col=col)

    def row(role, owner, ph, terms, rhs):
        coef = {}
        for j, v in terms:
            coef[j] = coef.get(j, 0.0) + v
        coef = {j: v for j, v in coef.items() if v != 0.0}
        lp.rows.append(Row(role, owner, ph, coef, float(rhs)))

    lines_of = [[] for _ in range(f.n_bus)]
    for e in range(f.n_line):                                   # incidence lists, line index ascending
        lines_of[int(f.line_from[e])].append(e)
        if int(f.line_to[e]) != int(f.line_from[e]):
            lines_of[int(f.line_to[e])].append(e)
    loads_of = [[] for _ in range(f.n_bus)]
    for l in range(f.n_load):
        loads_of[int(f.load_bus[l])].append(l)
    gens_of = [[] for _ in range(f.n_bus)]
    for k in range(f.n_gen):
        gens_of[int(f.gen_bus[k])].append(k)

    for i in range(f.n_bus):
        lines_at, loads_at, gens_at = sorted(lines_of[i]), loads_of[i], gens_of[i]
        # (3) power balance, PAPER.md:128-129:
        #   sum_{(e,i,j) in E_i} p_eij + sum_l p^b_l + g^sh w = sum_k p^g_k   (and the q analogue, -b^sh w)
        # The flow "leaving i into e" is p_eij = pf when i is e's from-bus, p_eji = pt when i is its to-bus.
        for kind in ("p", "q"):
            for ph in phase_list(f.bus_phases[i]):
                t = []
                for e in lines_at:
                    if ph in phase_list(f.line_phases[e]):
                        t.append((col[(kind + ("f" if f.line_from[e] == i else "t"), e, ph)], 1.0))
                for l in loads_at:
                    if ph in phase_list(f.load_phases[l]):
                        t.append((col[(kind + "b", l, ph)], 1.0))
                sh = f.bus_gsh[i, ph] if kind == "p" else -f.bus_bsh[i, ph]
                t.append((col[("w", i, ph)], sh))
                for k in gens_at:
                    if ph in phase_list(f.gen_phases[k]):
                        t.append((col[(kind + "g", k, ph)], -1.0))
                row("balance-" + kind, ("bus", i), ph, t, 0.0)
        # (4) voltage-dependent loads.
        for l in loads_at:
            pl = phase_list(f.load_phases[l])
            kappa = 3.0 if f.load_conn[l] == 1 else 1.0          # w-hat = w (VDLM-3) or 3w (VDLM-4)
            for ph in pl:                                       # VDLM-1: p^d = (a alpha/2)(w-hat - 1) + a
                a, al = f.load_a[l, ph], f.load_alpha[l, ph]
                row("vdlm-1", ("bus", i), ph,
                    [(col[("pd", l, ph)], 1.0), (col[("w", i, ph)], -(a * al / 2.0) * kappa)],
                    a * (1.0 - al / 2.0))
            for ph in pl:                                       # VDLM-2: q^d = (b beta/2)(w-hat - 1) + b
                bb, be = f.load_b[l, ph], f.load_beta[l, ph]
                row("vdlm-2", ("bus", i), ph,
                    [(col[("qd", l, ph)], 1.0), (col[("w", i, ph)], -(bb * be / 2.0) * kappa)],
                    bb * (1.0 - be / 2.0))
            if f.load_conn[l] == 0:                             # VDLM-5 (wye): p^b = p^d, q^b = q^d
                for ph in pl:
                    row("vdlm-5p", ("bus", i), ph, [(col[("pb", l, ph)], 1.0), (col[("pd", l, ph)], -1.0)], 0.0)
                for ph in pl:
                    row("vdlm-5q", ("bus", i), ph, [(col[("qb", l, ph)], 1.0), (col[("qd", l, ph)], -1.0)], 0.0)
            else:                                               # VDLM-6..10 (delta, phases 1,2,3 = a,b,c)
                pb = lambda p: col[("pb", l, p - 1)]  # noqa: E731   1-based phase as printed
                qb = lambda p: col[("qb", l, p - 1)]  # noqa: E731
                pd = lambda p: col[("pd", l, p - 1)]  # noqa: E731
                qd = lambda p: col[("qd", l, p - 1)]  # noqa: E731
                row("vdlm-6p", ("bus", i), -1, [(pb(p), 1.0) for p in (1, 2, 3)] + [(pd(p), -1.0) for p in (1, 2, 3)], 0.0)
                row("vdlm-6q", ("bus", i), -1, [(qb(p), 1.0) for p in (1, 2, 3)] + [(qd(p), -1.0) for p in (1, 2, 3)], 0.0)
                # VDLM-7: 3/2 pb2 - sqrt3/2 qb2 = pd2 + 1/2 pd1 - sqrt3/2 qd1
                row("vdlm-7", ("bus", i), -1, [(pb(2), 1.5), (qb(2), -SQ3 / 2), (pd(2), -1.0), (pd(1), -0.5),
                                               (qd(1), SQ3 / 2)], 0.0)
                # VDLM-8: sqrt3/2 pb2 + 3/2 qb2 = sqrt3/2 pd1 + 1/2 qd1 + qd2
                row("vdlm-8", ("bus", i), -1, [(pb(2), SQ3 / 2), (qb(2), 1.5), (pd(1), -SQ3 / 2), (qd(1), -0.5),
                                               (qd(2), -1.0)], 0.0)
                # VDLM-9: sqrt3 qb2 + 3/2 pb3 - sqrt3/2 qb3 = 1/2 pd1 + sqrt3/2 qd1 + pd3
                row("vdlm-9", ("bus", i), -1, [(qb(2), SQ3), (pb(3), 1.5), (qb(3), -SQ3 / 2), (pd(1), -0.5),
                                               (qd(1), -SQ3 / 2), (pd(3), -1.0)], 0.0)
                # VDLM-10: -sqrt3 pb2 + sqrt3/2 pb3 + 3/2 qb3 = -sqrt3/2 pd1 + 1/2 qd1 + qd3
                row("vdlm-10", ("bus", i), -1, [(pb(2), -SQ3), (pb(3), SQ3 / 2), (qb(3), 1.5), (pd(1), SQ3 / 2),
                                                (qd(1), -0.5), (qd(3), -1.0)], 0.0)

    for e in range(f.n_line):
        i, j = int(f.line_from[e]), int(f.line_to[e])
        pl = phase_list(f.line_phases[e])
        gs_i, bs_i = f.line_gs_from[e], f.line_bs_from[e]
        gs_j, bs_j = f.line_gs_to[e], f.line_bs_to[e]
        Mp, Mq = m_matrices(f.line_r[e], f.line_x[e])
        for ph in pl:      # (5a) powerloss-1: p_eij + p_eji = g^s_eij w_i + g^s_eji w_j
            row("loss-p", ("line", e), ph, [(col[("pf", e, ph)], 1.0), (col[("pt", e, ph)], 1.0),
                                            (col[("w", i, ph)], -gs_i[ph]), (col[("w", j, ph)], -gs_j[ph])], 0.0)
        for ph in pl:      # (5b) powerloss-2: q_eij + q_eji = -b^s_eij w_i - b^s_eji w_j
            row("loss-q", ("line", e), ph, [(col[("qf", e, ph)], 1.0), (col[("qt", e, ph)], 1.0),
                                            (col[("w", i, ph)], bs_i[ph]), (col[("w", j, ph)], bs_j[ph])], 0.0)
        for ph in pl:      # (5c) voltage_mag_diff, moved to the left-hand side:
            # w_i - tau w_j + sum_psi Mp[ph,psi](p_eij,psi - g^s w_i,psi) + sum_psi Mq[ph,psi](q_eij,psi + b^s w_i,psi) = 0
            t = [(col[("w", i, ph)], 1.0), (col[("w", j, ph)], -f.line_tau[e, ph])]
            for ps in pl:
                t.append((col[("pf", e, ps)], Mp[ph, ps]))
                t.append((col[("w", i, ps)], -Mp[ph, ps] * gs_i[ps]))
                t.append((col[("qf", e, ps)], Mq[ph, ps]))
                t.append((col[("w", i, ps)], Mq[ph, ps] * bs_i[ps]))
            row("volt-drop", ("line", e), ph, t, 0.0)
    return lp
