"""Brute-force LP references used to pin the oracle (TEST INFRASTRUCTURE ONLY).

* `vertex_enumeration`  exact optimum of a tiny `min c'x, Ax=b, lo<=x<=hi` by enumerating every
                        basic solution in the null space of A (x = x0 + N z, d = dim null(A) active
                        bounds at a time) — no optimization solver involved.
* `highs`               SciPy's HiGHS (`scipy.optimize.linprog(method="highs")`) as a second,
                        independent reference ("solve_lp_reference").
* `kkt_check`           equality / bound violation and objective of a point.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.optimize import linprog

from .lp import LP


def lp_arrays(lp: LP):
    A, b = lp.dense()
    return A, b, lp.c.copy(), lp.lo.copy(), lp.hi.copy()


def vertex_enumeration(lp: LP, tol: float = 1e-9, max_dof: int = 4):
    """Return (x*, obj*, n_optimal_vertices).  Raises if dim null(A) > max_dof (too many subsets).
    Boundedness is not checked here: every fixture is cross-checked against `highs`."""
    A, b, c, lo, hi = lp_arrays(lp)
    x0, *_ = np.linalg.lstsq(A, b, rcond=None)
    if np.abs(A @ x0 - b).max() > 1e-9 * max(1.0, np.abs(b).max()):
        raise ValueError("Ax = b is inconsistent")
    N = sla.null_space(A)
    d = N.shape[1]
    if d == 0:
        ok = np.all(x0 >= lo - tol) and np.all(x0 <= hi + tol)
        return (x0, float(c @ x0), 1) if ok else (None, np.inf, 0)
    if d > max_dof:
        raise ValueError(f"null space dimension {d} > {max_dof}")
    cons = [(j, lo[j]) for j in range(lp.n) if np.isfinite(lo[j])] + \
           [(j, hi[j]) for j in range(lp.n) if np.isfinite(hi[j])]
    best, best_x, verts = np.inf, None, []
    for sub in itertools.combinations(range(len(cons)), d):
        idx = [cons[t][0] for t in sub]
        if len(set(idx)) < d:
            continue
        M = N[idx, :]
        if abs(np.linalg.det(M)) < 1e-12:
            continue
        z = np.linalg.solve(M, np.array([cons[t][1] for t in sub]) - x0[idx])
        x = x0 + N @ z
        if np.all(x >= lo - tol) and np.all(x <= hi + tol):
            val = float(c @ x)
            verts.append((val, x))
            if val < best:
                best, best_x = val, x
    n_opt = len({tuple(np.round(x, 9)) for v, x in verts if v <= best + 1e-9 * max(1.0, abs(best))})
    return best_x, best, n_opt


def highs(lp: LP):
    """HiGHS optimum (x, obj) or raises on a non-optimal status."""
    rows, cols, vals = [], [], []
    for r, row in enumerate(lp.rows):
        for j, v in row.coef.items():
            rows.append(r), cols.append(j), vals.append(v)
    A = sp.csr_matrix((vals, (rows, cols)), shape=(lp.m, lp.n))
    b = np.array([r.rhs for r in lp.rows])
    bounds = [(None if np.isinf(l) else l, None if np.isinf(h) else h) for l, h in zip(lp.lo, lp.hi)]
    res = linprog(lp.c, A_eq=A, b_eq=b, bounds=bounds, method="highs")
    if res.status != 0:
        raise RuntimeError(f"HiGHS status {res.status}: {res.message}")
    return res.x, float(res.fun)


def kkt_check(lp: LP, x: np.ndarray):
    """(max |Ax - b|, max bound violation, objective) — SPEC.md:244-252."""
    A, b, c, lo, hi = lp_arrays(lp)
    eq = float(np.abs(A @ x - b).max()) if lp.m else 0.0
    bnd = float(max(np.max(lo - x, initial=0.0), np.max(x - hi, initial=0.0)))
    return eq, bnd, float(c @ x)
