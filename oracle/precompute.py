"""Oracle precompute of the local-update operators (Algorithm 1 lines 2-3).

Test infrastructure only.  The operators are computed by their literal definition,

    Abar_s = A_s^T (A_s A_s^T)^{-1} A_s - I_{n_s}
    bbar_s = A_s^T (A_s A_s^T)^{-1} b_s

with the inverse applied by numpy.linalg.solve (LAPACK LU) — a library primitive used
as one step, no reformulation.  The paper assumes A_s has full row rank and says row
reduction "can be applied ... as a preprocessing step"; the
reduction here is plain Gaussian elimination with partial pivoting.
"""
from __future__ import annotations

import numpy as np


class InfeasibleSubsystem(ValueError):
    pass


def row_rank_reduce(A: np.ndarray, b: np.ndarray, tol: float = 1e-10):
    """Return (A', b') made of the rows of (A, b) that are linearly independent of the rows
    before them, in original order; {x : A'x = b'} = {x : Ax = b}.

    Gaussian elimination with partial pivoting on the augmented rows; a row reducing to
    0 = beta with |beta| > tol * scale raises InfeasibleSubsystem."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = A.shape
    scale = max(1.0, float(np.abs(A).max()) if A.size else 1.0)
    basis = []           # list of (pivot column, reduced row, reduced rhs)
    keep = []
    for r in range(m):
        v = A[r].copy()
        beta = float(b[r])
        for (pc, br, bb) in basis:
            if v[pc] != 0.0:
                fct = v[pc] / br[pc]
                v = v - fct * br
                beta = beta - fct * bb
        pc = int(np.argmax(np.abs(v))) if n else 0
        if n and abs(v[pc]) > tol * scale:
            basis.append((pc, v, beta))
            keep.append(r)
        elif abs(beta) > tol * max(1.0, abs(float(b[r]))) * 1e3:
            raise InfeasibleSubsystem(f"row {r} is dependent but inconsistent (0 = {beta:.3e})")
    return A[keep], b[keep], keep


def precompute(A: np.ndarray, b: np.ndarray, reduce: bool = True):
    """(Abar_s, bbar_s) of closed_2 for one subsystem.  m_s = 0 gives Abar = -I, bbar = 0
    (the closed form with no local equality)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = A.shape[1]
    if reduce and A.shape[0]:
        A, b, _ = row_rank_reduce(A, b)
    if A.shape[0] == 0:
        return -np.eye(n), np.zeros(n)
    G = A @ A.T                                   # A_s A_s^T
    Abar = A.T @ np.linalg.solve(G, A) - np.eye(n)
    bbar = A.T @ np.linalg.solve(G, b)
    return Abar, bbar
