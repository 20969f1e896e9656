"""Oracle component decomposition and consensus maps.

Test infrastructure only.  Readings:
* C10  leaf = degree-1 node that is not the root; each leaf bus j is merged with its only
       line e into one LEAF subsystem; every other bus / line is its own subsystem.
* C11  rows: balance (3) and load (4) rows -> the bus's subsystem, (5) rows -> the line's.
       I_s = ascending global columns with a nonzero coefficient in any row of s
       ("A_s assembled over the union of columns its rows touch").
* C12  canonical subsystem order: non-leaf buses by index, then lines by index
       (a merged line carries its leaf bus).  Copies are numbered by concatenating I_s
       in that order; B_s is the 0-1 selection by I_s.
The consensus map of PAPER.md:297, I_si = {j : (B_s)_{j,i} = 1}, is stored as CSR
global -> copies (ascending copy index) with nu_i = sum_s |I_si|.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from feedergen import Feeder
from .lp import LP

BUS, LINE, LEAF, COARSE = 0, 1, 2, 3


class DecompositionError(ValueError):
    pass


@dataclass
class Decomposition:
    kind: np.ndarray          # int32 [S]   BUS / LINE / LEAF
    comp: np.ndarray          # int32 [S]   bus index (BUS) or line index (LINE, LEAF)
    leaf_bus: np.ndarray      # int32 [S]   merged leaf bus (LEAF) else -1
    rows: list                # rows[s] = list of LP row indices (owner order)
    cols: list                # cols[s] = I_s, ascending global ids
    A: list                   # A[s] dense m_s x n_s
    b: list                   # b[s] m_s
    sub_ptr: np.ndarray       # int64 [S+1] copy offsets
    copy_global: np.ndarray   # int32 [N_c]
    seg_ptr: np.ndarray       # int64 [n+1] CSR global -> copies
    seg_copy: np.ndarray      # int32 [N_c] copies of each global, ascending
    nu: np.ndarray            # int64 [n]

    @property
    def S(self) -> int:
        return int(self.kind.shape[0])

    @property
    def n_copies(self) -> int:
        return int(self.copy_global.shape[0])

    def m_s(self) -> np.ndarray:
        return np.array([len(r) for r in self.rows], dtype=np.int64)

    def n_s(self) -> np.ndarray:
        return np.array([len(c) for c in self.cols], dtype=np.int64)


def leaves_of(f: Feeder) -> np.ndarray:
    """Bool mask of leaf buses: degree 1 in the component graph and not the root (C10)."""
    deg = np.zeros(f.n_bus, dtype=np.int64)
    for e in range(f.n_line):
        deg[int(f.line_from[e])] += 1
        deg[int(f.line_to[e])] += 1
    leaf = deg == 1
    if 0 <= f.root_bus < f.n_bus:
        leaf[f.root_bus] = False
    return leaf


def dfs_components(f: Feeder, kinds, comps, leafb) -> list:
    """Component subsystems in depth-first order from the root bus (reading C25): the root's subsystem, then
    for each bus its incident lines in ascending index, each line's subsystem followed by the subtree behind
    it (the far bus's subsystem first).  A LEAF subsystem (line + leaf bus) appears once."""
    sub_of_bus, sub_of_line = {}, {}
    for s, (k, c, lb) in enumerate(zip(kinds, comps, leafb)):
        if k == BUS:
            sub_of_bus[c] = s
        else:
            sub_of_line[c] = s
            if k == LEAF:
                sub_of_bus[lb] = s
    adj = {i: [] for i in range(f.n_bus)}
    for e in range(f.n_line):
        adj[int(f.line_from[e])].append(e)
        adj[int(f.line_to[e])].append(e)
    order, seen_sub, seen_bus = [], set(), set()

    def emit(s):
        if s is not None and s not in seen_sub:
            seen_sub.add(s)
            order.append(s)

    def visit(b):                                   # iterative DFS, explicit stack of (bus, next line position)
        seen_bus.add(b)
        emit(sub_of_bus.get(b))
        stack = [[b, 0]]
        while stack:
            top = stack[-1]
            lines = sorted(adj[top[0]])
            if top[1] >= len(lines):
                stack.pop()
                continue
            e = lines[top[1]]
            top[1] += 1
            o = int(f.line_to[e]) if int(f.line_from[e]) == top[0] else int(f.line_from[e])
            emit(sub_of_line.get(e))
            if o not in seen_bus:
                seen_bus.add(o)
                emit(sub_of_bus.get(o))
                stack.append([o, 0])

    visit(f.root_bus)
    for b in range(f.n_bus):
        if b not in seen_bus:
            visit(b)
    for s in range(len(kinds)):
        emit(s)
    return order


def decompose(f: Feeder, lp: LP, single: bool = False, coarse: int = 0) -> Decomposition:
    """Component-wise decomposition with leaf merging; `single=True`
    gives the S = 1 partition (all rows in one subsystem); `coarse=B` merges
    consecutive runs of B component subsystems in depth-first order into one larger subsystem (the
    coarse-partition regime of PAPER.md:245, 399-402, still closed-form for any S >= 1;
    reading C25).  A coarse subsystem holds its members' rows in that order; kind COARSE, comp = run index."""
    if coarse and coarse > 1 and not single:
        base = decompose(f, lp)
        order = dfs_components(f, list(base.kind), list(base.comp), list(base.leaf_bus))
        runs = [order[i:i + coarse] for i in range(0, len(order), coarse)]
        rows = [[r for s in run for r in base.rows[s]] for run in runs]
        return _assemble(lp, [COARSE] * len(runs), list(range(len(runs))), [-1] * len(runs), rows)
    return _component(f, lp, single)


def _component(f: Feeder, lp: LP, single: bool) -> Decomposition:
    leaf = leaves_of(f)
    line_of_leaf = {}
    for e in range(f.n_line):
        i, j = int(f.line_from[e]), int(f.line_to[e])
        if leaf[i] and leaf[j]:
            raise DecompositionError(f"line {e} joins two leaves (disconnected network)")
        if leaf[i]:
            line_of_leaf[i] = e
        if leaf[j]:
            line_of_leaf[j] = e
    leaf_of_line = {e: j for j, e in line_of_leaf.items()}

    if single:
        kinds, comps, leafb = [BUS], [-1], [-1]
        owner_sub = None
    else:
        kinds, comps, leafb = [], [], []
        sub_of_bus, sub_of_line = {}, {}
        for i in range(f.n_bus):                 # non-leaf buses by index
            if not leaf[i]:
                sub_of_bus[i] = len(kinds)
                kinds.append(BUS), comps.append(i), leafb.append(-1)
        for e in range(f.n_line):                # lines by index; a merged line carries its leaf
            s = len(kinds)
            sub_of_line[e] = s
            if e in leaf_of_line:
                j = leaf_of_line[e]
                sub_of_bus[j] = s
                kinds.append(LEAF), comps.append(e), leafb.append(j)
            else:
                kinds.append(LINE), comps.append(e), leafb.append(-1)
        owner_sub = (sub_of_bus, sub_of_line)

    S = len(kinds)
    rows = [[] for _ in range(S)]
    for r, row in enumerate(lp.rows):            # attribution C11; LEAF: line rows come first (appended below)
        if single:
            rows[0].append(r)
            continue
        kind, idx = row.owner
        s = owner_sub[0][idx] if kind == "bus" else owner_sub[1][idx]
        rows[s].append(r)
    if not single:                               # LEAF row order: line rows, then the leaf bus rows (C12)
        for s in range(S):
            if kinds[s] == LEAF:
                rows[s] = ([r for r in rows[s] if lp.rows[r].owner[0] == "line"]
                           + [r for r in rows[s] if lp.rows[r].owner[0] == "bus"])

    return _assemble(lp, kinds, comps, leafb, rows)


def _assemble(lp: LP, kinds, comps, leafb, rows) -> Decomposition:
    """I_s = ascending columns touched by the rows of s (C11); dense A_s, b_s; copies; CSR; nu; orphans."""
    S = len(kinds)
    cols, As, bs = [], [], []
    for s in range(S):
        touched = set()
        for r in rows[s]:
            touched.update(lp.rows[r].coef.keys())
        I = sorted(touched)
        pos = {g: k for k, g in enumerate(I)}
        A = np.zeros((len(rows[s]), len(I)))
        b = np.zeros(len(rows[s]))
        for a, r in enumerate(rows[s]):
            for g, v in lp.rows[r].coef.items():
                A[a, pos[g]] = v
            b[a] = lp.rows[r].rhs
        cols.append(I), As.append(A), bs.append(b)

    sub_ptr = np.zeros(S + 1, dtype=np.int64)
    for s in range(S):
        sub_ptr[s + 1] = sub_ptr[s] + len(cols[s])
    copy_global = np.array([g for I in cols for g in I], dtype=np.int32)
    nu = np.bincount(copy_global, minlength=lp.n).astype(np.int64) if copy_global.size else np.zeros(lp.n, np.int64)
    orphans = np.nonzero(nu == 0)[0]
    if orphans.size:
        role, comp, ph = lp.var[int(orphans[0])]
        raise DecompositionError(f"orphan global variable {int(orphans[0])} ({role}, component {comp}, "
                                 f"phase {'abc'[ph]}): nu = 0")
    seg_ptr = np.zeros(lp.n + 1, dtype=np.int64)
    seg_ptr[1:] = np.cumsum(nu)
    seg_copy = np.argsort(copy_global, kind="stable").astype(np.int32)   # ascending copy index per global
    return Decomposition(kind=np.array(kinds, np.int32), comp=np.array(comps, np.int32),
                         leaf_bus=np.array(leafb, np.int32), rows=rows, cols=cols, A=As, b=bs,
                         sub_ptr=sub_ptr, copy_global=copy_global, seg_ptr=seg_ptr, seg_copy=seg_copy, nu=nu)
