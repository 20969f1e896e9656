"""f4: the coarse-partition regime (closed form for any S >= 1,
PAPER.md:63; reading C25) and the IEEE37-shaped delta-only feeder (Tables
II-IV column 2).  CPU tests: oracle pins and library setup parity."""
import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from oracle.lp_reference import highs


def test_delta37_matches_tables():
    """57 buses, 56 lines, 16 leaves -> S = 97 (Table III; a tree, reading C14), and
    sum m_s = 1206 rows (Table II / IV); every load is a 3-phase delta load."""
    f = fg.make_feeder("37")
    st = fg.graph_stats(f)
    assert (st["nodes"], st["lines"], st["leaves"]) == (57, 56, 16)
    lp = oracle.assemble_lp(f)
    d = oracle.decompose(f, lp)
    assert d.S == 97 and lp.m == 1206 and int(d.m_s().sum()) == 1206
    assert np.all(f.load_conn == fg.DELTA) and np.all(f.load_phases == fg.ALL3)
    roles = {r.role for r in lp.rows}
    assert {"vdlm-6p", "vdlm-7", "vdlm-10"} <= roles and "vdlm-5p" not in roles
    _, oh = highs(lp)
    assert np.isfinite(oh)


def test_coarse_one_is_component():
    f = fg.make_feeder("123")
    lp = oracle.assemble_lp(f)
    a, b = oracle.decompose(f, lp), oracle.decompose(f, lp, coarse=1)
    assert np.array_equal(a.copy_global, b.copy_global) and np.array_equal(a.kind, b.kind)


@pytest.mark.parametrize("B", [2, 5, 16])
def test_coarse_structure(B):
    """Every LP row in exactly one subsystem; B_s B_s^T = I and sum_s B_s^T B_s = diag(nu);
    each coarse subsystem is the union of B consecutive depth-first component subsystems."""
    f = fg.make_feeder("123")
    lp = oracle.assemble_lp(f)
    base = oracle.decompose(f, lp)
    c = oracle.decompose(f, lp, coarse=B)
    assert sorted(r for rs in c.rows for r in rs) == list(range(lp.m))
    assert c.S == -(-base.S // B) and np.all(c.kind == 3)
    nu = np.zeros(lp.n)
    for s in range(c.S):
        I = np.array(c.cols[s])
        assert np.all(np.diff(I) > 0)                                   # B_s B_s^T = I (distinct columns)
        nu[I] += 1
    assert np.array_equal(nu, c.nu)
    order = oracle.decompose.__globals__["dfs_components"](f, list(base.kind), list(base.comp), list(base.leaf_bus))
    assert sorted(order) == list(range(base.S))
    for s in range(c.S):                                                 # rows = members' rows, DFS order
        assert c.rows[s] == [r for m in order[s * B:(s + 1) * B] for r in base.rows[m]]


@pytest.mark.parametrize("make,B", [(fx.four_bus, 3), (fx.physical, 4), (lambda: fx.chain_1ph(4), 2)])
def test_coarse_reaches_lp_optimum(make, B):
    """Coarser subsystems leave the LP, hence the fixed point, unchanged."""
    f = make()
    lp = oracle.assemble_lp(f)
    _, oh = highs(lp)
    q = oracle.build_problem(f, eps_rel=1e-10, lp=lp, coarse=B)
    r = oracle.solve(q, max_iter=3_000_000)
    assert r.converged and abs(r.objective - oh) <= 1e-6 * abs(oh)


@pytest.mark.parametrize("make,B", [(lambda: fg.make_feeder("123"), 4), (lambda: fg.make_feeder("123"), 16),
                                    (lambda: fg.make_feeder("37"), 1), (lambda: fg.make_feeder("37"), 8),
                                    (fx.physical, 16)])
def test_library_coarse_setup_matches_oracle(make, B):
    from oracle.precompute import precompute
    from paper_2310_09410_b200 import Lopf
    f = make()
    h = Lopf.setup(f, coarse=B)
    lp = oracle.assemble_lp(f)
    dec = oracle.decompose(f, lp, coarse=B)
    d = h.get_decomposition()
    assert np.array_equal(d.kind, dec.kind) and np.array_equal(d.comp, dec.comp)
    assert np.array_equal(d.sub_ptr, dec.sub_ptr) and np.array_equal(d.copy_global, dec.copy_global)
    rp, ci = h.get_consensus()
    assert np.array_equal(rp, dec.seg_ptr) and np.array_equal(ci, dec.seg_copy)
    for s in range(dec.S):
        ab, bb = h.get_operator(s, int(d.n_s[s]))
        ea, eb = precompute(dec.A[s], dec.b[s])
        assert np.abs(ab - ea).max() <= 1e-12 and np.abs(bb - eb).max(initial=0) <= 1e-12
