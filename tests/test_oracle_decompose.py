"""Pins of the oracle decomposition (Tables III-IV) by graph arithmetic,
hand counts and the B_s algebra."""
import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from feedergen import PH_A, PH_C, FeederBuilder
from oracle.decompose import BUS, LEAF, LINE, DecompositionError, decompose


def _tree(parents, root=0):
    fb = FeederBuilder("tree")
    for _ in range(len(parents) + 1):
        fb.bus(PH_A)
    fb.gen(root, PH_A)
    for child, par in enumerate(parents, start=1):
        fb.line(par, child, PH_A, np.eye(3) * 0.01, np.eye(3) * 0.02)
        fb.load(child, PH_A, fg.WYE, [1, 0, 0], [1, 0, 0], [0.1, 0, 0], [0.05, 0, 0])
    return fb.build()


def test_spec_path_and_star():
    # 3-bus path rooted at an end -> S = 3 + 2 - 1 = 4 (root not merged)
    f = _tree([0, 1])
    assert decompose(f, oracle.assemble_lp(f)).S == 4
    # star, centre + 3 leaves, rooted at the centre -> S = 4 + 3 - 3 = 4
    f = _tree([0, 0, 0])
    d = decompose(f, oracle.assemble_lp(f))
    assert d.S == 4 and list(d.kind) == [BUS, LEAF, LEAF, LEAF]


def test_s_identity_random_trees():
    """S = #nodes + #lines - #non-root leaves (Table III)."""
    rng = np.random.default_rng(3)
    for n in (2, 5, 17, 40):
        parents = [int(rng.integers(k)) for k in range(1, n)]
        f = _tree(parents)
        st = fg.graph_stats(f)
        assert decompose(f, oracle.assemble_lp(f)).S == st["nodes"] + st["lines"] - st["leaves"]


@pytest.mark.parametrize("shape,S", [("13", 50), ("123", 250), ("8500", 25001)])
def test_shapes_reproduce_table3_S(shape, S):
    """Table III S column: 50 = 29 + 28 - 7 etc."""
    f = fg.make_feeder(shape)
    if shape == "8500":                         # decomposition only needs the graph: count without the LP
        st = fg.graph_stats(f)
        assert st["nodes"] + st["lines"] - st["leaves"] == S
    else:
        assert decompose(f, oracle.assemble_lp(f)).S == S


def test_b_algebra_and_counts():
    """sum m_s = m; sum n_s = sum nu = N_c; B_s B_s^T = I; sum_s B_s^T B_s = diag(nu)."""
    for f in (fg.make_feeder("13"), fg.make_feeder("123"), fx.four_bus()):
        lp = oracle.assemble_lp(f)
        d = decompose(f, lp)
        assert d.m_s().sum() == lp.m
        assert d.n_s().sum() == d.nu.sum() == d.n_copies
        D = np.zeros((lp.n, lp.n))
        for s in range(d.S):
            I = d.cols[s]
            B = np.zeros((len(I), lp.n))
            B[np.arange(len(I)), I] = 1.0
            assert np.array_equal(B @ B.T, np.eye(len(I)))
            assert list(I) == sorted(I)
            D += B.T @ B
        assert np.array_equal(D, np.diag(d.nu.astype(float)))
        # CSR: copies of every global ascending, and consistent with copy_global
        for i in range(lp.n):
            seg = d.seg_copy[d.seg_ptr[i]:d.seg_ptr[i + 1]]
            assert list(seg) == sorted(seg) and all(d.copy_global[k] == i for k in seg)
        # every row attributed once
        assert sorted(r for rs in d.rows for r in rs) == list(range(lp.m))


def test_table4_minima_column_rule():
    """Reading C11 reproduces Table IV minima: IEEE13 bus 684 (phases a,c;
    lines (a,c), (c), (a); no load) -> (m, n) = (4, 8); 1-phase pass-through bus -> (2, 4);
    1-phase line -> (3, 6)."""
    fb = FeederBuilder("684")
    up = fb.bus(PH_A | PH_C)
    b684 = fb.bus(PH_A | PH_C)
    b611, b652 = fb.bus(PH_C), fb.bus(PH_A)
    fb.gen(up, PH_A | PH_C)
    fb.line(up, b684, PH_A | PH_C, np.eye(3) * 0.01, np.eye(3) * 0.02)
    fb.line(b684, b611, PH_C, np.eye(3) * 0.01, np.eye(3) * 0.02)
    fb.line(b684, b652, PH_A, np.eye(3) * 0.01, np.eye(3) * 0.02)
    f = fb.build()
    lp = oracle.assemble_lp(f)
    d = decompose(f, lp)
    s684 = [s for s in range(d.S) if d.kind[s] == BUS and d.comp[s] == b684][0]
    assert (len(d.rows[s684]), len(d.cols[s684])) == (4, 8)
    # 1-phase chain: middle bus is a pass-through bus, lines are 1-phase lines
    f = _tree([0, 1, 2])
    f.load_a[:] = 0.0                       # no voltage-dependent load on the pass-through bus
    f.load_bus[:] = 3
    lp = oracle.assemble_lp(f)
    d = decompose(f, lp)
    mid = [s for s in range(d.S) if d.kind[s] == BUS and d.comp[s] == 1][0]
    assert (len(d.rows[mid]), len(d.cols[mid])) == (2, 4)
    line = [s for s in range(d.S) if d.kind[s] == LINE][0]
    assert (len(d.rows[line]), len(d.cols[line])) == (3, 6)


def test_single_partition_and_orphan():
    f = fx.four_bus()
    lp = oracle.assemble_lp(f)
    d = decompose(f, lp, single=True)
    assert d.S == 1 and d.n_copies == lp.n and np.all(d.nu == 1)       # S = 1: B_1 = I
    # the 1-bus feeder is one group with m_1 = 6, n_1 = 7
    f1 = fx.one_bus_wye()
    d1 = decompose(f1, oracle.assemble_lp(f1))
    assert d1.S == 1 and (len(d1.rows[0]), len(d1.cols[0])) == (6, 7)
    # constant-power load (alpha = beta = 0): w touches no row -> orphan
    g = f1.copy()
    g.load_alpha[:] = 0.0
    g.load_beta[:] = 0.0
    with pytest.raises(DecompositionError, match="orphan"):
        decompose(g, oracle.assemble_lp(g))
