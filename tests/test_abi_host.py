"""C-ABI library without a GPU: it loads, exports every symbol include/lopf.h declares, and its CPU
setup (LP assembly, decomposition, consensus map, Cholesky operators) matches the oracle —
decomposition / maps / LP data bit-exact, operators to 1e-12 (north_star parity bar)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle
from paper_2310_09410_b200 import Lopf, LopfError, load_library
from paper_2310_09410_b200.lopf import STATUS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    lib = load_library()
    header = open(os.path.join(ROOT, "include", "lopf.h")).read()
    names = set(re.findall(r"\b(lopf_[a-z_]+)\s*\(", header))
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert lib.lopf_abi_version() == 3


@pytest.mark.parametrize("make", [lambda: fg.make_feeder("13"), lambda: fg.make_feeder("123"), fx.four_bus,
                                  lambda: fx.two_bus_3ph(fg.DELTA), fx.one_bus_wye, fx.physical])
def test_setup_matches_oracle(make):
    f = make()
    h = Lopf.setup(f)
    p = oracle.build_problem(f)
    s = h.sizes
    assert (s.S, s.n, s.m, s.n_copies) == (p.dec.S, p.lp.n, p.lp.m, p.dec.n_copies)
    d = h.get_decomposition()
    assert np.array_equal(d.kind, p.dec.kind) and np.array_equal(d.comp, p.dec.comp)
    assert np.array_equal(d.leaf_bus, p.dec.leaf_bus)
    assert np.array_equal(d.m_s, p.dec.m_s()) and np.array_equal(d.n_s, p.dec.n_s())
    assert np.array_equal(d.sub_ptr, p.dec.sub_ptr) and np.array_equal(d.copy_global, p.dec.copy_global)
    rp, ci = h.get_consensus()
    assert np.array_equal(rp, p.dec.seg_ptr) and np.array_equal(ci, p.dec.seg_copy)
    g = h.get_globals()
    roles = {"pg": 0, "qg": 1, "w": 2, "pb": 3, "qb": 4, "pd": 5, "qd": 6, "pf": 7, "qf": 8, "pt": 9, "qt": 10}
    assert np.array_equal(g["role"], [roles[v[0]] for v in p.lp.var])
    assert np.array_equal(g["comp"], [v[1] for v in p.lp.var]) and np.array_equal(g["phase"], [v[2] for v in p.lp.var])
    for k in ("c", "lo", "hi"):
        assert np.array_equal(g[k], getattr(p.lp, k))
    for sidx in range(p.dec.S):
        ns = int(d.n_s[sidx])
        A, b = h.get_subsystem(sidx, int(d.m_s[sidx]), ns)
        assert A.shape == p.dec.A[sidx].shape
        assert np.abs(A - p.dec.A[sidx]).max(initial=0) <= 1e-15 and np.abs(b - p.dec.b[sidx]).max(initial=0) <= 1e-15
        ab, bb = h.get_operator(sidx, ns)
        assert np.abs(ab - p.abar[sidx]).max() <= 1e-12
        assert np.abs(bb - p.bbar[sidx]).max(initial=0) <= 1e-12
        assert np.array_equal(ab, ab.T)                              # W^T W - I is exactly symmetric


def test_setup_8500_decomposition_bit_exact():
    f = fg.make_feeder("8500")
    h = Lopf.setup(f)
    lp = oracle.assemble_lp(f)
    dec = oracle.decompose(f, lp)
    d = h.get_decomposition()
    assert d.kind.shape[0] == dec.S == 25001
    assert np.array_equal(d.copy_global, dec.copy_global) and np.array_equal(d.sub_ptr, dec.sub_ptr)
    rp, ci = h.get_consensus()
    assert np.array_equal(rp, dec.seg_ptr) and np.array_equal(ci, dec.seg_copy)
    rng = np.random.default_rng(0)
    from oracle.precompute import precompute
    for sidx in rng.choice(dec.S, 300, replace=False):            # operators on a sample
        ab, bb = h.get_operator(int(sidx), int(d.n_s[sidx]))
        ea, eb = precompute(dec.A[sidx], dec.b[sidx])
        assert np.abs(ab - ea).max() <= 1e-12 and np.abs(bb - eb).max(initial=0) <= 1e-12


def test_single_partition_matches_oracle():
    f = fx.four_bus()
    h = Lopf.setup(f, single=True)
    p = oracle.build_problem(f, single=True)
    d = h.get_decomposition()
    assert d.kind.shape[0] == 1 and np.array_equal(d.copy_global, p.dec.copy_global)
    ab, bb = h.get_operator(0, int(d.n_s[0]))
    assert np.abs(ab - p.abar[0]).max() <= 1e-11 and np.abs(bb - p.bbar[0]).max() <= 1e-11


def _status(exc):
    return STATUS[exc.value.status]


def test_error_behaviour():
    f = fx.four_bus()
    with pytest.raises(LopfError) as e:
        Lopf.setup(f, rho=0.0)
    assert _status(e) == "LOPF_E_ARG"
    with pytest.raises(LopfError) as e:
        Lopf.setup(f, eps_rel=-1.0)
    assert _status(e) == "LOPF_E_ARG"
    g = f.copy(); g.line_to[0] = 99
    with pytest.raises(LopfError) as e:
        Lopf.setup(g)
    assert _status(e) == "LOPF_E_NETWORK" and "dangling" in str(e.value)
    g = f.copy(); g.load_phases[0] = fg.PH_A
    with pytest.raises(LopfError) as e:                              # 1-phase delta load
        Lopf.setup(g)
    assert _status(e) == "LOPF_E_NETWORK"
    g = f.copy(); g.line_tau[1, 0] = 0.0
    with pytest.raises(LopfError) as e:
        Lopf.setup(g)
    assert _status(e) == "LOPF_E_NETWORK" and "tau" in str(e.value)
    g = fx.one_bus_wye(); g.load_alpha[:] = 0; g.load_beta[:] = 0
    with pytest.raises(LopfError) as e:
        Lopf.setup(g)
    assert _status(e) == "LOPF_E_ORPHAN" and "orphan" in str(e.value)
    h = Lopf.setup(f)
    with pytest.raises(LopfError) as e:                              # solve before bind
        h.solve(stream=0)
    assert _status(e) == "LOPF_E_STATE"


def test_sizes_byte_model():
    """alg_bytes follows the DESIGN.md byte model: 8 (P_sym + N_b + 6 N_c + 4 n + n_c) + 4 (2 N_c + n + 1)."""
    f = fg.make_feeder("123")
    h = Lopf.setup(f)
    s = h.sizes
    p = oracle.build_problem(f)
    ns = p.dec.n_s()
    psym = int((ns * (ns + 1) // 2).sum())
    nb = int(sum(ns[i] for i in range(p.dec.S) if np.any(p.dec.b[i] != 0)))
    nobj = int((p.lp.c != 0).sum())
    assert s.p_sym == psym
    assert s.alg_bytes == 8 * (psym + nb + 6 * p.dec.n_copies + 4 * p.lp.n + nobj) + 4 * (2 * p.dec.n_copies + p.lp.n + 1)


def test_kernel_selection():
    """auto picks the SMEM-resident kernel when every chunk fits one CTA's shared memory (all
    three shapes on 148 SMs) and the streaming kernel otherwise (S = 1: n_s > 64)."""
    for shape, g_max in (("13", 4), ("123", 8), ("8500", 148)):
        s = Lopf.setup(fg.make_feeder(shape)).sizes
        assert s.kernel == 2 and 1 <= s.grid <= g_max
    assert Lopf.setup(fx.four_bus(), single=True).sizes.kernel == 1
    assert Lopf.setup(fg.make_feeder("123"), kernel=1).sizes.kernel == 1
    with pytest.raises(LopfError):
        Lopf.setup(fg.make_feeder("8500"), kernel=2, max_ctas=16)        # does not fit 16 CTAs


def test_batch_byte_model():
    """Batch alg_bytes: the operators of subsystems without a load, lo / hi (2 n) and c are
    shared by every scenario and counted once; per scenario its load subsystems' packed A-bar and b-bar,
    the 6 N_c iterate terms and x (write + read, 2 n)."""
    f = fg.make_feeder("123")
    n_scen = 64
    p = oracle.build_problem(f)
    s1 = Lopf.setup(f).sizes
    sb = Lopf.setup_batch(f, fg.scenario_scales(f, n_scen)).sizes
    ns = p.dec.n_s()
    has_load = [bool(np.any(p.dec.b[i] != 0)) for i in range(p.dec.S)]
    psym_var = int(sum(n * (n + 1) // 2 for n, v in zip(ns, has_load) if v))
    nb = int(sum(n for n, v in zip(ns, has_load) if v))
    psym = int((ns * (ns + 1) // 2).sum())
    nobj = int((p.lp.c != 0).sum())
    per_scen = psym_var + nb + 6 * p.dec.n_copies + 2 * p.lp.n
    shared = (psym - psym_var) + 2 * p.lp.n + nobj
    assert sb.alg_bytes == 8 * (shared + n_scen * per_scen) + 4 * (2 * p.dec.n_copies + p.lp.n + 1)
    assert sb.alg_bytes < n_scen * s1.alg_bytes


def test_precision_option():
    """fp32 variant (reading F1): every kernel has an fp32 layout with half the (T) bytes of the byte model
    and a smaller arena; an unknown precision is LOPF_E_ARG."""
    f = fg.make_feeder("123")
    for kernel in (1, 2):
        s64 = Lopf.setup(f, kernel=kernel).sizes
        s32 = Lopf.setup(f, kernel=kernel, precision=32).sizes
        assert s32.kernel == s64.kernel == kernel and s32.device_bytes < s64.device_bytes
        int_bytes = 4 * (2 * s64.n_copies + s64.n + 1)
        assert (s32.alg_bytes - int_bytes) * 2 == s64.alg_bytes - int_bytes
    with pytest.raises(Exception):
        Lopf.setup(f, precision=16)


def test_block_threads_must_be_zero():
    """lopf_options.block_threads is fixed per kernel at build time: a nonzero value is LOPF_E_ARG."""
    import ctypes as C
    from paper_2310_09410_b200 import lopf as L
    lib = L.load_library()
    o = L.Options()
    lib.lopf_options_default(C.byref(o))
    o.block_threads = 256
    net, keep = L._network(fg.make_feeder("13"))
    h = C.c_void_p()
    assert lib.lopf_setup(C.byref(net), C.byref(o), C.byref(h)) == 1          # LOPF_E_ARG
    assert b"block_threads" in lib.lopf_last_error()
