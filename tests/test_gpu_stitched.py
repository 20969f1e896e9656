"""Config 5 family (BASELINE.json configs[4]): feeders stitched from several subfeeders onto a trunk
(feedergen.make_stitched).  Oracle parity on the small members (4 x 13-shaped, 2 x 8500-shaped: several
hundred tiles, ragged tails, the trunk's high-degree buses), and at the full 64 x 8500 size the
properties that hold at any size: bounds, run-to-run / grid-size bit-determinism, the ADMM-3 identity
and agreement of the two consensus inputs.  Bars as in test_gpu_parity.py."""
import json
import os

import numpy as np
import pytest

import feedergen as fg
import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json")))["configs"]
TOL = 1e-9


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


_cache = {}


def _problem(key):
    if key not in _cache:
        f = fg.make_stitched(4, "13") if key == "s4x13" else fg.make_stitched(2, "8500")
        _cache[key] = (f, oracle.build_problem(f))
    return _cache[key]


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def _solver(f, **kw):
    from paper_2310_09410_b200 import Lopf
    return Lopf.setup(f, **kw).bind("cuda")


@pytest.mark.parametrize("key,ks,kernel", [("s4x13", (1, 10, 1000), 1), ("s4x13", (1, 10, 1000), 2),
                                           ("s2x8500", (1, 10, 100), 1)])   # 2 x 8500 exceeds the SMEM of 148 CTAs
def test_stitched_fixed_k_and_k_to_tolerance(torch_cuda, key, ks, kernel):
    f, p = _problem(key)
    g = GOLD[key]
    assert f.sha256() == g["sha256"]
    h = _solver(f, kernel=kernel)
    done = 0
    for k in ks:
        h.run(k - done)
        done = k
        ref = oracle.run_k(p, k)
        x, xl, lam = h.get_state()
        assert _rel(x, ref.x) <= TOL and _rel(xl, ref.x_loc) <= TOL and _rel(lam, ref.lam) <= TOL
    h.reset()
    r = h.solve()
    assert r.iters == g["iters"], (r.iters, g["iters"])
    assert abs(r.objective - g["objective"]) <= 1e-6 * abs(g["objective"])


@pytest.fixture(scope="module")
def full_instance(torch_cuda):
    f = fg.make_stitched(64, "8500")
    return f


def test_full_64x8500_properties(full_instance):
    """The bench's config-5 instance and launch configuration (streaming kernel, whole GPU)."""
    f = full_instance
    h = _solver(f)
    s = h.sizes
    assert s.kernel == 1 and s.S > 1_500_000 and s.n_copies > 10_000_000
    rp, ci = h.get_consensus()
    dec = h.get_decomposition()
    gl = h.get_globals()
    assert rp[-1] == s.n_copies and np.all(np.diff(rp) >= 1)              # every global has a copy
    assert np.array_equal(np.sort(ci), np.arange(s.n_copies))
    assert np.all(dec.copy_global[ci] == np.repeat(np.arange(s.n), np.diff(rp)))
    h.run(20)
    x0, xl0, lam0 = h.get_state()
    h.run(1)
    x1, xl1, lam1 = h.get_state()
    # ADMM-3 at sweep 21: lambda' = lambda + rho (x[I(j)] - x_s) per copy
    rho = 100.0
    v = x1[dec.copy_global]
    assert np.allclose(lam1, lam0 + rho * (v - xl1), rtol=0, atol=1e-9 * max(1.0, np.abs(lam1).max()))
    assert np.all(x1 >= gl["lo"]) and np.all(x1 <= gl["hi"])                # closed_1 clamp
    # closed_1 at sweep 21 from the sweep-20 copies (reading C1)
    u = xl0 - lam0 / rho
    sig = np.add.reduceat(u[ci], rp[:-1])
    nu = np.diff(rp)
    xr = np.minimum(np.maximum((sig - gl["c"] / rho) / nu, gl["lo"]), gl["hi"])
    assert _rel(x1, xr) <= 1e-12
    # bit-determinism: reset + rerun, and a smaller grid
    h.reset()
    h.run(21)
    assert all(np.array_equal(a, b) for a, b in zip(h.get_state(), (x1, xl1, lam1)))
    h2 = _solver(f, grid_cap=37)
    h2.run(21)
    for a, b in zip(h2.get_state(), (x1, xl1, lam1)):
        assert np.array_equal(a, b)                                         # per-copy arithmetic is grid-independent


def test_stitched_8x8500_oracle_k100_and_partitions():
    """SURVEY §8(c) parity matrix, config 5: an 8 x 8500 stitched instance (1.32M copies) after K = 100
    sweeps -- the streaming kernel against the oracle (1e-9 relative), and the partitioned mode with the
    device-initiated exchange (2 and 4 ranks emulated in one launch) bit-identical to the streaming kernel."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_09410_b200 import Lopf
    from paper_2310_09410_b200.partition import merge_owned
    f = fg.make_stitched(8, "8500")
    p = oracle.build_problem(f)
    ref = oracle.run_k(p, 100)
    h = Lopf.setup(f, kernel=1).bind("cuda")
    h.run(100)
    single = h.get_state()
    for a, b in zip(single, (ref.x, ref.x_loc, ref.lam)):
        assert float(np.abs(a - b).max() / max(1.0, np.abs(b).max())) <= 1e-9
    for world in (2, 4):
        hs = [Lopf.setup_part(f, r, world, bus_owner=fg.stitched_bus_owner(f, world)).bind("cuda") for r in range(world)]
        for x in hs:
            x.reset()
        Lopf.part_emulate(hs, 100, test=False)
        parts = [x.get_state() for x in hs]
        for i in range(3):
            assert np.array_equal(merge_owned([q[i] for q in parts]), single[i]), (world, i)
