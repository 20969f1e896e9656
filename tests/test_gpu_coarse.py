"""f4 on the GPU: the IEEE37-shaped delta-only feeder and coarse partitions (reading
C25) through the C-ABI against the oracle -- fixed-K iterates within 1e-9 relative, K to (termination)
bit-exact, objective 1e-6.  Coarse subsystems with n_s > 63 take the streaming kernel's full-task path
(Abar as column tiles of 32 R rows, R = 2 / 4 / 8)."""
import json
import os

import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-9
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json")))["configs"]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def _check(h, ref):
    x, xl, lam = h.get_state()
    assert _rel(x, ref.x) <= TOL and _rel(xl, ref.x_loc) <= TOL and _rel(lam, ref.lam) <= TOL


@pytest.mark.parametrize("kernel", [1, 2])
def test_delta37(torch_cuda, kernel):
    from paper_2310_09410_b200 import CONVERGED, Lopf
    f = fg.make_feeder("37")
    g = GOLD["37"]
    assert f.sha256() == g["sha256"]
    p = oracle.build_problem(f)
    h = Lopf.setup(f, kernel=kernel).bind("cuda")
    done = 0
    for k in (1, 10, 300):
        h.run(k - done)
        done = k
        _check(h, oracle.run_k(p, k))
    h.reset()
    r = h.solve()
    assert r.outcome == CONVERGED and r.iters == g["iters"]
    assert abs(r.objective - g["objective"]) <= 1e-6 * abs(g["objective"])


@pytest.mark.parametrize("make,B,kernel", [(lambda: fg.make_feeder("123"), 4, 2), (lambda: fg.make_feeder("123"), 4, 1),
                                           (lambda: fg.make_feeder("123"), 16, 0), (lambda: fg.make_feeder("37"), 8, 0),
                                           (fx.physical, 16, 0)],
                         ids=["123-B4-resident", "123-B4-streaming", "123-B16", "37-B8", "physical-B16 (S=1)"])
def test_coarse(torch_cuda, make, B, kernel):
    from paper_2310_09410_b200 import CONVERGED, Lopf
    f = make()
    p = oracle.build_problem(f, coarse=B)
    h = Lopf.setup(f, coarse=B, kernel=kernel).bind("cuda")
    if kernel:
        assert h.sizes.kernel == kernel
    assert h.sizes.S == p.dec.S
    h.run(300)
    _check(h, oracle.run_k(p, 300))
    h.reset()
    r = h.solve()
    o = oracle.solve(p)
    assert r.outcome == CONVERGED and o.converged
    assert r.iters == o.iters and abs(r.objective - o.objective) <= 1e-6 * abs(o.objective)


def test_coarse_fp32(torch_cuda):
    """Coarse runs in the fp32 variant against the oracle's binary32 loop on the same coarse decomposition,
    within twice the forward-error bound K (n_max + nu_max + 4) 2^-24 (as tests/test_gpu_f32.py)."""
    from paper_2310_09410_b200 import Lopf
    f = fg.make_feeder("123")
    p = oracle.build_problem(f, coarse=16)
    h = Lopf.setup(f, coarse=16, precision=32).bind("cuda")
    h.run(100)
    ref = oracle.run_k_f32(p, 100)
    tol = 2.0 * 100 * (int(p.dec.n_s().max()) + int(np.diff(p.dec.seg_ptr).max()) + 4) * 2.0 ** -24
    x, xl, lam = h.get_state()
    assert _rel(x, ref.x) <= tol and _rel(xl, ref.x_loc) <= tol and _rel(lam / 100.0, ref.lam / 100.0) <= tol
