"""Residual balancing on the GPU (reading F2): the streaming kernel with
the on-device rho update against the oracle's adaptive loop (oracle.solve_adaptive, pinned in
test_oracle_adaptive.py) on the same seeded inputs -- the rho in force and the number of changes equal,
iterates after fixed K within 1e-9 relative, iteration count to (termination) bit-exact, objective 1e-6."""
import numpy as np
import pytest

import feedergen as fg
import fixtures as fx
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


@pytest.mark.parametrize("every", [1, 10])
@pytest.mark.parametrize("make", [lambda: fg.make_feeder("13"), lambda: fg.make_feeder("123"), fx.physical],
                         ids=["13", "123", "physical"])
def test_adaptive_fixed_k_and_solve(torch_cuda, make, every):
    from paper_2310_09410_b200 import CONVERGED, Lopf
    f = make()
    p = oracle.build_problem(f)
    h = Lopf.setup(f, adapt_every=every).bind("cuda")
    assert h.sizes.kernel == 1                                        # auto picks the streaming kernel
    for k in (7, 300):
        h.reset()
        h.run(k)
        o, rho, n = oracle.solve_adaptive(p, every=every, max_iter=k, test=False)
        assert h.get_rho() == (rho, n)
        x, xl, lam = h.get_state()
        assert _rel(x, o.x) <= TOL and _rel(xl, o.x_loc) <= TOL and _rel(lam, o.lam) <= TOL, k
    h.reset()
    r = h.solve()
    o, rho, n = oracle.solve_adaptive(p, every=every)
    assert r.outcome == CONVERGED and o.converged
    assert r.iters == o.iters and h.get_rho() == (rho, n)
    assert abs(r.objective - o.objective) <= 1e-6 * abs(o.objective)


def test_adaptive_rejected_where_unsupported(torch_cuda):
    from paper_2310_09410_b200 import Lopf, LopfError
    f = fg.make_feeder("13")
    with pytest.raises(LopfError):
        Lopf.setup(f, adapt_every=10, kernel=2)
    with pytest.raises(LopfError):
        Lopf.setup(f, adapt_every=10, adapt_mu=0.5)                    # mu must exceed 1
