"""The seeded input generator: determinism, validity and the paper's instance shapes."""
import numpy as np
import pytest

import feedergen as fg
from feedergen import phase_list


@pytest.mark.parametrize("shape", ["13", "123", "8500"])
def test_deterministic_and_valid(shape):
    f, g = fg.make_feeder(shape), fg.make_feeder(shape)
    assert f.sha256() == g.sha256()
    assert fg.make_feeder(shape, seed=999).sha256() != f.sha256()
    assert f.n_line == f.n_bus - 1                                   # radial
    par = {}
    for e in range(f.n_line):                                        # tree rooted at root_bus
        par[int(f.line_to[e])] = int(f.line_from[e])
        pl = set(phase_list(f.line_phases[e]))
        assert pl <= set(phase_list(f.bus_phases[f.line_from[e]])) and pl <= set(phase_list(f.bus_phases[f.line_to[e]]))
    for b in range(f.n_bus):
        seen, x = set(), b
        while x != f.root_bus:
            assert x not in seen
            seen.add(x)
            x = par[x]
    for l in range(f.n_load):
        assert set(phase_list(f.load_phases[l])) <= set(phase_list(f.bus_phases[f.load_bus[l]]))
        if f.load_conn[l] == fg.DELTA:
            assert f.load_phases[l] == fg.ALL3
    assert np.all(f.bus_wmin <= f.bus_wmax) and np.all(f.load_alpha >= 0) and np.all(f.load_beta >= 0)


def test_text_roundtrip_and_unknown_keys():
    f = fg.make_feeder("13")
    assert fg.from_text(f.to_text()).sha256() == f.sha256()
    with pytest.raises(ValueError, match="unknown key"):
        fg.from_text("bus id=0 phases=a wmin=0,0,0 wmax=0,0,0 gsh=0,0,0 bsh=0,0,0 color=red\n")


def test_8500_shape_counts():
    """N3 = 1566, N1 = 11545, 1222 leaves -> 13112 nodes; S = 25001."""
    st = fg.graph_stats(fg.make_feeder("8500"))
    assert st == dict(nodes=13112, lines=13111, leaves=1222, load_phases=1222)


def test_scenario_scales():
    f = fg.make_feeder("123")
    k = fg.scenario_scales(f, 8)
    assert k.shape == (8, f.n_load) and k.min() >= 0.5 and k.max() <= 1.5
    g = fg.scale_loads(f, k[3])
    assert np.allclose(g.load_a, f.load_a * k[3][:, None])
