"""Tiny hand-built feeders (each cites the example it reproduces)."""
import numpy as np

from feedergen import ALL3, DELTA, PH_A, PH_B, PH_C, WYE, FeederBuilder

R3 = np.array([[0.010, 0.004, 0.004], [0.004, 0.010, 0.004], [0.004, 0.004, 0.010]])
X3 = np.array([[0.030, 0.012, 0.012], [0.012, 0.030, 0.012], [0.012, 0.012, 0.030]])


def one_bus_wye():
    """1 bus, 1 single-phase wye load, 1 single-phase generator, no lines:
    n = 7 (pg, qg, w, pb, qb, pd, qd), m = 6 (2 balance + 2 VDLM defs + 2 wye couplings)."""
    fb = FeederBuilder("spec-1bus")
    b = fb.bus(PH_A, 0.9, 1.1)
    fb.gen(b, PH_A, 0.0, 1.0, -1.0, 1.0)
    fb.load(b, PH_A, WYE, alpha=[1, 0, 0], beta=[2, 0, 0], a=[0.5, 0, 0], b=[0.2, 0, 0])
    return fb.build()


def two_bus_line():
    """two buses, one three-phase line, no loads/generators: m = 2*2*3 + 3*3 = 21."""
    fb = FeederBuilder("spec-2bus")
    b0 = fb.bus(ALL3)
    b1 = fb.bus(ALL3)
    fb.line(b0, b1, ALL3, R3, X3)
    return fb.build()


def chain_1ph(n_bus=3, alpha=1.0, beta=2.0):
    """1-phase chain root -> 1 -> ... with a wye load (alpha, beta > 0) on every non-root bus and
    one substation generator: the LP has a unique vertex (reading C19)."""
    fb = FeederBuilder(f"chain{n_bus}")
    prev = fb.bus(PH_A, 0.9025, 1.1025)
    fb.gen(prev, PH_A, -10, 10, -10, 10)
    rng = np.random.default_rng(n_bus)
    for k in range(1, n_bus):
        b = fb.bus(PH_A, 0.81, 1.21)
        r = rng.uniform(0.01, 0.03)
        fb.line(prev, b, PH_A, np.eye(3) * r, np.eye(3) * 2.5 * r)
        a = rng.uniform(0.2, 0.6)
        fb.load(b, PH_A, WYE, [alpha, 0, 0], [beta, 0, 0], [a, 0, 0], [0.4 * a, 0, 0])
        prev = b
    return fb.build()


def two_bus_3ph(conn=WYE, shunts=True):
    """3-phase root (generator) -> 3-phase line -> bus with one 3-phase load (alpha, beta = 1..2)."""
    fb = FeederBuilder(f"2bus3ph-{'delta' if conn else 'wye'}")
    b0 = fb.bus(ALL3, 0.9025, 1.1025)
    fb.gen(b0, ALL3, -10, 10, -10, 10)
    b1 = fb.bus(ALL3, 0.81, 1.21, bsh=(0.01, 0.0, 0.02) if shunts else (0, 0, 0))
    bs = np.array([1e-3, 2e-3, 1.5e-3]) if shunts else np.zeros(3)
    fb.line(b0, b1, ALL3, R3 * 3, X3 * 3, bs_from=bs, bs_to=bs / 2)
    fb.load(b1, ALL3, conn, alpha=[1, 2, 1], beta=[2, 1, 2], a=[0.5, 0.3, 0.4], b=[0.2, 0.15, 0.1])
    return fb.build()


def four_bus():
    """synthetic 4-bus feeder: 4 buses, 3 lines, 2 wye + 1 delta load."""
    fb = FeederBuilder("spec-4bus")
    b0 = fb.bus(ALL3, 0.9025, 1.1025)
    fb.gen(b0, ALL3, -10, 10, -10, 10)
    b1 = fb.bus(ALL3)
    b2 = fb.bus(ALL3, bsh=(0.02, 0.02, 0.02))
    b3 = fb.bus(PH_A)
    fb.line(b0, b1, ALL3, R3, X3, bs_from=[1e-4] * 3, bs_to=[1e-4] * 3)
    fb.line(b1, b2, ALL3, R3 * 2, X3 * 2)
    fb.line(b1, b3, PH_A, np.eye(3) * 0.02, np.eye(3) * 0.05)
    fb.load(b2, ALL3, DELTA, alpha=[1, 1, 2], beta=[2, 2, 1], a=[0.3, 0.2, 0.25], b=[0.1, 0.1, 0.05])
    fb.load(b2, ALL3, WYE, alpha=[2, 0, 1], beta=[2, 1, 0], a=[0.1, 0.15, 0.12], b=[0.05, 0.04, 0.03])
    fb.load(b3, PH_A, WYE, alpha=[1, 0, 0], beta=[1, 0, 0], a=[0.2, 0, 0], b=[0.08, 0, 0])
    return fb.build()


def physical():
    """Every input class of Table I in one small radial feeder, used by the
    physically-consistent-point pin (tests/test_oracle_physics.py) and by the library/GPU parity tests:
    * a zero-impedance 3-phase regulator line with tap tau = 1.02 (the tau of (5c));
    * a 3-phase line with nonzero g^s and b^s at both ends ((5a)-(5c));
    * shunt conductance g^sh and capacitors b^sh on buses ((3));
    * a 3-phase delta load and 3-phase / 2-phase / 1-phase wye loads, alpha, beta in {0, 1, 2};
    * a 2-phase {a,c} line into a 2-phase bus with no load and three incident lines — the IEEE13
      bus-684 pattern of Table IV's minimum (m_s, n_s) = (4, 8);
    * a 2-phase {a,b} lateral, and a 1-phase pass-through bus whose only reason to own its w is g^sh
      (the column rule C11)."""
    fb = FeederBuilder("physical")
    r3 = np.array([[0.012, 0.004, 0.005], [0.004, 0.011, 0.0045], [0.005, 0.0045, 0.013]])
    x3 = np.array([[0.031, 0.013, 0.011], [0.013, 0.029, 0.012], [0.011, 0.012, 0.033]])
    b0 = fb.bus(ALL3, 0.9025, 1.1025)                                       # 0 substation
    fb.gen(b0, ALL3, -10, 10, -10, 10)
    b1 = fb.bus(ALL3, gsh=(0.002, 0.0, 0.001), bsh=(0.010, 0.012, 0.008))   # 1 capacitor + g^sh
    fb.line(b0, b1, ALL3, np.zeros((3, 3)), np.zeros((3, 3)), tau=(1.02, 1.02, 1.02))   # regulator
    b2 = fb.bus(ALL3)                                                       # 2 delta + wye loads
    fb.line(b1, b2, ALL3, r3, x3, gs_from=(2e-4, 1e-4, 3e-4), bs_from=(1e-3, 2e-3, 1.5e-3),
            gs_to=(1e-4, 2e-4, 1e-4), bs_to=(5e-4, 1e-3, 8e-4))
    fb.load(b2, ALL3, DELTA, alpha=[1, 2, 0], beta=[2, 1, 2], a=[0.12, 0.10, 0.08], b=[0.05, 0.04, 0.03])
    fb.load(b2, ALL3, WYE, alpha=[2, 0, 1], beta=[0, 1, 2], a=[0.05, 0.06, 0.04], b=[0.02, 0.03, 0.01])
    b3 = fb.bus(PH_A | PH_C)                                                # 3 (a,c), no load: (4, 8)
    fb.line(b2, b3, PH_A | PH_C, r3 * 1.5, x3 * 1.5, gs_from=(1e-4, 0, 1e-4), bs_from=(2e-4, 0, 2e-4))
    b4 = fb.bus(PH_C)                                                       # 4 leaf, 1-phase load
    fb.line(b3, b4, PH_C, np.eye(3) * 0.02, np.eye(3) * 0.05)
    fb.load(b4, PH_C, WYE, alpha=[0, 0, 1], beta=[0, 0, 1], a=[0, 0, 0.07], b=[0, 0, 0.03])
    b5 = fb.bus(PH_A, gsh=(0.003, 0, 0))                                    # 5 leaf, constant-power load
    fb.line(b3, b5, PH_A, np.eye(3) * 0.025, np.eye(3) * 0.06)
    fb.load(b5, PH_A, WYE, alpha=[0, 0, 0], beta=[0, 0, 0], a=[0.05, 0, 0], b=[0.02, 0, 0])
    b6 = fb.bus(PH_A | PH_B, bsh=(0.004, 0.005, 0))                          # 6 (a,b) lateral, 2-phase load
    fb.line(b1, b6, PH_A | PH_B, r3 * 2, x3 * 2, bs_from=(3e-4, 3e-4, 0), bs_to=(3e-4, 3e-4, 0))
    fb.load(b6, PH_A | PH_B, WYE, alpha=[1, 2, 0], beta=[2, 2, 0], a=[0.04, 0.05, 0], b=[0.015, 0.02, 0])
    b7 = fb.bus(PH_B, gsh=(0, 0.002, 0))                                    # 7 pass-through, w only via g^sh
    fb.line(b6, b7, PH_B, np.eye(3) * 0.03, np.eye(3) * 0.07)
    b8 = fb.bus(PH_B)                                                       # 8 leaf, 1-phase load
    fb.line(b7, b8, PH_B, np.eye(3) * 0.02, np.eye(3) * 0.04)
    fb.load(b8, PH_B, WYE, alpha=[0, 1, 0], beta=[0, 2, 0], a=[0, 0.03, 0], b=[0, 0.012, 0])
    return fb.build()
