"""Seeded synthetic radial feeders shaped like the paper's IEEE 13/123/8500 instances.

This module is the ONLY code shared by the oracle (`oracle/`) and the CUDA path
(`paper_2310_09410_b200/`): it produces network *data* (Table I records) and
holds none of the method's arithmetic (no LP rows, no decomposition, no ADMM).

Data model (Table I "Nomenclature"), structure-of-arrays,
phase slots [3] = phases a, b, c (1, 2, 3 in the paper's notation):

* buses      phases (bitmask: a=1, b=2, c=4), w bounds, shunts g^sh, b^sh
* lines      from/to, phases, 3x3 r and x (row-major [9]), from/to shunts
             g^s, b^s, tap tau, flow bounds
* generators bus, phases, p^g / q^g bounds
* loads      bus, phases, connection (0 wye, 1 delta), alpha, beta, a, b
             

Values for absent phases are 0 and never read.  The recipe for each shape
 follows SURVEY.md Appendix B / §8(d): a radial
3-phase primary with 1-phase chain laterals, voltage-dependent wye/delta loads
(alpha, beta in {0,1,2} = constant P/I/Z), capacitors, one
regulator tap, all drawn from numpy.random.default_rng(seed).
"""
from __future__ import annotations

import dataclasses
import hashlib
from dataclasses import dataclass, field

import numpy as np

PH_A, PH_B, PH_C = 1, 2, 4
ALL3 = PH_A | PH_B | PH_C
WYE, DELTA = 0, 1
INF = float("inf")


def phase_list(mask: int) -> list[int]:
    """Phase slots (0=a, 1=b, 2=c) present in a bitmask, ascending."""
    return [p for p in range(3) if (int(mask) >> p) & 1]


def _mask_str(mask: int) -> str:
    return "".join("abc"[p] for p in phase_list(mask))


def _mask_parse(s: str) -> int:
    m = 0
    for ch in s:
        m |= 1 << "abc".index(ch)
    return m


@dataclass
class Feeder:
    """A feeder in structure-of-arrays form (the `lopf_network` layout of include/lopf.h)."""

    name: str
    root_bus: int
    bus_phases: np.ndarray            # uint8 [n_bus]
    bus_wmin: np.ndarray              # f64 [n_bus,3]
    bus_wmax: np.ndarray
    bus_gsh: np.ndarray
    bus_bsh: np.ndarray
    line_from: np.ndarray             # int32 [n_line]
    line_to: np.ndarray
    line_phases: np.ndarray           # uint8 [n_line]
    line_r: np.ndarray                # f64 [n_line,9] row-major 3x3
    line_x: np.ndarray
    line_gs_from: np.ndarray          # f64 [n_line,3]
    line_bs_from: np.ndarray
    line_gs_to: np.ndarray
    line_bs_to: np.ndarray
    line_tau: np.ndarray
    line_pmin: np.ndarray
    line_pmax: np.ndarray
    line_qmin: np.ndarray
    line_qmax: np.ndarray
    gen_bus: np.ndarray               # int32 [n_gen]
    gen_phases: np.ndarray            # uint8
    gen_pmin: np.ndarray              # f64 [n_gen,3]
    gen_pmax: np.ndarray
    gen_qmin: np.ndarray
    gen_qmax: np.ndarray
    load_bus: np.ndarray              # int32 [n_load]
    load_phases: np.ndarray           # uint8
    load_conn: np.ndarray             # uint8 (0 wye, 1 delta)
    load_alpha: np.ndarray            # f64 [n_load,3]
    load_beta: np.ndarray
    load_a: np.ndarray
    load_b: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def n_bus(self) -> int:
        return int(self.bus_phases.shape[0])

    @property
    def n_line(self) -> int:
        return int(self.line_phases.shape[0])

    @property
    def n_gen(self) -> int:
        return int(self.gen_phases.shape[0])

    @property
    def n_load(self) -> int:
        return int(self.load_phases.shape[0])

    def copy(self) -> "Feeder":
        kw = {}
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            kw[f.name] = v.copy() if isinstance(v, np.ndarray) else (dict(v) if isinstance(v, dict) else v)
        return Feeder(**kw)

    # ---- canonical text form ("line-oriented records") -------------
    def to_text(self) -> str:
        f3 = lambda a: ",".join(repr(float(v)) for v in a)  # noqa: E731  (repr round-trips fp64 exactly)
        out = ["# lopf feeder v1", f"feeder name={self.name} root={self.root_bus}"]
        for i in range(self.n_bus):
            out.append(f"bus id={i} phases={_mask_str(self.bus_phases[i])} wmin={f3(self.bus_wmin[i])} "
                       f"wmax={f3(self.bus_wmax[i])} gsh={f3(self.bus_gsh[i])} bsh={f3(self.bus_bsh[i])}")
        for e in range(self.n_line):
            out.append(f"line id={e} from={self.line_from[e]} to={self.line_to[e]} "
                       f"phases={_mask_str(self.line_phases[e])} r={f3(self.line_r[e])} x={f3(self.line_x[e])} "
                       f"gs_from={f3(self.line_gs_from[e])} bs_from={f3(self.line_bs_from[e])} "
                       f"gs_to={f3(self.line_gs_to[e])} bs_to={f3(self.line_bs_to[e])} tau={f3(self.line_tau[e])} "
                       f"pmin={f3(self.line_pmin[e])} pmax={f3(self.line_pmax[e])} "
                       f"qmin={f3(self.line_qmin[e])} qmax={f3(self.line_qmax[e])}")
        for k in range(self.n_gen):
            out.append(f"gen id={k} bus={self.gen_bus[k]} phases={_mask_str(self.gen_phases[k])} "
                       f"pmin={f3(self.gen_pmin[k])} pmax={f3(self.gen_pmax[k])} "
                       f"qmin={f3(self.gen_qmin[k])} qmax={f3(self.gen_qmax[k])}")
        for l in range(self.n_load):
            out.append(f"load id={l} bus={self.load_bus[l]} phases={_mask_str(self.load_phases[l])} "
                       f"conn={'delta' if self.load_conn[l] else 'wye'} alpha={f3(self.load_alpha[l])} "
                       f"beta={f3(self.load_beta[l])} a={f3(self.load_a[l])} b={f3(self.load_b[l])}")
        return "\n".join(out) + "\n"

    def sha256(self) -> str:
        return hashlib.sha256(self.to_text().encode()).hexdigest()


_BUS_KEYS = {"id", "phases", "wmin", "wmax", "gsh", "bsh"}
_LINE_KEYS = {"id", "from", "to", "phases", "r", "x", "gs_from", "bs_from", "gs_to", "bs_to", "tau",
              "pmin", "pmax", "qmin", "qmax"}
_GEN_KEYS = {"id", "bus", "phases", "pmin", "pmax", "qmin", "qmax"}
_LOAD_KEYS = {"id", "bus", "phases", "conn", "alpha", "beta", "a", "b"}


def from_text(text: str) -> Feeder:
    """Parse the canonical text form; unknown keys or record kinds raise ValueError."""
    recs: dict[str, list[dict]] = {"bus": [], "line": [], "gen": [], "load": []}
    name, root = "feeder", 0
    for lineno, raw in enumerate(text.splitlines(), 1):
        s = raw.strip()
        if not s or s.startswith("#"):
            continue
        kind, *kvs = s.split()
        d = {}
        for kv in kvs:
            if "=" not in kv:
                raise ValueError(f"line {lineno}: malformed field {kv!r}")
            k, v = kv.split("=", 1)
            d[k] = v
        if kind == "feeder":
            name, root = d.get("name", "feeder"), int(d.get("root", 0))
            continue
        allowed = {"bus": _BUS_KEYS, "line": _LINE_KEYS, "gen": _GEN_KEYS, "load": _LOAD_KEYS}.get(kind)
        if allowed is None:
            raise ValueError(f"line {lineno}: unknown record kind {kind!r}")
        bad = set(d) - allowed
        if bad:
            raise ValueError(f"line {lineno}: unknown key(s) {sorted(bad)} in {kind} record")
        recs[kind].append(d)

    def vec(d, key, n):
        v = [float(t) for t in d[key].split(",")]
        if len(v) != n:
            raise ValueError(f"{key}: expected {n} values, got {len(v)}")
        return v

    B, L, G, D = recs["bus"], recs["line"], recs["gen"], recs["load"]
    arr = lambda rows, key, n: np.array([vec(r, key, n) for r in rows], dtype=np.float64).reshape(len(rows), n)  # noqa
    return Feeder(
        name=name, root_bus=root,
        bus_phases=np.array([_mask_parse(r["phases"]) for r in B], dtype=np.uint8),
        bus_wmin=arr(B, "wmin", 3), bus_wmax=arr(B, "wmax", 3), bus_gsh=arr(B, "gsh", 3), bus_bsh=arr(B, "bsh", 3),
        line_from=np.array([int(r["from"]) for r in L], dtype=np.int32),
        line_to=np.array([int(r["to"]) for r in L], dtype=np.int32),
        line_phases=np.array([_mask_parse(r["phases"]) for r in L], dtype=np.uint8),
        line_r=arr(L, "r", 9), line_x=arr(L, "x", 9),
        line_gs_from=arr(L, "gs_from", 3), line_bs_from=arr(L, "bs_from", 3),
        line_gs_to=arr(L, "gs_to", 3), line_bs_to=arr(L, "bs_to", 3), line_tau=arr(L, "tau", 3),
        line_pmin=arr(L, "pmin", 3), line_pmax=arr(L, "pmax", 3),
        line_qmin=arr(L, "qmin", 3), line_qmax=arr(L, "qmax", 3),
        gen_bus=np.array([int(r["bus"]) for r in G], dtype=np.int32),
        gen_phases=np.array([_mask_parse(r["phases"]) for r in G], dtype=np.uint8),
        gen_pmin=arr(G, "pmin", 3), gen_pmax=arr(G, "pmax", 3), gen_qmin=arr(G, "qmin", 3), gen_qmax=arr(G, "qmax", 3),
        load_bus=np.array([int(r["bus"]) for r in D], dtype=np.int32),
        load_phases=np.array([_mask_parse(r["phases"]) for r in D], dtype=np.uint8),
        load_conn=np.array([1 if r["conn"] == "delta" else 0 for r in D], dtype=np.uint8),
        load_alpha=arr(D, "alpha", 3), load_beta=arr(D, "beta", 3), load_a=arr(D, "a", 3), load_b=arr(D, "b", 3),
    )


# ----------------------------------------------------------------------------------------------
# Builder used by the generator and by hand-written fixtures
# ----------------------------------------------------------------------------------------------
class FeederBuilder:
    """Incremental construction of a Feeder (all per-phase arrays zero for absent phases)."""

    def __init__(self, name: str):
        self.name = name
        self.root = 0
        self.buses: list[dict] = []
        self.lines: list[dict] = []
        self.gens: list[dict] = []
        self.loads: list[dict] = []

    def bus(self, phases: int, wmin=0.81, wmax=1.21, gsh=(0, 0, 0), bsh=(0, 0, 0)) -> int:
        pl = phase_list(phases)
        z = lambda v: [float(v[p]) if p in pl else 0.0 for p in range(3)]  # noqa: E731
        wl = [float(wmin) if p in pl else 0.0 for p in range(3)]
        wh = [float(wmax) if p in pl else 0.0 for p in range(3)]
        self.buses.append(dict(phases=phases, wmin=wl, wmax=wh, gsh=z(gsh), bsh=z(bsh)))
        return len(self.buses) - 1

    def line(self, f: int, t: int, phases: int, r, x, gs_from=(0, 0, 0), bs_from=(0, 0, 0),
             gs_to=(0, 0, 0), bs_to=(0, 0, 0), tau=(1, 1, 1), fmin=-10.0, fmax=10.0) -> int:
        pl = phase_list(phases)
        r = np.asarray(r, dtype=np.float64).reshape(3, 3)
        x = np.asarray(x, dtype=np.float64).reshape(3, 3)
        keep = np.zeros((3, 3))
        for p in pl:
            for q in pl:
                keep[p, q] = 1.0
        z = lambda v: [float(v[p]) if p in pl else 0.0 for p in range(3)]  # noqa: E731
        lo = [float(fmin) if p in pl else 0.0 for p in range(3)]
        hi = [float(fmax) if p in pl else 0.0 for p in range(3)]
        self.lines.append(dict(f=f, t=t, phases=phases, r=(r * keep).ravel().tolist(), x=(x * keep).ravel().tolist(),
                               gs_from=z(gs_from), bs_from=z(bs_from), gs_to=z(gs_to), bs_to=z(bs_to), tau=z(tau),
                               pmin=lo, pmax=hi, qmin=list(lo), qmax=list(hi)))
        return len(self.lines) - 1

    def gen(self, bus: int, phases: int, pmin=-10.0, pmax=10.0, qmin=-10.0, qmax=10.0) -> int:
        pl = phase_list(phases)
        v = lambda s: [float(s) if p in pl else 0.0 for p in range(3)]  # noqa: E731
        self.gens.append(dict(bus=bus, phases=phases, pmin=v(pmin), pmax=v(pmax), qmin=v(qmin), qmax=v(qmax)))
        return len(self.gens) - 1

    def load(self, bus: int, phases: int, conn: int, alpha, beta, a, b) -> int:
        pl = phase_list(phases)
        z = lambda v: [float(v[p]) if p in pl else 0.0 for p in range(3)]  # noqa: E731
        self.loads.append(dict(bus=bus, phases=phases, conn=conn, alpha=z(alpha), beta=z(beta), a=z(a), b=z(b)))
        return len(self.loads) - 1

    def build(self) -> Feeder:
        B, L, G, D = self.buses, self.lines, self.gens, self.loads
        a = lambda rows, k, n: np.array([r[k] for r in rows], dtype=np.float64).reshape(len(rows), n)  # noqa
        i32 = lambda rows, k: np.array([r[k] for r in rows], dtype=np.int32)  # noqa
        u8 = lambda rows, k: np.array([r[k] for r in rows], dtype=np.uint8)  # noqa
        return Feeder(
            name=self.name, root_bus=self.root,
            bus_phases=u8(B, "phases"), bus_wmin=a(B, "wmin", 3), bus_wmax=a(B, "wmax", 3),
            bus_gsh=a(B, "gsh", 3), bus_bsh=a(B, "bsh", 3),
            line_from=i32(L, "f"), line_to=i32(L, "t"), line_phases=u8(L, "phases"),
            line_r=a(L, "r", 9), line_x=a(L, "x", 9),
            line_gs_from=a(L, "gs_from", 3), line_bs_from=a(L, "bs_from", 3),
            line_gs_to=a(L, "gs_to", 3), line_bs_to=a(L, "bs_to", 3), line_tau=a(L, "tau", 3),
            line_pmin=a(L, "pmin", 3), line_pmax=a(L, "pmax", 3), line_qmin=a(L, "qmin", 3), line_qmax=a(L, "qmax", 3),
            gen_bus=i32(G, "bus"), gen_phases=u8(G, "phases"), gen_pmin=a(G, "pmin", 3), gen_pmax=a(G, "pmax", 3),
            gen_qmin=a(G, "qmin", 3), gen_qmax=a(G, "qmax", 3),
            load_bus=i32(D, "bus"), load_phases=u8(D, "phases"), load_conn=u8(D, "conn"),
            load_alpha=a(D, "alpha", 3), load_beta=a(D, "beta", 3), load_a=a(D, "a", 3), load_b=a(D, "b", 3),
        )


# ----------------------------------------------------------------------------------------------
# Synthetic shapes (SURVEY.md App. B and §8(d) value distributions)
# ----------------------------------------------------------------------------------------------
@dataclass
class Shape:
    n3: int                    # 3-phase non-root nodes (the primary)
    n1: int                    # 1-phase nodes (laterals)
    n_lat: int                 # number of 1-phase laterals (each a chain ending in one leaf)
    window: int                # primary parent chosen among the last `window` primary nodes (depth control)
    r3: tuple                  # primary self-resistance range
    r1: tuple                  # lateral resistance range
    load_a: tuple              # load a range (p.u.)
    n_extra3: int              # extra 3-phase loads on internal primary buses
    delta_frac: float          # fraction of 3-phase loads that are delta-connected
    n_caps: int                # capacitor buses
    lat_load_every: int = 0    # also put a 1-phase load on every k-th internal lateral node (0 = leaves only)
    n_lat2: int = 0            # laterals widened to 2 phases (IEEE13 684-611/652 style)
    n_gsh: int = 0             # load-free pass-through buses given a shunt conductance g^sh (Table I)
    gs_frac: float = 0.0       # fraction of primary lines with line shunt conductances g^s at both ends


SHAPES = {
    # 13-shaped: 29 nodes, 28 lines, 7 leaves, S = 50 target; ~15 load-phases.
    "13": Shape(n3=25, n1=3, n_lat=3, window=4, r3=(0.002, 0.008), r1=(0.004, 0.016), load_a=(0.005, 0.03),
                n_extra3=1, delta_frac=0.35, n_caps=2, n_lat2=1, n_gsh=2, gs_frac=0.3),
    # 123-shaped: 147 nodes, 146 lines, 43 leaves, S = 250 target.
    "123": Shape(n3=73, n1=73, n_lat=43, window=6, r3=(0.002, 0.008), r1=(0.004, 0.016), load_a=(0.002, 0.01),
                 n_extra3=8, delta_frac=0.4, n_caps=4, lat_load_every=3, n_lat2=10, n_gsh=6, gs_frac=0.3),
    # 8500-shaped: N3=1566, N1=11545, 1222 leaves => S = 25001 (SURVEY.md App. B closed form).
    "8500": Shape(n3=1566, n1=11545, n_lat=1222, window=40, r3=(0.0002, 0.0008), r1=(0.004, 0.016),
                  load_a=(0.0005, 0.002), n_extra3=0, delta_frac=0.0, n_caps=8),
}

SEEDS = {"13": 13, "37": 37, "123": 123, "8500": 8500}


def _sym3(rng, self_lo, self_hi, mut_lo, mut_hi):
    d = rng.uniform(self_lo, self_hi, size=3)
    m = np.zeros((3, 3))
    for p in range(3):
        m[p, p] = d[p]
    for p in range(3):
        for q in range(p + 1, 3):
            m[p, q] = m[q, p] = rng.uniform(mut_lo, mut_hi) * 0.5 * (d[p] + d[q])
    return m


def make_radial(shape: Shape, seed: int, name: str) -> Feeder:
    """Radial feeder: root (3-phase, substation generator) + windowed random 3-phase primary
    + 1-phase chain laterals; every primary end carries a lateral when laterals suffice."""
    rng = np.random.default_rng(seed)
    fb = FeederBuilder(name)
    root = fb.bus(ALL3, wmin=0.9025, wmax=1.1025)
    fb.root = root
    fb.gen(root, ALL3, -10.0, 10.0, -10.0, 10.0)

    # --- primary (3-phase) tree --------------------------------------------------------------
    prim = [root]
    children = {root: 0}
    parent_of = {}
    for _ in range(shape.n3):
        cand = [b for b in prim[-shape.window:] if children[b] < 3]
        if not cand:
            cand = [b for b in prim if children[b] < 3]
        par = cand[int(rng.integers(len(cand)))]
        b = fb.bus(ALL3)
        children[par] += 1
        children[b] = 0
        parent_of[b] = par
        prim.append(b)
        r = _sym3(rng, *shape.r3, 0.25, 0.4)
        x = _sym3(rng, 2.0 * shape.r3[0], 3.0 * shape.r3[1], 0.35, 0.5)
        bs = rng.uniform(0.0, 2e-5, size=3)
        fb.line(par, b, ALL3, r, x, bs_from=bs / 2, bs_to=bs / 2)
    prim_leaves = [b for b in prim[1:] if children[b] == 0]

    # one regulator (tap) on the first primary line
    if fb.lines:
        tau = 0.98 if rng.uniform() < 0.5 else 1.02
        fb.lines[0]["tau"] = [tau, tau, tau]

    # --- 1-phase chain laterals ---------------------------------------------------------------
    lat_leaves, lat_chains = [], []
    if shape.n_lat > 0 and shape.n1 >= shape.n_lat:
        extra = rng.multinomial(shape.n1 - shape.n_lat, np.full(shape.n_lat, 1.0 / shape.n_lat))
        lengths = 1 + extra
        hosts = list(prim_leaves[: shape.n_lat])
        pool = prim[1:] if len(prim) > 1 else prim
        while len(hosts) < shape.n_lat:
            hosts.append(pool[int(rng.integers(len(pool)))])
        rng.shuffle(hosts)
        for li in range(shape.n_lat):                       # chain of lengths[li] nodes, random phase
            ph = 1 << int(rng.integers(3))
            prev = hosts[li]
            chain = (ph, [], [])
            for k in range(int(lengths[li])):
                b = fb.bus(ph)
                r = rng.uniform(*shape.r1)
                x = rng.uniform(2.0, 3.0) * r
                chain[2].append(fb.line(prev, b, ph, np.eye(3) * r, np.eye(3) * x))
                chain[1].append(b)
                if shape.lat_load_every and k < lengths[li] - 1 and (k + 1) % shape.lat_load_every == 0:
                    _add_load(fb, rng, b, ph, WYE, shape)
                prev = b
            lat_leaves.append(prev)
            lat_chains.append(chain)

    # --- loads ----------------------------------------------------------------------------------
    covered = set(lat_leaves)
    for b in lat_leaves:                                   # 1-phase wye load on every lateral end
        _add_load(fb, rng, b, fb.buses[b]["phases"], WYE, shape)
    # 3-phase leaves that did not receive a lateral keep a 3-phase load
    has_child = set(int(l["f"]) for l in fb.lines)
    for b in prim[1:]:
        if b not in has_child:
            conn = DELTA if rng.uniform() < shape.delta_frac else WYE
            _add_load(fb, rng, b, ALL3, conn, shape)
            covered.add(b)
    internal3 = [b for b in prim[1:] if b not in covered]
    for k in range(min(shape.n_extra3, len(internal3))):
        b = internal3[int(rng.integers(len(internal3)))]
        conn = DELTA if rng.uniform() < shape.delta_frac else WYE
        _add_load(fb, rng, b, ALL3, conn, shape)

    # --- capacitors ------------------------------------------------------------------------------
    for _ in range(shape.n_caps):
        b = prim[1 + int(rng.integers(len(prim) - 1))] if len(prim) > 1 else root
        bsh = rng.uniform(0.005, 0.02, size=3) * (0.1 if shape.n3 > 1000 else 1.0)
        fb.buses[b]["bsh"] = [float(v) for v in bsh]

    _widen_and_shunts(fb, shape, seed, root, lat_chains)
    f = fb.build()
    f.meta = dict(shape=name, seed=seed, n_prim_leaves=len(prim_leaves))
    return f


def _widen_and_shunts(fb: FeederBuilder, shape: Shape, seed: int, root: int, lat_chains: list):
    """The Table I input classes the base recipe leaves out, drawn from a second stream (seed + 7919) so
    the rest of the feeder is unchanged: `n_lat2` laterals widened to 2 phases (the second phase gets
    its own self r/x ~ the lateral range and mutuals U[0.25, 0.4] r / U[0.35, 0.5] x; loads on the chain
    get a second-phase a, b, alpha, beta), `n_gsh` load- and capacitor-free non-leaf buses with
    g^sh ~ U[1e-4, 5e-4], and a `gs_frac` share of the 3-phase lines with
    g^s ~ U[1e-6, 1e-5] at both ends."""
    if not (shape.n_lat2 or shape.n_gsh or shape.gs_frac):
        return
    rng = np.random.default_rng(seed + 7919)
    loads_at = {}
    for l, d in enumerate(fb.loads):
        loads_at.setdefault(d["bus"], []).append(l)
    n2 = min(shape.n_lat2, len(lat_chains))
    for ci in (rng.choice(len(lat_chains), n2, replace=False) if n2 else []):
        ph, buses, lines = lat_chains[int(ci)]
        p0 = phase_list(ph)[0]
        p1 = [p for p in range(3) if p != p0][int(rng.integers(2))]
        mask = ph | (1 << p1)
        for b in buses:
            d = fb.buses[b]
            d["phases"] = mask
            d["wmin"][p1], d["wmax"][p1] = d["wmin"][p0], d["wmax"][p0]
            for l in loads_at.get(b, []):
                ld = fb.loads[l]
                ld["phases"] = mask
                a = rng.uniform(*shape.load_a)
                ld["a"][p1] = float(a)
                ld["b"][p1] = float(a * np.tan(np.arccos(rng.uniform(0.85, 0.98))))
                ld["alpha"][p1] = float(rng.integers(0, 3))
                ld["beta"][p1] = float(rng.integers(0, 3))
        for e in lines:
            d = fb.lines[e]
            d["phases"] = mask
            r = np.array(d["r"]).reshape(3, 3)
            x = np.array(d["x"]).reshape(3, 3)
            r[p1, p1] = rng.uniform(*shape.r1)
            x[p1, p1] = rng.uniform(2.0, 3.0) * r[p1, p1]
            r[p0, p1] = r[p1, p0] = rng.uniform(0.25, 0.4) * 0.5 * (r[p0, p0] + r[p1, p1])
            x[p0, p1] = x[p1, p0] = rng.uniform(0.35, 0.5) * 0.5 * (x[p0, p0] + x[p1, p1])
            d["r"], d["x"] = r.ravel().tolist(), x.ravel().tolist()
            d["pmin"][p1], d["pmax"][p1] = d["pmin"][p0], d["pmax"][p0]
            d["qmin"][p1], d["qmax"][p1] = d["qmin"][p0], d["qmax"][p0]
            d["tau"][p1] = d["tau"][p0]
    has_child = {int(d["f"]) for d in fb.lines}
    cand = [b for b in range(len(fb.buses)) if b != root and b in has_child and b not in loads_at
            and not any(fb.buses[b]["bsh"])]
    for b in (rng.choice(cand, min(shape.n_gsh, len(cand)), replace=False) if shape.n_gsh and cand else []):
        d = fb.buses[int(b)]
        d["gsh"] = [float(rng.uniform(1e-4, 5e-4)) if p in phase_list(d["phases"]) else 0.0 for p in range(3)]
    for d in fb.lines:
        if d["phases"] == ALL3 and rng.uniform() < shape.gs_frac:
            d["gs_from"] = [float(v) for v in rng.uniform(1e-6, 1e-5, size=3)]
            d["gs_to"] = [float(v) for v in rng.uniform(1e-6, 1e-5, size=3)]


def _add_load(fb: FeederBuilder, rng, bus: int, phases: int, conn: int, shape: Shape):
    a = rng.uniform(*shape.load_a, size=3)
    pf = rng.uniform(0.85, 0.98, size=3)
    b = a * np.tan(np.arccos(pf))
    alpha = rng.integers(0, 3, size=3).astype(np.float64)
    beta = rng.integers(0, 3, size=3).astype(np.float64)
    fb.load(bus, phases, conn, alpha, beta, a, b)


def make_delta37(seed: int = 37) -> Feeder:
    """IEEE37-shaped (Table II-IV column 2): a 3-wire, 3-phase feeder whose loads are all
    delta-connected (VDLM-4 and VDLM-6..10).  Radial tree (reading C14) of 57 buses and
    56 lines with exactly 16 leaves, so S = 57 + 56 - 16 = 97 (Table III); 30 three-phase delta loads (the 16
    leaves and 14 internal buses) give sum m_s = 6 * 57 + 9 * 56 + 12 * 30 = 1206 rows (Table II, IV).
    A trunk from the substation with 15 side branches (lengths multinomial), a regulator tap on the first
    line, no capacitors, alpha, beta in {0, 1, 2}, a ~ U[0.01, 0.05], b = a tan(acos pf)."""
    rng = np.random.default_rng(seed)
    fb = FeederBuilder("ieee37-shaped")
    root = fb.bus(ALL3, wmin=0.9025, wmax=1.1025)
    fb.root = root
    fb.gen(root, ALL3, -10.0, 10.0, -10.0, 10.0)
    n_leaf, n_nodes = 16, 56
    lengths = 1 + rng.multinomial(n_nodes - n_leaf, np.full(n_leaf, 1.0 / n_leaf))   # trunk + 15 branches
    shape = Shape(n3=n_nodes, n1=0, n_lat=0, window=1, r3=(0.002, 0.008), r1=(0.004, 0.016), load_a=(0.01, 0.05),
                  n_extra3=14, delta_frac=1.0, n_caps=0)

    def line(par, b):
        r = _sym3(rng, *shape.r3, 0.25, 0.4)
        x = _sym3(rng, 2.0 * shape.r3[0], 3.0 * shape.r3[1], 0.35, 0.5)
        fb.line(par, b, ALL3, r, x)

    trunk, prev = [], root
    for _ in range(int(lengths[0])):
        b = fb.bus(ALL3)
        line(prev, b)
        trunk.append(b)
        prev = b
    leaves = [trunk[-1]]
    internal = list(trunk[:-1])
    for li in range(1, n_leaf):
        prev = trunk[int(rng.integers(len(trunk) - 1))] if len(trunk) > 1 else root
        for k in range(int(lengths[li])):
            b = fb.bus(ALL3)
            line(prev, b)
            if k < lengths[li] - 1:
                internal.append(b)
            prev = b
        leaves.append(prev)
    tau = 0.98 if rng.uniform() < 0.5 else 1.02
    fb.lines[0]["tau"] = [tau, tau, tau]
    for b in leaves:
        _add_load(fb, rng, b, ALL3, DELTA, shape)
    for b in rng.choice(internal, shape.n_extra3, replace=False):
        _add_load(fb, rng, int(b), ALL3, DELTA, shape)
    f = fb.build()
    f.meta = dict(shape="37", seed=seed)
    return f


def make_feeder(shape: str, seed: int | None = None) -> Feeder:
    """The synthetic instance for configs 1-3 (shape '13', '123', '8500') and the IEEE37-shaped delta feeder."""
    if seed is None:
        seed = SEEDS[shape]
    if shape == "37":
        return make_delta37(seed)
    return make_radial(SHAPES[shape], seed, f"ieee{shape}-shaped")


def scale_loads(f: Feeder, kappa: np.ndarray) -> Feeder:
    """Scenario sigma of config 4: every load's (a, b) scaled by kappa[l] (BASELINE.json configs[3])."""
    g = f.copy()
    g.load_a = g.load_a * kappa[:, None]
    g.load_b = g.load_b * kappa[:, None]
    return g


def scenario_scales(f: Feeder, n_scen: int, seed: int = 4096) -> np.ndarray:
    """kappa[sigma, l] ~ U[0.5, 1.5] iid."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0.5, 1.5, size=(n_scen, f.n_load))


def graph_stats(f: Feeder) -> dict:
    """Nodes / lines / leaves (degree-1 non-root) of the component graph."""
    deg = np.zeros(f.n_bus, dtype=np.int64)
    np.add.at(deg, f.line_from, 1)
    np.add.at(deg, f.line_to, 1)
    leaves = int(np.sum((deg == 1) & (np.arange(f.n_bus) != f.root_bus)))
    load_phases = int(sum(len(phase_list(m)) for m in f.load_phases))
    return dict(nodes=f.n_bus, lines=f.n_line, leaves=leaves, load_phases=load_phases)


def make_stitched(n_sub: int = 64, shape: str = "8500", seed0: int | None = None, trunk_scale: float = 0.01) -> Feeder:
    """Config 5 (BASELINE.json configs[4]): n_sub subfeeders of `shape` (seeds seed0 + f, their own
    substation generators removed) each hung by a 3-phase line off bus f of an n_sub-bus 3-phase trunk
    chain that starts at the substation; trunk r, x scaled by `trunk_scale`; the trunk, the tie lines and
    the substation generator carry the whole load, so their bounds are widened to +-1000 p.u."""
    seed0 = SEEDS[shape] if seed0 is None else seed0
    rng = np.random.default_rng(seed0 + 10_000)
    fb = FeederBuilder(f"stitched{n_sub}x{shape}")
    root = fb.bus(ALL3, wmin=0.9025, wmax=1.1025)
    fb.root = root
    fb.gen(root, ALL3, -1000.0, 1000.0, -1000.0, 1000.0)
    trunk, prev = [], root
    for f in range(n_sub):
        b = fb.bus(ALL3)
        r = _sym3(rng, 0.0002 * trunk_scale, 0.0008 * trunk_scale, 0.25, 0.4)
        x = _sym3(rng, 0.0004 * trunk_scale, 0.0024 * trunk_scale, 0.35, 0.5)
        fb.line(prev, b, ALL3, r, x, fmin=-1000.0, fmax=1000.0)
        trunk.append(b)
        prev = b
    subs = [make_radial(SHAPES[shape], seed0 + f, "sub") for f in range(n_sub)]
    off = np.cumsum([1 + n_sub] + [s.n_bus for s in subs])[:-1]           # bus offset of each subfeeder
    for f in range(n_sub):                                                  # tie lines trunk f -> sub root
        r = _sym3(rng, 0.0002, 0.0008, 0.25, 0.4)
        x = _sym3(rng, 0.0004, 0.0024, 0.35, 0.5)
        fb.line(trunk[f], int(off[f] + subs[f].root_bus), ALL3, r, x, fmin=-1000.0, fmax=1000.0)
    head = fb.build()
    cat = lambda name, conv=None: np.concatenate([getattr(head, name)] + [  # noqa: E731
        conv(getattr(s, name), f) if conv else getattr(s, name) for f, s in enumerate(subs)])
    shift = lambda a, f: (a + off[f]).astype(np.int32)  # noqa: E731
    kw = {}
    for fld in dataclasses.fields(Feeder):
        n = fld.name
        if n in ("name", "root_bus", "meta") or n.startswith("gen_"):
            continue
        kw[n] = cat(n, shift if n in ("line_from", "line_to", "load_bus") else None)
    for n in ("gen_bus", "gen_phases", "gen_pmin", "gen_pmax", "gen_qmin", "gen_qmax"):
        kw[n] = getattr(head, n)                                            # only the substation generator
    g = Feeder(name=head.name, root_bus=root, **kw)
    g.meta = dict(shape=f"stitched{n_sub}x{shape}", seed0=seed0, n_sub=n_sub,
                  sub_bus_off=[int(v) for v in off] + [int(off[-1] + subs[-1].n_bus)])
    return g


def stitched_bus_owner(f: Feeder, world: int) -> np.ndarray:
    """The natural partition of a stitched feeder over `world` ranks: rank
    r = floor(f * world / n_sub) owns subfeeder f and trunk bus f; the substation bus goes to rank 0."""
    n_sub, off = f.meta["n_sub"], f.meta["sub_bus_off"]
    own = np.zeros(f.n_bus, np.int32)
    for k in range(n_sub):
        r = k * world // n_sub
        own[1 + k] = r                                   # trunk bus k
        own[off[k]:off[k + 1]] = r
    return own
