"""Thin ctypes binding of include/lopf.h (argument marshalling only).

Every step of the ADMM path runs inside liblopf.so (host setup in C++, iterations in the
sm_100a kernels).  PyTorch supplies device memory (the arena is a uint8 CUDA tensor) and
streams.  There is no fallback: if liblopf.so is missing or a call fails, an exception is raised.

Method names mirror the C ABI (`lopf_setup` -> `Lopf.setup`, `lopf_solve` -> `Lopf.solve`, ...).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOPF_LIB", os.path.join(_HERE, "liblopf.so"))   # override: A/B of builds

STATUS = {0: "LOPF_OK", 1: "LOPF_E_ARG", 2: "LOPF_E_NETWORK", 3: "LOPF_E_ORPHAN", 4: "LOPF_E_INFEASIBLE_SUB",
          5: "LOPF_E_RANK", 6: "LOPF_E_CUDA", 7: "LOPF_E_NCCL", 8: "LOPF_E_NUMERIC", 9: "LOPF_E_STATE"}
CONVERGED, MAX_ITER = 0, 2
ROLES = ["pg", "qg", "w", "pb", "qb", "pd", "qd", "pf", "qf", "pt", "qt"]   # p_eij = pf, ..., q_eji = qt


class LopfError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


_vp, _i32, _i64, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double


class Network(C.Structure):
    _fields_ = [("n_bus", _i32), ("n_line", _i32), ("n_gen", _i32), ("n_load", _i32), ("root_bus", _i32)] + \
               [(k, _vp) for k in ("bus_phases", "bus_wmin", "bus_wmax", "bus_gsh", "bus_bsh", "line_from", "line_to",
                                   "line_phases", "line_r", "line_x", "line_gs_from", "line_bs_from", "line_gs_to",
                                   "line_bs_to", "line_tau", "line_pmin", "line_pmax", "line_qmin", "line_qmax",
                                   "gen_bus", "gen_phases", "gen_pmin", "gen_pmax", "gen_qmin", "gen_qmax", "load_bus",
                                   "load_phases", "load_conn", "load_alpha", "load_beta", "load_a", "load_b")]


class Options(C.Structure):
    _fields_ = [("rho", _f64), ("eps_rel", _f64), ("max_iter", _i64), ("trace_every", _i32), ("trace_cap", _i32),
                ("single", _i32), ("kernel", _i32), ("block_threads", _i32), ("max_ctas", _i32), ("grid_cap", _i32),
                ("reserved", _i32 * 2), ("precision", _i32), ("adapt_every", _i32), ("coarse", _i32),
                ("adapt_mu", _f64), ("adapt_tau", _f64)]


class Sizes(C.Structure):
    _fields_ = [(k, _i64) for k in ("S", "n", "m", "n_copies", "p_sym", "n_tasks", "n_slots", "device_bytes",
                                    "abar_doubles", "alg_bytes")] + \
               [(k, _i32) for k in ("kernel", "grid", "block", "max_ns", "max_ms", "n_scen")] + [("reserved", _i32 * 2)] + \
               [(k, _i64) for k in ("upload_bytes", "fetch_bytes")]


class Result(C.Structure):
    _fields_ = [("outcome", _i32), ("reserved0", _i32), ("iters", _i64), ("pres", _f64), ("dres", _f64),
                ("eps_prim", _f64), ("eps_dual", _f64), ("objective", _f64), ("solve_ms", _f64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("reserved")}


_lib = None


def load_library(path: str = LIB_PATH):
    """Load liblopf.so (raises if it has not been built: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(the CUDA path has no fallback)")
    lib = C.CDLL(path)
    H = _vp
    sig = {
        "lopf_options_default": ([C.POINTER(Options)], _i32),
        "lopf_setup": ([C.POINTER(Network), C.POINTER(Options), C.POINTER(H)], _i32),
        "lopf_sizes_get": ([H, C.POINTER(Sizes)], _i32),
        "lopf_bind": ([H, _vp, C.c_size_t, _vp], _i32),
        "lopf_reset": ([H, _vp], _i32),
        "lopf_solve": ([H, _vp, C.POINTER(Result)], _i32),
        "lopf_run": ([H, _i64, _i32, _vp, C.POINTER(Result)], _i32),
        "lopf_solve_async": ([H, _i64, _i32, _vp], _i32),
        "lopf_result_get": ([H, _vp, C.POINTER(Result)], _i32),
        "lopf_fetch_async": ([H, _vp, _vp], _i32),
        "lopf_get_rho": ([H, _vp, _vp, _vp], _i32),
        "lopf_get_decomposition": ([H] + [_vp] * 7, _i32),
        "lopf_get_consensus": ([H, _vp, _vp], _i32),
        "lopf_get_globals": ([H] + [_vp] * 6, _i32),
        "lopf_get_operator": ([H, _i64, _vp, _vp], _i32),
        "lopf_get_subsystem": ([H, _i64, _vp, _vp, _vp], _i32),
        "lopf_get_state": ([H, _vp, _vp, _vp, _vp], _i32),
        "lopf_set_state": ([H, _vp, _vp, _vp], _i32),
        "lopf_get_trace": ([H, _vp, _vp, _i64, _vp], _i32),
        "lopf_get_profile": ([H, _vp, _vp, _i64, _vp], _i32),
        "lopf_setup_batch": ([C.POINTER(Network), C.POINTER(Options), _i32, _vp, C.POINTER(H)], _i32),
        "lopf_get_batch_results": ([H, _vp, _vp, _vp, _vp, _vp], _i32),
        "lopf_get_state_scen": ([H, _vp, _i32, _vp, _vp, _vp], _i32),
        "lopf_get_operator_scen": ([H, _i64, _i32, _vp, _vp], _i32),
        "lopf_setup_part": ([C.POINTER(Network), C.POINTER(Options), _i32, _i32, _vp, C.POINTER(H)], _i32),
        "lopf_part_info": ([H, _vp, _vp, _vp, _vp], _i32),
        "lopf_part_owner": ([H, _vp, _vp, _vp], _i32),
        "lopf_part_sweep": ([H, _vp], _i32),
        "lopf_part_import": ([H, _vp], _i32),
        "lopf_part_p2p_info": ([H, _vp, _vp], _i32),
        "lopf_part_connect": ([H, _vp, _vp], _i32),
        "lopf_part_solve_p2p": ([H, _i64, _i32, _vp], _i32),
        "lopf_part_emulate": ([_vp, _i32, _i64, _i32, _vp], _i32),
        "lopf_ipc_export": ([_vp, _vp], _i32),
        "lopf_nccl_unique_id": ([_vp], _i32),
        "lopf_part_nccl_init": ([H, _vp], _i32),
        "lopf_part_step": ([H, _vp], _i32),
        "lopf_ipc_open": ([H, _vp, _vp], _i32),
        "lopf_destroy": ([H], None),
        "lopf_last_error": ([], C.c_char_p),
        "lopf_abi_version": ([], _i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(st: int, where: str):
    if st != 0:
        raise LopfError(st, where, load_library().lopf_last_error().decode(errors="replace"))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _network(feeder) -> tuple[Network, list]:
    """Marshal a feedergen.Feeder-like object (structure of arrays) into lopf_network."""
    keep = []

    def arr(name, dtype):
        a = np.ascontiguousarray(getattr(feeder, name), dtype=dtype)
        keep.append(a)
        return _ptr(a)

    net = Network(n_bus=feeder.n_bus, n_line=feeder.n_line, n_gen=feeder.n_gen, n_load=feeder.n_load,
                  root_bus=int(feeder.root_bus))
    u8 = {"bus_phases", "line_phases", "gen_phases", "load_phases", "load_conn"}
    i32 = {"line_from", "line_to", "gen_bus", "load_bus"}
    for k, _ in Network._fields_[5:]:
        setattr(net, k, arr(k, np.uint8 if k in u8 else np.int32 if k in i32 else np.float64))
    return net, keep


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


@dataclass
class Decomp:
    kind: np.ndarray
    comp: np.ndarray
    leaf_bus: np.ndarray
    m_s: np.ndarray
    n_s: np.ndarray
    sub_ptr: np.ndarray
    copy_global: np.ndarray


class Lopf:
    """One problem instance: `Lopf.setup(feeder)` -> `.bind()` -> `.solve()` / `.run(k)`."""

    def __init__(self, handle: int, opts: Options):
        self._h = _vp(handle)
        self.opts = opts
        self.arena = None
        self._sizes = None

    # ---- lopf_setup / lopf_sizes_get ---------------------------------------------------------
    @classmethod
    def setup(cls, feeder, rho: float = 100.0, eps_rel: float = 1e-3, max_iter: int = 1_000_000,
              trace_every: int = 0, trace_cap: int = 4096, single: bool = False, kernel: int = 0,
              grid_cap: int = 0, max_ctas: int = 0, diag_profile: bool = False,
              precision: int = 64, adapt_every: int = 0, adapt_mu: float = 0.0, adapt_tau: float = 0.0,
              coarse: int = 0) -> "Lopf":
        """lopf_setup; precision 32 selects the fp32 variant (the paper's GPU precision);
        adapt_every > 0 enables residual balancing of rho (reading F2)."""
        lib = load_library()
        o = Options()
        _check(lib.lopf_options_default(C.byref(o)), "lopf_options_default")
        o.rho, o.eps_rel, o.max_iter = float(rho), float(eps_rel), int(max_iter)
        o.trace_every, o.trace_cap, o.single, o.kernel = int(trace_every), int(trace_cap), int(bool(single)), int(kernel)
        o.grid_cap, o.max_ctas = int(grid_cap), int(max_ctas)
        o.reserved[0] = int(bool(diag_profile))
        o.precision = int(precision)
        o.adapt_every, o.adapt_mu, o.adapt_tau = int(adapt_every), float(adapt_mu), float(adapt_tau)
        o.coarse = int(coarse)
        net, keep = _network(feeder)
        h = _vp()
        _check(lib.lopf_setup(C.byref(net), C.byref(o), C.byref(h)), "lopf_setup")
        del keep
        return cls(h.value, o)

    @classmethod
    def setup_batch(cls, feeder, load_scale, rho: float = 100.0, eps_rel: float = 1e-3, max_iter: int = 1_000_000,
                    precision: int = 64) -> "Lopf":
        """lopf_setup_batch: load_scale [n_scen, n_load] (> 0) scales every load's (a, b) per scenario."""
        lib = load_library()
        o = Options()
        _check(lib.lopf_options_default(C.byref(o)), "lopf_options_default")
        o.rho, o.eps_rel, o.max_iter = float(rho), float(eps_rel), int(max_iter)
        o.precision = int(precision)
        net, keep = _network(feeder)
        sc = np.ascontiguousarray(load_scale, dtype=np.float64)
        if sc.ndim != 2 or sc.shape[1] != feeder.n_load:
            raise ValueError("load_scale must be [n_scen, n_load]")
        h = _vp()
        _check(lib.lopf_setup_batch(C.byref(net), C.byref(o), int(sc.shape[0]), _ptr(sc), C.byref(h)), "lopf_setup_batch")
        del keep
        return cls(h.value, o)

    @classmethod
    def setup_part(cls, feeder, rank: int, world: int, bus_owner=None, rho: float = 100.0, eps_rel: float = 1e-3,
                   max_iter: int = 1_000_000, precision: int = 64) -> "Lopf":
        """lopf_setup_part: this rank's share of a feeder partitioned over `world` ranks (config 5)."""
        lib = load_library()
        o = Options()
        _check(lib.lopf_options_default(C.byref(o)), "lopf_options_default")
        o.rho, o.eps_rel, o.max_iter, o.kernel = float(rho), float(eps_rel), int(max_iter), 1
        o.precision = int(precision)
        net, keep = _network(feeder)
        own = None if bus_owner is None else np.ascontiguousarray(bus_owner, dtype=np.int32)
        h = _vp()
        _check(lib.lopf_setup_part(C.byref(net), C.byref(o), int(rank), int(world),
                                   None if own is None else _ptr(own), C.byref(h)), "lopf_setup_part")
        del keep
        return cls(h.value, o)

    def part_info(self) -> dict:
        off, nd = _i64(0), _i64(0)
        nb, ni = _i32(0), _i32(0)
        _check(load_library().lopf_part_info(self._h, C.byref(off), C.byref(nd), C.byref(nb), C.byref(ni)),
               "lopf_part_info")
        return dict(offset=off.value, doubles=nd.value, n_bnd=nb.value, n_imp=ni.value)

    def part_owner(self, n_bus: int):
        nc = int(self.sizes.n_copies)
        bo = np.zeros(n_bus, np.int32)
        co = np.zeros(nc, np.int32)
        bi = np.zeros(nc, np.int32)
        _check(load_library().lopf_part_owner(self._h, _ptr(bo), _ptr(co), _ptr(bi)), "lopf_part_owner")
        return bo, co, bi

    def exchange(self):
        """The exchange buffer as a float64 torch view of the arena (for the allreduce)."""
        import torch
        inf = self.part_info()
        return self.arena[inf["offset"]: inf["offset"] + 8 * inf["doubles"]].view(torch.float64)

    def part_sweep(self, stream=None):
        _check(load_library().lopf_part_sweep(self._h, _vp(_stream_handle(stream))), "lopf_part_sweep")

    def part_import(self, stream=None):
        _check(load_library().lopf_part_import(self._h, _vp(_stream_handle(stream))), "lopf_part_import")

    # ---- device-initiated exchange ------------------------------------------------------------
    def p2p_entries(self) -> int:
        """Device address of this rank's p2p entry buffer (valid in this process)."""
        xo, nb = _i64(0), _i64(0)
        _check(load_library().lopf_part_p2p_info(self._h, C.byref(xo), C.byref(nb)), "lopf_part_p2p_info")
        return self.arena.data_ptr() + xo.value

    def part_connect(self, peer_entries, stream=None):
        xe = np.ascontiguousarray(peer_entries, dtype=np.uint64)
        _check(load_library().lopf_part_connect(self._h, _ptr(xe), _vp(_stream_handle(stream))), "lopf_part_connect")

    def part_solve_p2p(self, max_iter: int, test: bool = True, stream=None):
        _check(load_library().lopf_part_solve_p2p(self._h, int(max_iter), int(bool(test)), _vp(_stream_handle(stream))),
               "lopf_part_solve_p2p")

    @staticmethod
    def part_emulate(handles, max_iter: int, test: bool = True, stream=None):
        """All ranks (handles[q] = rank q, bound on this GPU) in one cooperative launch (lopf_part_emulate)."""
        arr = (_vp * len(handles))(*[h._h.value for h in handles])
        _check(load_library().lopf_part_emulate(arr, len(handles), int(max_iter), int(bool(test)),
                                                _vp(_stream_handle(stream))), "lopf_part_emulate")

    @staticmethod
    def nccl_unique_id() -> bytes:
        out = C.create_string_buffer(128)
        _check(load_library().lopf_nccl_unique_id(out), "lopf_nccl_unique_id")
        return out.raw

    def part_nccl_init(self, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(load_library().lopf_part_nccl_init(self._h, buf), "lopf_part_nccl_init")

    def part_step(self, stream=None):
        _check(load_library().lopf_part_step(self._h, _vp(_stream_handle(stream))), "lopf_part_step")

    @staticmethod
    def ipc_export(dev_ptr: int) -> bytes:
        out = C.create_string_buffer(72)
        _check(load_library().lopf_ipc_export(_vp(dev_ptr), out), "lopf_ipc_export")
        return out.raw

    def ipc_open(self, record: bytes) -> int:
        p = _vp()
        buf = C.create_string_buffer(bytes(record), 72)
        _check(load_library().lopf_ipc_open(self._h, buf, C.byref(p)), "lopf_ipc_open")
        return p.value

    def get_batch_results(self, stream=None) -> dict:
        ns = int(self.sizes.n_scen)
        it = np.zeros(ns, np.int64)
        oc = np.zeros(ns, np.int32)
        rs = np.zeros((ns, 4))
        ob = np.zeros(ns)
        _check(load_library().lopf_get_batch_results(self._h, _vp(_stream_handle(stream)), _ptr(it), _ptr(oc), _ptr(rs),
                                                     _ptr(ob)), "lopf_get_batch_results")
        return dict(iters=it, outcome=oc, res=rs, objective=ob)

    def get_state_scen(self, scen: int, stream=None):
        s = self.sizes
        x = np.zeros(int(s.n))
        xl = np.zeros(int(s.n_copies))
        lam = np.zeros(int(s.n_copies))
        _check(load_library().lopf_get_state_scen(self._h, _vp(_stream_handle(stream)), int(scen), _ptr(x), _ptr(xl),
                                                  _ptr(lam)), "lopf_get_state_scen")
        return x, xl, lam

    def get_operator_scen(self, s: int, scen: int, n_s: int):
        ab = np.zeros(n_s * n_s)
        bb = np.zeros(n_s)
        _check(load_library().lopf_get_operator_scen(self._h, int(s), int(scen), _ptr(ab), _ptr(bb)),
               "lopf_get_operator_scen")
        return ab.reshape(n_s, n_s), bb

    def sizes_get(self) -> Sizes:
        s = Sizes()
        _check(load_library().lopf_sizes_get(self._h, C.byref(s)), "lopf_sizes_get")
        return s

    @property
    def sizes(self) -> Sizes:
        """lopf_sizes_get, cached (the sizes are fixed at setup; grid and block once bound)."""
        if self._sizes is None or (self._sizes.grid == 0 and self.arena is not None):
            self._sizes = self.sizes_get()
        return self._sizes

    # ---- device ---------------------------------------------------------------------------------
    def bind(self, device="cuda", stream=None, arena=None):
        """lopf_bind: allocate (or reuse) the device arena as a torch uint8 tensor and upload."""
        import torch
        nbytes = int(self.sizes.device_bytes)
        if arena is None:
            arena = self.arena if self.arena is not None else torch.empty(nbytes, dtype=torch.uint8, device=device)
        first = self.arena is None
        self.arena = arena
        _check(load_library().lopf_bind(self._h, _vp(arena.data_ptr()), arena.numel(), _vp(_stream_handle(stream))),
               "lopf_bind")
        if first:
            self._sizes = None                          # grid / block are known now
        return self

    def reset(self, stream=None):
        _check(load_library().lopf_reset(self._h, _vp(_stream_handle(stream))), "lopf_reset")

    def solve(self, stream=None) -> Result:
        r = Result()
        _check(load_library().lopf_solve(self._h, _vp(_stream_handle(stream)), C.byref(r)), "lopf_solve")
        return r

    def run(self, k: int, test: bool = False, stream=None) -> Result:
        r = Result()
        _check(load_library().lopf_run(self._h, int(k), int(bool(test)), _vp(_stream_handle(stream)), C.byref(r)),
               "lopf_run")
        return r

    def solve_async(self, max_iter: int, test: bool = True, stream=None):
        _check(load_library().lopf_solve_async(self._h, int(max_iter), int(bool(test)), _vp(_stream_handle(stream))),
               "lopf_solve_async")

    def get_rho(self, stream=None):
        """(rho in force, number of residual-balancing changes since the reset)."""
        r, n = _f64(0.0), _i64(0)
        _check(load_library().lopf_get_rho(self._h, _vp(_stream_handle(stream)), C.byref(r), C.byref(n)), "lopf_get_rho")
        return r.value, n.value

    def fetch_async(self, host_buf, stream=None):
        """lopf_fetch_async into a host buffer of sizes.fetch_bytes bytes (a pinned torch uint8 tensor for a
        truly asynchronous copy); decode it with `Lopf.decode_fetch` after the stream has reached it."""
        ptr = host_buf.data_ptr() if hasattr(host_buf, "data_ptr") else host_buf.ctypes.data
        _check(load_library().lopf_fetch_async(self._h, _vp(_stream_handle(stream)), _vp(ptr)), "lopf_fetch_async")

    @staticmethod
    def decode_fetch(host_buf, n: int, with_x: bool = True):
        """(Result, x) from a buffer filled by fetch_async (x is None with with_x=False)."""
        raw = host_buf.numpy() if hasattr(host_buf, "numpy") else np.asarray(host_buf)
        raw = raw.view(np.uint8)
        r = Result.from_buffer_copy(raw[: C.sizeof(Result)].tobytes())
        x = raw[64: 64 + 8 * n].view(np.float64).copy() if with_x else None
        return r, x

    def result_get(self, stream=None) -> Result:
        r = Result()
        _check(load_library().lopf_result_get(self._h, _vp(_stream_handle(stream)), C.byref(r)), "lopf_result_get")
        return r

    # ---- canonical getters -------------------------------------------------------------------------
    def get_decomposition(self) -> Decomp:
        s = self.sizes
        S, nc = int(s.S), int(s.n_copies)
        kind, comp, leaf, ms, ns = (np.zeros(S, np.int32) for _ in range(5))
        sub_ptr = np.zeros(S + 1, np.int64)
        cg = np.zeros(nc, np.int32)
        _check(load_library().lopf_get_decomposition(self._h, _ptr(kind), _ptr(comp), _ptr(leaf), _ptr(ms), _ptr(ns),
                                                     _ptr(sub_ptr), _ptr(cg)), "lopf_get_decomposition")
        return Decomp(kind, comp, leaf, ms, ns, sub_ptr, cg)

    def get_consensus(self):
        s = self.sizes
        rp = np.zeros(int(s.n) + 1, np.int64)
        ci = np.zeros(int(s.n_copies), np.int32)
        _check(load_library().lopf_get_consensus(self._h, _ptr(rp), _ptr(ci)), "lopf_get_consensus")
        return rp, ci

    def get_globals(self):
        n = int(self.sizes.n)
        role, comp, ph = (np.zeros(n, np.int32) for _ in range(3))
        c, lo, hi = (np.zeros(n) for _ in range(3))
        _check(load_library().lopf_get_globals(self._h, _ptr(role), _ptr(comp), _ptr(ph), _ptr(c), _ptr(lo), _ptr(hi)),
               "lopf_get_globals")
        return dict(role=role, comp=comp, phase=ph, c=c, lo=lo, hi=hi)

    def get_operator(self, s: int, n_s: int):
        ab = np.zeros(n_s * n_s)
        bb = np.zeros(n_s)
        _check(load_library().lopf_get_operator(self._h, int(s), _ptr(ab), _ptr(bb)), "lopf_get_operator")
        return ab.reshape(n_s, n_s), bb

    def get_subsystem(self, s: int, m_s: int, n_s: int):
        A = np.zeros(max(m_s, 1) * n_s)
        b = np.zeros(max(m_s, 1))
        m = _i32(0)
        _check(load_library().lopf_get_subsystem(self._h, int(s), _ptr(A), _ptr(b), C.byref(m)), "lopf_get_subsystem")
        return A[: m.value * n_s].reshape(m.value, n_s), b[: m.value]

    def get_state(self, stream=None):
        s = self.sizes
        x = np.zeros(int(s.n))
        xl = np.zeros(int(s.n_copies))
        lam = np.zeros(int(s.n_copies))
        _check(load_library().lopf_get_state(self._h, _vp(_stream_handle(stream)), _ptr(x), _ptr(xl), _ptr(lam)),
               "lopf_get_state")
        return x, xl, lam

    def get_x(self, stream=None) -> np.ndarray:
        """Only the solution x (D2H of n doubles)."""
        x = np.zeros(int(self.sizes.n))
        _check(load_library().lopf_get_state(self._h, _vp(_stream_handle(stream)), _ptr(x), None, None),
               "lopf_get_state")
        return x

    def set_state(self, x_loc, lam, stream=None):
        xl = np.ascontiguousarray(x_loc, np.float64)
        lm = np.ascontiguousarray(lam, np.float64)
        _check(load_library().lopf_set_state(self._h, _vp(_stream_handle(stream)), _ptr(xl), _ptr(lm)), "lopf_set_state")

    def get_trace(self, cap: int = 4096, stream=None) -> np.ndarray:
        buf = np.zeros((cap, 5))
        n = _i64(0)
        _check(load_library().lopf_get_trace(self._h, _vp(_stream_handle(stream)), _ptr(buf), cap, C.byref(n)),
               "lopf_get_trace")
        return buf[: n.value].copy()

    def get_profile(self, stream=None, timeline: bool = False) -> np.ndarray:
        """Diagnostics: per-CTA cycles {work, publish + neighbour wait, -, sweeps} of the last resident launch
        (timeline=True: followed by the 32 G rows of a LOPF_RES_TIMELINE build's events).
        The counters perturb the kernel: use them for relative shares, not absolute times."""
        g = int(self.sizes.grid) * (41 if timeline else 1)
        buf = np.zeros((g, 4), np.int64)
        n = _i64(0)
        _check(load_library().lopf_get_profile(self._h, _vp(_stream_handle(stream)), _ptr(buf), g, C.byref(n)),
               "lopf_get_profile")
        return buf[: n.value]

    def destroy(self):
        if self._h:
            load_library().lopf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
