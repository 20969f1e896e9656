"""Oracle driver for Algorithm 1.  TEST INFRASTRUCTURE ONLY.

Python builds the problem (LP -> decomposition -> precompute, all oracle code) and the
initial point; the sweeps themselves run in the plain-C `admm_loop.c` (one thread,
-ffp-contract=off), reached through ctypes.  Each step is also exported on its own
(`global_update`, `local_update`, `dual_update`, `residuals`) so the tests can pin it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from feedergen import Feeder
from .lp import LP, assemble_lp
from .decompose import Decomposition, decompose
from .precompute import precompute

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_admm.so")
_SO_OMP = os.path.join(_HERE, "_build", "liboracle_admm_omp.so")
_SRC = os.path.join(_HERE, "admm_loop.c")


def build_lib(force: bool = False, openmp: bool = False) -> str:
    """Compile admm_loop.c (gcc -O2 -ffp-contract=off); the checker is built, never shipped.  openmp=True:
    the multi-core timing build of bench.py's cpu_baseline mode (ii) (not a parity reference)."""
    so = _SO_OMP if openmp else _SO
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(so), exist_ok=True)
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-std=c11", *(["-fopenmp"] if openmp else []), "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, so)
    return so


class _Problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("S", C.c_int64), ("nc", C.c_int64),
                ("c", C.c_void_p), ("lo", C.c_void_p), ("hi", C.c_void_p),
                ("seg_ptr", C.c_void_p), ("seg_copy", C.c_void_p), ("copy_global", C.c_void_p),
                ("sub_ptr", C.c_void_p), ("abar_ptr", C.c_void_p), ("abar", C.c_void_p), ("bbar", C.c_void_p),
                ("rho", C.c_double), ("eps_rel", C.c_double)]


class _ProblemF32(C.Structure):
    _fields_ = [("n", C.c_int64), ("S", C.c_int64), ("nc", C.c_int64),
                ("c", C.c_void_p), ("lo", C.c_void_p), ("hi", C.c_void_p),
                ("seg_ptr", C.c_void_p), ("seg_copy", C.c_void_p), ("copy_global", C.c_void_p),
                ("sub_ptr", C.c_void_p), ("abar_ptr", C.c_void_p), ("abar", C.c_void_p), ("bbar", C.c_void_p),
                ("rho", C.c_float), ("rho64", C.c_double), ("eps_rel", C.c_double)]


_lib = None
_lib_omp = None


def _declare(lib_):
    P = C.POINTER(_Problem)
    vp = C.c_void_p
    lib_.oracle_run.argtypes = [P, vp, vp, vp, C.c_int64, C.c_int32, vp, vp, vp, C.c_int64, C.c_int32, vp]
    lib_.oracle_run.restype = C.c_int64
    return lib_


def lib_omp():
    """The OpenMP build (timing only: its residual sums are reduced in a different order)."""
    global _lib_omp
    if _lib_omp is None:
        _lib_omp = _declare(C.CDLL(build_lib(openmp=True)))
    return _lib_omp


def run_k_omp(prob: "OracleProblem", k: int, state=None) -> int:
    """k sweeps of the OpenMP build from `state` (default: the initial point); returns k.  For timing."""
    xl, lam = state if state is not None else initial_state(prob)
    x = np.zeros(prob.n)
    xl = np.array(xl, dtype=np.float64, copy=True)
    lam = np.array(lam, dtype=np.float64, copy=True)
    res = np.zeros(4)
    conv = C.c_int32(0)
    nrow = C.c_int64(0)
    return int(lib_omp().oracle_run(C.byref(prob._st), _p(x), _p(xl), _p(lam), int(k), 0, _p(res), C.byref(conv), None,
                                    0, 0, C.byref(nrow)))


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_lib())
        P = C.POINTER(_Problem)
        vp = C.c_void_p
        _lib.oracle_global_update.argtypes = [P, vp, vp, vp]
        _lib.oracle_local_update.argtypes = [P, vp, vp, vp]
        _lib.oracle_dual_update.argtypes = [P, vp, vp, vp]
        _lib.oracle_residuals.argtypes = [P, vp, vp, vp, vp, vp]
        _lib.oracle_run.argtypes = [P, vp, vp, vp, C.c_int64, C.c_int32, vp, vp, vp, C.c_int64, C.c_int32, vp]
        _lib.oracle_run.restype = C.c_int64
        _lib.oracle_run_adaptive.argtypes = [P, vp, vp, vp, C.c_int64, C.c_int32, vp, vp, C.c_int32, C.c_double,
                                             C.c_double, vp, vp]
        _lib.oracle_run_adaptive.restype = C.c_int64
        _lib.oracle_run_f32.argtypes = [C.POINTER(_ProblemF32), vp, vp, vp, C.c_int64, C.c_int32, vp, vp]
        _lib.oracle_run_f32.restype = C.c_int64
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class OracleProblem:
    lp: LP
    dec: Decomposition
    abar: list                 # dense Abar_s
    bbar: list
    rho: float
    eps_rel: float
    abar_flat: np.ndarray = None
    abar_ptr: np.ndarray = None
    bbar_flat: np.ndarray = None

    def __post_init__(self):
        ns = self.dec.n_s()
        self.abar_ptr = np.zeros(self.dec.S + 1, dtype=np.int64)
        self.abar_ptr[1:] = np.cumsum(ns * ns)
        self.abar_flat = np.concatenate([a.ravel() for a in self.abar]) if self.abar else np.zeros(0)
        self.abar_flat = np.ascontiguousarray(self.abar_flat, dtype=np.float64)
        self.bbar_flat = np.ascontiguousarray(np.concatenate(self.bbar) if self.bbar else np.zeros(0), np.float64)
        d = self.dec
        self._keep = [np.ascontiguousarray(a) for a in (self.lp.c, self.lp.lo, self.lp.hi, d.seg_ptr, d.seg_copy,
                                                        d.copy_global, d.sub_ptr)]
        c, lo, hi, seg_ptr, seg_copy, copy_global, sub_ptr = self._keep
        self._st = _Problem(self.lp.n, d.S, d.n_copies, _p(c).value, _p(lo).value, _p(hi).value,
                            _p(seg_ptr).value, _p(seg_copy).value, _p(copy_global).value, _p(sub_ptr).value,
                            _p(self.abar_ptr).value, _p(self.abar_flat).value, _p(self.bbar_flat).value,
                            float(self.rho), float(self.eps_rel))

    @property
    def n(self):
        return self.lp.n

    @property
    def nc(self):
        return self.dec.n_copies

    # ---- single steps (each pinned separately in tests/) ----------------------------------
    def global_update(self, xl, lam):
        x = np.zeros(self.n)
        lib().oracle_global_update(C.byref(self._st), _p(xl), _p(lam), _p(x))
        return x

    def local_update(self, x, lam):
        xl = np.zeros(self.nc)
        lib().oracle_local_update(C.byref(self._st), _p(x), _p(lam), _p(xl))
        return xl

    def dual_update(self, x, xl, lam):
        lam = np.array(lam, dtype=np.float64, copy=True)
        lib().oracle_dual_update(C.byref(self._st), _p(x), _p(xl), _p(lam))
        return lam

    def residuals(self, x, xl, xl_old, lam):
        out = np.zeros(4)
        lib().oracle_residuals(C.byref(self._st), _p(x), _p(xl), _p(xl_old), _p(lam), _p(out))
        return out


def build_problem(f: Feeder, rho: float = 100.0, eps_rel: float = 1e-3, single: bool = False,
                  lp: LP | None = None, coarse: int = 0) -> OracleProblem:
    """LP -> decomposition (coarse runs: reading C25) -> precompute
    (PAPER.md:374-380).  Defaults rho = 100, eps_rel = 1e-3."""
    lp = lp if lp is not None else assemble_lp(f)
    dec = decompose(f, lp, single=single, coarse=coarse)
    ab, bb = [], []
    for s in range(dec.S):
        a, b = precompute(dec.A[s], dec.b[s])
        ab.append(a), bb.append(b)
    return OracleProblem(lp=lp, dec=dec, abar=ab, bbar=bb, rho=rho, eps_rel=eps_rel)


def problem_from_parts(A_list, b_list, cols_list, c, lo, hi, rho=100.0, eps_rel=1e-3, var=None) -> OracleProblem:
    """An OracleProblem from raw subsystems (A_s, b_s, I_s) and global (c, lo, hi) — used by the
    pins that exercise the closed forms on random instances."""
    n = len(c)
    var = var if var is not None else [("x", j, 0) for j in range(n)]
    lp = LP(n=n, c=np.asarray(c, np.float64), lo=np.asarray(lo, np.float64), hi=np.asarray(hi, np.float64),
            var=var, col={v: j for j, v in enumerate(var)})
    S = len(A_list)
    sub_ptr = np.zeros(S + 1, dtype=np.int64)
    for s in range(S):
        sub_ptr[s + 1] = sub_ptr[s] + len(cols_list[s])
    copy_global = np.array([g for I in cols_list for g in I], dtype=np.int32)
    nu = np.bincount(copy_global, minlength=n).astype(np.int64)
    seg_ptr = np.zeros(n + 1, dtype=np.int64)
    seg_ptr[1:] = np.cumsum(nu)
    dec = Decomposition(kind=np.zeros(S, np.int32), comp=np.arange(S, dtype=np.int32), leaf_bus=-np.ones(S, np.int32),
                        rows=[list(range(len(b))) for b in b_list], cols=[list(I) for I in cols_list],
                        A=[np.asarray(a, np.float64) for a in A_list], b=[np.asarray(b, np.float64) for b in b_list],
                        sub_ptr=sub_ptr, copy_global=copy_global, seg_ptr=seg_ptr,
                        seg_copy=np.argsort(copy_global, kind="stable").astype(np.int32), nu=nu)
    ab, bb = [], []
    for s in range(S):
        a, b = precompute(dec.A[s], dec.b[s])
        ab.append(a), bb.append(b)
    return OracleProblem(lp=lp, dec=dec, abar=ab, bbar=bb, rho=rho, eps_rel=eps_rel)


def initial_state(prob: OracleProblem):
    """Algorithm 1 line 1 with the initial point of PAPER.md:495: lambda = 0; each x_s entry
    is 1 if it is a voltage (w) copy, else the midpoint of its bounds if both are finite,
    else 0 (reading C7)."""
    lp, d = prob.lp, prob.dec
    xl = np.zeros(d.n_copies)
    for k in range(d.n_copies):
        g = int(d.copy_global[k])
        role = lp.var[g][0]
        if role == "w":
            xl[k] = 1.0
        elif np.isfinite(lp.lo[g]) and np.isfinite(lp.hi[g]):
            xl[k] = 0.5 * (lp.lo[g] + lp.hi[g])
    return xl, np.zeros(d.n_copies)


@dataclass
class OracleResult:
    converged: bool
    iters: int
    x: np.ndarray
    x_loc: np.ndarray
    lam: np.ndarray
    pres: float
    dres: float
    eps_prim: float
    eps_dual: float
    objective: float
    trace: np.ndarray


def _run(prob: OracleProblem, xl, lam, max_iter: int, test: bool, trace_every: int = 0) -> OracleResult:
    x = np.zeros(prob.n)
    xl = np.array(xl, dtype=np.float64, copy=True)
    lam = np.array(lam, dtype=np.float64, copy=True)
    res = np.zeros(4)
    conv = C.c_int32(0)
    cap = (max_iter // trace_every + 1) if trace_every > 0 else 0
    trace = np.zeros((max(cap, 1), 4))
    nrow = C.c_int64(0)
    k = lib().oracle_run(C.byref(prob._st), _p(x), _p(xl), _p(lam), int(max_iter), int(bool(test)), _p(res),
                         C.byref(conv), _p(trace) if cap else None, cap, int(trace_every), C.byref(nrow))
    return OracleResult(converged=bool(conv.value), iters=int(k), x=x, x_loc=xl, lam=lam, pres=res[0], dres=res[1],
                        eps_prim=res[2], eps_dual=res[3], objective=float(prob.lp.c @ x),
                        trace=trace[: nrow.value].copy())


def solve(prob: OracleProblem, max_iter: int = 1_000_000, trace_every: int = 0, state=None) -> OracleResult:
    """Run Algorithm 1 until (termination) or max_iter."""
    xl, lam = state if state is not None else initial_state(prob)
    return _run(prob, xl, lam, max_iter, True, trace_every)


def run_k(prob: OracleProblem, k: int, state=None) -> OracleResult:
    """Exactly k sweeps with the test disabled (fixed-K parity)."""
    xl, lam = state if state is not None else initial_state(prob)
    return _run(prob, xl, lam, k, False)


# ---- residual balancing (reading F2) ---------------------------------
def solve_adaptive(prob: OracleProblem, every: int = 10, mu: float = 10.0, tau: float = 2.0, max_iter: int = 1_000_000,
                   test: bool = True, state=None):
    """Algorithm 1 with residual balancing of rho every `every` sweeps (oracle_run_adaptive in admm_loop.c).
    Returns (OracleResult, final rho, number of rho changes).  test=False: exactly max_iter sweeps."""
    xl, lam = state if state is not None else initial_state(prob)
    x = np.zeros(prob.n)
    xl = np.array(xl, dtype=np.float64, copy=True)
    lam = np.array(lam, dtype=np.float64, copy=True)
    res = np.zeros(4)
    conv = C.c_int32(0)
    rho = C.c_double(0.0)
    nch = C.c_int64(0)
    k = lib().oracle_run_adaptive(C.byref(prob._st), _p(x), _p(xl), _p(lam), int(max_iter), int(bool(test)), _p(res),
                                  C.byref(conv), int(every), float(mu), float(tau), C.byref(rho), C.byref(nch))
    r = OracleResult(converged=bool(conv.value), iters=int(k), x=x, x_loc=xl, lam=lam, pres=res[0], dres=res[1],
                     eps_prim=res[2], eps_dual=res[3], objective=float(prob.lp.c @ x), trace=np.zeros((0, 4)))
    return r, rho.value, nch.value


# ---- fp32 variant (reading F1) ---------------------------------------
def _f32_struct(prob: OracleProblem):
    """The binary32 copy of the problem: every fp64 datum rounded once to nearest (+-inf preserved)."""
    if getattr(prob, "_st32", None) is None:
        d = prob.dec
        keep = [np.ascontiguousarray(a, dtype=np.float32) for a in (prob.lp.c, prob.lp.lo, prob.lp.hi,
                                                                    prob.abar_flat, prob.bbar_flat)]
        c, lo, hi, ab, bb = keep
        idx = prob._keep
        prob._keep32 = keep
        prob._st32 = _ProblemF32(prob.lp.n, d.S, d.n_copies, _p(c).value, _p(lo).value, _p(hi).value,
                                 _p(idx[3]).value, _p(idx[4]).value, _p(idx[5]).value, _p(idx[6]).value,
                                 _p(prob.abar_ptr).value, _p(ab).value, _p(bb).value,
                                 float(np.float32(prob.rho)), float(prob.rho), float(prob.eps_rel))
    return prob._st32


def _run_f32(prob: OracleProblem, xl, lam, max_iter: int, test: bool) -> OracleResult:
    st = _f32_struct(prob)
    x = np.zeros(prob.n, np.float32)
    xl = np.array(xl, dtype=np.float32, copy=True)
    lam = np.array(lam, dtype=np.float32, copy=True)
    res = np.zeros(4)
    conv = C.c_int32(0)
    k = lib().oracle_run_f32(C.byref(st), _p(x), _p(xl), _p(lam), int(max_iter), int(bool(test)), _p(res),
                             C.byref(conv))
    x64 = x.astype(np.float64)
    return OracleResult(converged=bool(conv.value), iters=int(k), x=x64, x_loc=xl.astype(np.float64),
                        lam=lam.astype(np.float64), pres=res[0], dres=res[1], eps_prim=res[2], eps_dual=res[3],
                        objective=float(prob.lp.c @ x64), trace=np.zeros((0, 4)))


def solve_f32(prob: OracleProblem, max_iter: int = 1_000_000, state=None) -> OracleResult:
    """Algorithm 1 in binary32 (the paper's GPU precision) until (termination) or max_iter."""
    xl, lam = state if state is not None else initial_state(prob)
    return _run_f32(prob, xl, lam, max_iter, True)


def run_k_f32(prob: OracleProblem, k: int, state=None) -> OracleResult:
    """Exactly k binary32 sweeps with the test disabled (fixed-K parity of the fp32 variant)."""
    xl, lam = state if state is not None else initial_state(prob)
    return _run_f32(prob, xl, lam, k, False)
