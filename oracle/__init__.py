"""CPU ORACLE for arXiv 2310.09410 (Ryu, Byeon, Kim) — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA path
(`paper_2310_09410_b200/`) is checked against.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  It shares no code with the product path: its only common
dependency is the seeded input generator `feedergen`, which holds no arithmetic
of the method.

Layout (each function cites the PAPER.md passage it follows):

* `lp`          LP assembly (eqs. (2)-(5), LP_model)
* `decompose`   component decomposition + consensus maps
* `precompute`  Abar_s, bbar_s by the literal definition + row reduction
* `admm`        Algorithm 1 — the iteration itself is `admm_loop.c`
                (plain C, -O2 -ffp-contract=off, one thread), driven from Python via ctypes
* `lp_reference` brute-force LP solutions (vertex enumeration, HiGHS) and the KKT checker
                used to pin the oracle

Readings of the paper where it is silent or garbled are listed in DESIGN.md §3
(C1 ... C23 follow SURVEY.md §8(c)).  Functions whose parity has no pin say
"parity unpinned" in their docstring; currently: none of the arithmetic, only
the comparison with Table V's iteration counts (needs the real IEEE feeders).
"""
from .lp import assemble_lp, LP  # noqa: F401
from .decompose import decompose, Decomposition  # noqa: F401
from .precompute import precompute, row_rank_reduce  # noqa: F401
from .admm import OracleProblem, build_problem, initial_state, solve, run_k, solve_f32, run_k_f32, solve_adaptive  # noqa: F401
