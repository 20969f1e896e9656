"""Multi-GPU orchestration (plumbing only; every sweep runs in liblopf.so on the rank's own GPU).

Scenario sharding (BASELINE.json configs[3]): the n_scen load scenarios are independent
problems, so rank r of W takes the contiguous slice `shard_range(n_scen, r, W)`, solves it with the batch
kernel on its own device with NO data-path collective, and the per-scenario results are gathered once at
the end (torch.distributed all_gather; NCCL on GPUs, gloo in the CPU tests).

Independent replicas (`bench.py` under torchrun): every rank solves its own feeder; only the timing is
reduced (max over ranks).
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n items for `rank` of `world` (sizes differ by <= 1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank / world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gpu_batch_solver(device=None, max_iter: int | None = None, fixed_k: int | None = None):
    """Local solver for one shard: the batch kernel on `device` (lopf_setup_batch / lopf_solve)."""
    def solve(feeder, scales):
        from .lopf import Lopf
        h = Lopf.setup_batch(feeder, scales, **({} if max_iter is None else {"max_iter": max_iter}))
        h.bind(device or "cuda")
        r = h.run(fixed_k) if fixed_k else h.solve()
        out = h.get_batch_results()
        out["solve_ms"] = np.array([r.solve_ms])
        h.destroy()
        return out
    return solve


def solve_scenarios_sharded(feeder, load_scale: np.ndarray, local_solve=None, group=None) -> dict:
    """Solve all scenarios, sharded over the ranks of `group`; every rank returns the full results
    (iters, outcome, objective [n_scen]; res [n_scen, 4]) in scenario order."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(load_scale.shape[0], rank, world)
    local_solve = local_solve or gpu_batch_solver()
    part = local_solve(feeder, load_scale[lo:hi]) if hi > lo else None
    mine = {"lo": lo, "hi": hi, "part": part}
    if world == 1:
        parts = [mine]
    else:
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
    n = load_scale.shape[0]
    out = {"iters": np.zeros(n, np.int64), "outcome": np.zeros(n, np.int32), "objective": np.zeros(n),
           "res": np.zeros((n, 4)), "solve_ms": np.zeros(world)}
    for r, p in enumerate(parts):
        if p["part"] is None:
            continue
        for k in ("iters", "outcome", "objective", "res"):
            out[k][p["lo"]:p["hi"]] = p["part"][k]
        out["solve_ms"][r] = float(np.max(p["part"].get("solve_ms", [0.0])))
    return out
