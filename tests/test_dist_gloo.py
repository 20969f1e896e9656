"""Multi-process host logic on CPU (gloo, world_size 2): scenario sharding covers every scenario exactly
once and the gathered results equal a single-process run; the same oracle is the local solver, so the
test exercises the sharding / gathering code path the GPUs use."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import feedergen as fg
from paper_2310_09410_b200.dist import shard_range, solve_scenarios_sharded


def test_shard_range_partition():
    for n in (0, 1, 7, 4096, 4097):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _oracle_solver(k):
    def solve(feeder, scales):
        import oracle
        it, oc, ob, rs = [], [], [], []
        for s in scales:
            p = oracle.build_problem(fg.scale_loads(feeder, s))
            r = oracle.solve(p, max_iter=k)
            it.append(r.iters), oc.append(0 if r.converged else 2), ob.append(r.objective)
            rs.append([r.pres, r.dres, r.eps_prim, r.eps_dual])
        return {"iters": np.array(it), "outcome": np.array(oc), "objective": np.array(ob), "res": np.array(rs)}
    return solve


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f = fg.make_feeder("13")
    K = fg.scenario_scales(f, 5, seed=7)
    out = solve_scenarios_sharded(f, K, local_solve=_oracle_solver(400))
    q.put((rank, out["iters"].tolist(), out["objective"].tolist()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = fg.make_feeder("13")
    K = fg.scenario_scales(f, 5, seed=7)
    ref = _oracle_solver(400)(f, K)
    for rank, iters, obj in got:
        assert iters == ref["iters"].tolist()                       # every rank holds the full result
        assert np.allclose(obj, ref["objective"], rtol=0, atol=0)
