"""Partitioned mode on two GPUs, one process per GPU over NCCL (skipped on a machine with fewer GPUs:
the builder's boxes have one).  The exchange modes -- PyTorch's NCCL allreduce, liblopf's own NCCL
communicator, and the device-initiated exchange over CUDA-IPC-mapped peer memory -- must all
stop at the golden K with the golden objective, and the three final iterates must be
bit-identical."""
import json
import os
import socket

import numpy as np
import pytest

import feedergen as fg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json")))["configs"]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2310_09410_b200 import CONVERGED
    from paper_2310_09410_b200.partition import PartitionedSolver
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        f = fg.make_stitched(2, "8500")
        own = fg.stitched_bus_owner(f, world)
        out = {}
        for mode in ("torch", "nccl", "p2p"):
            sol = PartitionedSolver(f, bus_owner=own, exchange=mode, graph_block=25 if mode != "p2p" else 0)
            sol.reset()
            r = sol.run(200_000, check_every=500)
            out[mode] = (int(r.outcome) == CONVERGED, int(r.iters), sol.objective(), sol.h.get_state()[1])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_gpu_partitioned_modes():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one process per GPU)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    g = GOLD["s2x8500"]
    for rank in (0, 1):
        for mode, (conv, k, obj, xl) in res[rank].items():
            assert conv and k == g["iters"], (rank, mode, k)
            assert abs(obj - g["objective"]) <= 1e-6 * abs(g["objective"])
        xs = [res[rank][m][3] for m in ("torch", "nccl", "p2p")]
        assert np.array_equal(xs[0], xs[1], equal_nan=True) and np.array_equal(xs[0], xs[2], equal_nan=True)
