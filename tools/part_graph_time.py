"""Partitioned loop on one GPU with a one-rank NCCL group: host-launched sweeps vs CUDA-graph replays
(per sweep: cooperative sweep launch + NCCL allreduce of the exchange buffer + import launch).
Usage: python tools/part_graph_time.py [n_sub] [K]"""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200.partition import PartitionedSolver  # noqa: E402

n_sub = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K = int(sys.argv[2]) if len(sys.argv) > 2 else 500
with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
f = fg.make_stitched(n_sub, "8500")
for gb in (0, 50):
    sol = PartitionedSolver(f, rank=0, world=1, always_reduce=True, graph_block=gb, max_iter=100_000)
    sol.sweeps(100)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        sol.reset()
        torch.cuda.synchronize()
        t = time.perf_counter()
        sol.sweeps(K)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t) / K * 1e6)
    print(f"stitched {n_sub} x 8500, graph_block={gb}: {best:.1f} us per sweep (wall, incl. allreduce)", flush=True)
dist.destroy_process_group()
