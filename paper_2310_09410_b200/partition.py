"""Partitioned mode (BASELINE.json configs[4]): one feeder split over the
ranks of a torch.distributed group, one GPU per rank.

Every sweep of Algorithm 1 runs in liblopf on each rank's own subsystems
(`lopf_part_sweep`); the only data that crosses ranks is the exchange buffer: the u values of the
boundary copies (copies of globals shared by two ranks) plus five residual sums per rank.  Each slot
is written by exactly one rank and the buffer is zero elsewhere, so one sum-allreduce (NCCL over
NVLink on GPUs) is an exact gather; `lopf_part_import` then fills the ghost slots, takes the
termination decision on the rank-ordered sums (identical everywhere) and clears the buffer.  The
paper's own multi-GPU runs stage the same exchange through the host with MPI.

PyTorch here is plumbing only (the arena tensor, the stream, the process group and its allreduce).
Two more exchange modes: liblopf's own NCCL communicator (`exchange="nccl"`), and the
device-initiated exchange over peer memory (`exchange="p2p"`) that needs no per-sweep launch.
"""
from __future__ import annotations

import numpy as np

from .lopf import CONVERGED, Lopf


class PartitionedSolver:
    """This rank's share of a partitioned feeder.  All ranks construct it with the same feeder and
    options; `solve` / `run` are collective calls.

    exchange = "torch": per sweep lopf_part_sweep, torch.distributed.all_reduce of the exchange buffer,
               lopf_part_import (the PyTorch NCCL communicator);
               "nccl":  the same three steps inside liblopf with its own NCCL communicator (lopf_part_step;
               the id is created on rank 0 and broadcast once through torch.distributed);
               "p2p":   the device-initiated exchange: every rank's entry buffer mapped into every
               process by CUDA IPC once, then ONE persistent launch per solve (lopf_part_solve_p2p) -- no host
               and no collective library in the sweep loop."""

    def __init__(self, feeder, group=None, device=None, bus_owner=None, rank=None, world=None, graph_block=0,
                 always_reduce=False, exchange="torch", **opts):
        """graph_block > 0: `sweeps` / `run` replay a CUDA graph of `graph_block` captured sweeps (launch,
        allreduce, import per sweep) instead of launching every sweep from the host.  always_reduce: run the
        allreduce even with one rank (tests the captured collective on a single GPU)."""
        import torch
        import torch.distributed as dist
        if exchange not in ("torch", "nccl", "p2p"):
            raise ValueError("exchange must be 'torch', 'nccl' or 'p2p'")
        self.group = group
        self.exchange_mode = exchange
        self.graph_block = int(graph_block)
        self.always_reduce = bool(always_reduce)
        self._graph = None
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank, self.world = int(rank), int(world)
        self.feeder = feeder
        self.h = Lopf.setup_part(feeder, self.rank, self.world, bus_owner=bus_owner, **opts)
        self.h.bind(device or (torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cuda"))
        self.xbuf = self.h.exchange()
        if exchange == "nccl":
            uid = [Lopf.nccl_unique_id() if self.rank == 0 else None]
            if self.world > 1:
                dist.broadcast_object_list(uid, src=0, group=self.group)
            self.h.part_nccl_init(uid[0])
        elif exchange == "p2p":
            own = self.h.p2p_entries()
            recs = [Lopf.ipc_export(own)]
            if self.world > 1:
                recs = [None] * self.world
                dist.all_gather_object(recs, Lopf.ipc_export(own), group=self.group)
            ptrs = [own if q == self.rank else self.h.ipc_open(recs[q]) for q in range(self.world)]
            self.h.part_connect(ptrs)
            torch.cuda.synchronize()

    def _barrier(self):
        import torch
        torch.cuda.synchronize()
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)

    def solve_p2p(self, max_iter: int, test: bool = True, stream=None):
        """exchange = "p2p": up to max_iter sweeps in one launch per rank (collective: every rank's launch
        runs at the same time); returns this rank's lopf_result."""
        self._barrier()                                  # every rank reset / connected before any launch
        self.h.part_solve_p2p(max_iter, test, stream)
        return self.h.result_get(stream)

    def _allreduce(self):
        if self.world > 1 or self.always_reduce:
            import torch.distributed as dist
            dist.all_reduce(self.xbuf, group=self.group)

    def sweep(self, stream=None):
        """One sweep on every rank (collective).  The three steps are ordered on one stream: a given
        stream becomes torch's current stream for the allreduce too."""
        import contextlib
        import torch
        if stream is None:
            ctx = contextlib.nullcontext()
        elif isinstance(stream, int):
            ctx = torch.cuda.stream(torch.cuda.ExternalStream(stream))
        else:
            ctx = torch.cuda.stream(stream)
        with ctx:                                     # everything on torch's current stream
            if self.exchange_mode == "nccl":
                self.h.part_step(None)
            else:
                self.h.part_sweep(None)
                self._allreduce()
                self.h.part_import(None)

    def reset(self, stream=None):
        self.h.reset(stream)

    def _captured(self):
        """The CUDA graph of graph_block sweeps (captured once; the arena, and so every kernel argument,
        stays where bind put it).  The sweep count lives on the device, so replays continue the iteration,
        and after (termination) every captured kernel returns at once."""
        import torch
        if self._graph is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):                # warm the collective outside the capture
                self._allreduce()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            self.xbuf.zero_()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(self.graph_block):
                    self.sweep()
            self._graph = g
        return self._graph

    def sweeps(self, k: int, stream=None):
        """k sweeps on every rank (collective): graph replays of graph_block sweeps, then single sweeps."""
        if self.exchange_mode == "p2p":
            self.solve_p2p(k, False, stream)
            return
        done = 0
        if self.graph_block > 0:
            g = self._captured()
            while k - done >= self.graph_block:
                g.replay()
                done += self.graph_block
        for _ in range(k - done):
            self.sweep(stream)

    def run(self, k: int, check_every: int = 64, stream=None):
        """Up to k sweeps, stopping early at (termination); polls the device result every
        `check_every` sweeps (the kernels become no-ops once the test has fired)."""
        if self.exchange_mode == "p2p":
            return self.solve_p2p(k, True, stream)
        if self.graph_block > 0:
            check_every = max(self.graph_block, check_every // self.graph_block * self.graph_block)
        done = 0
        r = None
        while done < k:
            n = min(check_every, k - done)
            self.sweeps(n, stream)
            done += n
            r = self.h.result_get(stream)
            if r.outcome == CONVERGED:
                break
        return r if r is not None else self.h.result_get(stream)

    def gather_x(self) -> np.ndarray:
        """The full solution x (each global from the rank holding its first copy)."""
        x = self.h.get_x()
        if self.world > 1:
            import torch.distributed as dist
            parts = [None] * self.world
            dist.all_gather_object(parts, x, group=self.group)
            return merge_owned(parts)
        return x

    def objective(self) -> float:
        """c^T x summed over the ranks' shares."""
        share = float(self.h.result_get().objective)
        if self.world > 1:
            import torch.distributed as dist
            parts = [None] * self.world
            dist.all_gather_object(parts, share, group=self.group)
            return float(sum(parts))
        return share


def merge_owned(parts) -> np.ndarray:
    """Combine per-rank arrays that are NaN where another rank owns the entry."""
    out = np.array(parts[0], copy=True)
    for p in parts[1:]:
        m = ~np.isnan(p)
        out[m] = p[m]
    return out


def emulate_sweeps(handles, k: int, xbufs=None):
    """Test helper: k sweeps of several partitioned handles of ONE process (one device), the
    allreduce replaced by a device-side sum of their exchange buffers.  Every launch is stream-ordered
    after the previous one, so no kernel waits on another rank's kernel."""
    xbufs = xbufs or [h.exchange() for h in handles]
    for _ in range(k):
        for h in handles:
            h.part_sweep()
        total = xbufs[0].clone()
        for xb in xbufs[1:]:
            total += xb
        for xb in xbufs:
            xb.copy_(total)
        for h in handles:
            h.part_import()
    return xbufs
