"""Partitioned mode on one GPU (config 5): the ranks of a partitioned feeder run as
several handles of one process, their exchange buffers summed on the device between the sweep and the
import launches (every launch stream-ordered; no kernel waits on another's).  The merged iterates must
equal the single-GPU streaming kernel bit for bit (each rank computes the same per-copy arithmetic and
adds a boundary global's copies in canonical order), and K / the objective must match the oracle's
golden values.  Multi-GPU NCCL runs use the same library calls with a real allreduce."""
import json
import os

import numpy as np
import pytest

import feedergen as fg
from paper_2310_09410_b200 import CONVERGED, Lopf
from paper_2310_09410_b200.partition import emulate_sweeps, merge_owned

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json")))["configs"]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _feeder(key):
    return {"123": lambda: fg.make_feeder("123"), "s4x13": lambda: fg.make_stitched(4, "13"),
            "s2x8500": lambda: fg.make_stitched(2, "8500")}[key]()


def _ranks(f, world, owner=None, precision=64):
    return [Lopf.setup_part(f, r, world, bus_owner=owner, precision=precision).bind("cuda") for r in range(world)]


def _merged_state(hs):
    xs, xls, lams = zip(*[h.get_state() for h in hs])
    return merge_owned(xs), merge_owned(xls), merge_owned(lams)


@pytest.mark.parametrize("key,world,natural", [("s4x13", 2, True), ("s4x13", 4, True), ("123", 3, False),
                                               ("s2x8500", 2, True), ("s2x8500", 3, False)])
def test_partitioned_equals_single_gpu(torch_cuda, key, world, natural):
    f = _feeder(key)
    owner = fg.stitched_bus_owner(f, world) if natural else None
    hs = _ranks(f, world, owner)
    single = Lopf.setup(f, kernel=1).bind("cuda")
    xb = None
    done = 0
    for k in (1, 7, 50):
        xb = emulate_sweeps(hs, k - done, xb)
        single.run(k - done)
        done = k
        for a, b in zip(_merged_state(hs), single.get_state()):
            assert not np.isnan(a).any()
            assert np.array_equal(a, b)
    for h in hs:
        r = h.result_get()
        assert r.iters == done


@pytest.mark.parametrize("key,world", [("s4x13", 2), ("s2x8500", 2)])
def test_partitioned_k_to_tolerance(torch_cuda, key, world):
    f = _feeder(key)
    g = GOLD[key]
    hs = _ranks(f, world, fg.stitched_bus_owner(f, world))
    xb = None
    for _ in range(200_000 // 100):
        xb = emulate_sweeps(hs, 100, xb)
        rs = [h.result_get() for h in hs]
        if rs[0].outcome == CONVERGED:
            break
    assert all(r.outcome == CONVERGED and r.iters == g["iters"] for r in rs), [(r.outcome, r.iters) for r in rs]
    obj = sum(r.objective for r in rs)
    assert abs(obj - g["objective"]) <= 1e-6 * abs(g["objective"])
    assert len({(r.pres, r.dres, r.eps_prim, r.eps_dual) for r in rs}) == 1        # one decision everywhere


def test_graph_captured_sweeps_with_nccl(torch_cuda):
    """The partitioned loop as a CUDA graph (PartitionedSolver(graph_block=...)): per captured sweep the
    cooperative sweep launch, an NCCL sum-allreduce of the exchange buffer (a one-rank NCCL group, so no
    kernel waits on another GPU) and the import launch.  Graph replays must equal host-launched sweeps bit
    for bit, and the solve must stop at the golden K with the golden objective."""
    import socket

    import torch.distributed as dist
    from paper_2310_09410_b200.partition import PartitionedSolver
    own = not dist.is_initialized()
    if own:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        f = _feeder("s2x8500")
        g = GOLD["s2x8500"]
        eager = PartitionedSolver(f, rank=0, world=1, always_reduce=True)
        graph = PartitionedSolver(f, rank=0, world=1, always_reduce=True, graph_block=25)
        eager.sweeps(60)
        graph.sweeps(60)                                  # two replays + ten host-launched sweeps
        for a, b in zip(eager.h.get_state(), graph.h.get_state()):
            assert np.array_equal(a, b)
        graph.reset()
        r = graph.run(200_000, check_every=500)
        assert r.outcome == CONVERGED and r.iters == g["iters"], (r.outcome, r.iters)
        assert abs(r.objective - g["objective"]) <= 1e-6 * abs(g["objective"])
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("key,world,natural", [("s4x13", 2, True), ("s4x13", 4, True), ("123", 3, False),
                                               ("s2x8500", 2, True), ("s2x8500", 4, False)])
def test_p2p_emulation_equals_single_gpu(torch_cuda, key, world, natural):
    """the device-initiated exchange (lopf_part_emulate: every rank's share in one cooperative
    launch, exchanging through the same peer-store / flag protocol as one process per GPU) gives iterates
    bit-identical to the single-GPU streaming kernel after fixed K, across launches (state, flags and
    exchange parity carry over)."""
    f = _feeder(key)
    owner = fg.stitched_bus_owner(f, world) if natural else None
    hs = _ranks(f, world, owner)
    for h in hs:
        h.reset()
    single = Lopf.setup(f, kernel=1).bind("cuda")
    done = 0
    for k in (1, 7, 50):
        Lopf.part_emulate(hs, k - done, test=False)
        single.run(k - done)
        done = k
        for a, b in zip(_merged_state(hs), single.get_state()):
            assert not np.isnan(a).any()
            assert np.array_equal(a, b)
    assert all(h.result_get().iters == 43 for h in hs)            # the last launch's sweeps


@pytest.mark.parametrize("key,world", [("s4x13", 2), ("s2x8500", 2), ("s2x8500", 4)])
def test_p2p_emulation_k_to_tolerance(torch_cuda, key, world):
    f = _feeder(key)
    g = GOLD[key]
    hs = _ranks(f, world, fg.stitched_bus_owner(f, world) if world <= 2 else None)
    for h in hs:
        h.reset()
    Lopf.part_emulate(hs, 1_000_000, test=True)
    rs = [h.result_get() for h in hs]
    assert all(r.outcome == CONVERGED and r.iters == g["iters"] for r in rs), [(r.outcome, r.iters) for r in rs]
    assert abs(sum(r.objective for r in rs) - g["objective"]) <= 1e-6 * abs(g["objective"])
    assert len({(r.pres, r.dres, r.eps_prim, r.eps_dual) for r in rs}) == 1        # one decision everywhere


def test_p2p_single_rank_solve(torch_cuda):
    """world = 1: lopf_part_solve_p2p runs without peers (its own tables) and equals the streaming kernel."""
    f = _feeder("s2x8500")
    h = Lopf.setup_part(f, 0, 1).bind("cuda")
    h.reset()
    h.part_solve_p2p(300, test=False)
    s = Lopf.setup(f, kernel=1).bind("cuda")
    s.run(300)
    for a, b in zip(h.get_state(), s.get_state()):
        assert np.array_equal(a, b)


def test_library_owned_nccl_step(torch_cuda):
    """exchange="nccl": liblopf's own NCCL communicator (one rank, so no kernel waits on another GPU):
    lopf_part_step sweeps equal host-launched torch-allreduce sweeps bit for bit, eager and graph-captured."""
    import socket

    import torch.distributed as dist
    from paper_2310_09410_b200.partition import PartitionedSolver
    own = not dist.is_initialized()
    if own:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        f = _feeder("s4x13")
        a = PartitionedSolver(f, rank=0, world=1, always_reduce=True)
        b = PartitionedSolver(f, rank=0, world=1, exchange="nccl")
        c = PartitionedSolver(f, rank=0, world=1, exchange="nccl", graph_block=20)
        for s_ in (a, b, c):
            s_.reset()
            s_.sweeps(70)
        for x, y, z in zip(a.h.get_state(), b.h.get_state(), c.h.get_state()):
            assert np.array_equal(x, y) and np.array_equal(x, z)
    finally:
        if own:
            dist.destroy_process_group()


def test_p2p_emulation_fp32_equals_single_gpu(torch_cuda):
    """The device-initiated exchange in the fp32 variant (reading F1): u travels widened to fp64 in the
    tagged entries and is rounded back exactly, so 3 emulated ranks equal the fp32 streaming kernel bit for bit."""
    f = _feeder("s4x13")
    hs = _ranks(f, 3, None, precision=32)
    for h in hs:
        h.reset()
    single = Lopf.setup(f, kernel=1, precision=32).bind("cuda")
    Lopf.part_emulate(hs, 120, test=False)
    single.run(120)
    for a, b in zip(_merged_state(hs), single.get_state()):
        assert np.array_equal(a, b)
