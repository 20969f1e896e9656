"""Partitioned mode, host side on CPU.

1. The partition maps liblopf builds (lopf_setup_part: bus / copy owners, boundary-copy exchange slots,
   ghost counts) are consistent and identical on every rank.
2. The exchange protocol, run with the oracle's arithmetic on each rank's share only: every rank keeps
   the full-length arrays but trusts only its own copies; remote copies of the globals it touches
   (ghosts) are refreshed from a sum-allreduce of a zero buffer in which each rank writes only its
   boundary copies (here x_s and lambda; the GPUs send u).  After K sweeps the merged state must
   equal the single-process oracle bit for bit -- single process (allreduce = local sum) and two gloo
   processes (allreduce = torch.distributed.all_reduce), which is the path the GPUs take with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import feedergen as fg
import oracle
from paper_2310_09410_b200 import Lopf


def _feeder(key):
    return {"13": lambda: fg.make_feeder("13"), "123": lambda: fg.make_feeder("123"),
            "s4x13": lambda: fg.make_stitched(4, "13")}[key]()


def _part(f, world, rank=0, owner=None):
    h = Lopf.setup_part(f, rank, world, bus_owner=owner)
    bo, co, bi = h.part_owner(f.n_bus)
    info = h.part_info()
    d = h.get_decomposition()
    h.destroy()
    return bo, co, bi, info, d


@pytest.mark.parametrize("key,world", [("13", 1), ("13", 2), ("123", 3), ("s4x13", 2), ("s4x13", 4)])
def test_partition_maps(key, world):
    f = _feeder(key)
    owner = fg.stitched_bus_owner(f, world) if key.startswith("s") else None
    ref = _part(f, world, 0, owner)
    bo, co, bi, info0, d = ref
    assert set(np.unique(bo)) == set(range(world))                     # every rank owns buses
    if owner is not None:
        assert np.array_equal(bo, owner)
    for s in range(len(d.n_s)):                                         # a subsystem lives on one rank
        cs = co[d.sub_ptr[s]:d.sub_ptr[s + 1]]
        assert (cs == cs[0]).all() if len(cs) else True
    n = int(d.copy_global.max()) + 1
    multi = np.zeros(n, bool)
    for g in range(n):
        multi[g] = len(np.unique(co[d.copy_global == g])) > 1
    assert np.array_equal(bi >= 0, multi[d.copy_global])                # boundary copies = copies of shared globals
    order = sorted(np.nonzero(bi >= 0)[0], key=lambda k: (d.copy_global[k], k))
    assert np.array_equal(bi[order], np.arange(len(order)))             # canonical (global, copy) numbering
    assert info0["n_bnd"] == len(order) and info0["doubles"] == len(order) + 8 * world
    for r in range(world):
        bo_r, co_r, bi_r, info_r, _ = _part(f, world, r, owner)
        assert np.array_equal(bo_r, bo) and np.array_equal(co_r, co) and np.array_equal(bi_r, bi)
        touched = np.unique(d.copy_global[co == r])
        ghosts = np.isin(d.copy_global, touched) & (co != r)
        assert info_r["n_imp"] == int(ghosts.sum())


def _rank_sweeps(p, co, bi, rank, world, k, allreduce):
    """K sweeps of Algorithm 1 on rank `rank`'s copies with the exchange protocol (see module doc)."""
    xl, lam = oracle.initial_state(p)
    xl, lam = xl.copy(), lam.copy()
    mine = co == rank
    nb = int(bi.max()) + 1 if (bi >= 0).any() else 0
    exp = mine & (bi >= 0)
    ghost = ~mine                                                        # the rows this rank may read remotely
    x = None
    for _ in range(k):
        x = p.global_update(xl, lam)                                     # ghosts carry the owners' values
        xn = p.local_update(x, lam)
        ln = p.dual_update(x, xn, lam)
        xl = np.where(mine, xn, xl)
        lam = np.where(mine, ln, lam)
        buf = np.zeros(2 * nb + 8 * world)
        buf[2 * bi[exp]] = xl[exp]
        buf[2 * bi[exp] + 1] = lam[exp]
        buf = allreduce(buf)
        imp = ghost & (bi >= 0)
        xl[imp] = buf[2 * bi[imp]]
        lam[imp] = buf[2 * bi[imp] + 1]
    return x, xl, lam


@pytest.mark.parametrize("key,world,k", [("s4x13", 2, 60), ("123", 3, 40)])
def test_partitioned_protocol_single_process(key, world, k):
    f = _feeder(key)
    owner = fg.stitched_bus_owner(f, world) if key.startswith("s") else None
    _, co, bi, _, _ = _part(f, world, 0, owner)
    p = oracle.build_problem(f)
    x, xl, lam = _lockstep(p, co, bi, world, k)
    ref = oracle.run_k(p, k)
    assert np.array_equal(xl, ref.x_loc) and np.array_equal(lam, ref.lam)
    assert np.array_equal(x, ref.x)


def _lockstep(p, co, bi, world, k):
    """All ranks in one process, one sweep at a time; returns the merged (x, x_loc, lambda)."""
    xl0, lam0 = oracle.initial_state(p)
    st = [(None, xl0.copy(), lam0.copy()) for _ in range(world)]
    nb = int(bi.max()) + 1 if (bi >= 0).any() else 0
    for _ in range(k):
        bufs, new = [], []
        for r in range(world):
            _, xl, lam = st[r]
            mine = co == r
            x = p.global_update(xl, lam)
            xn = p.local_update(x, lam)
            ln = p.dual_update(x, xn, lam)
            xl = np.where(mine, xn, xl)
            lam = np.where(mine, ln, lam)
            exp = mine & (bi >= 0)
            buf = np.zeros(2 * nb + 8 * world)
            buf[2 * bi[exp]] = xl[exp]
            buf[2 * bi[exp] + 1] = lam[exp]
            bufs.append(buf)
            new.append((x, xl, lam))
        total = np.sum(bufs, axis=0)
        st = []
        for r, (x, xl, lam) in enumerate(new):
            imp = (co != r) & (bi >= 0)
            xl, lam = xl.copy(), lam.copy()
            xl[imp] = total[2 * bi[imp]]
            lam[imp] = total[2 * bi[imp] + 1]
            st.append((x, xl, lam))
    # merge: a copy from its owner; x_g from the owner of g's first copy
    cg = p.dec.copy_global
    first = np.asarray(p.dec.seg_copy)[np.asarray(p.dec.seg_ptr)[:-1]]
    x = np.array([st[co[first[g]]][0][g] for g in range(p.n)])
    xl = np.array([st[co[c]][1][c] for c in range(len(cg))])
    lam = np.array([st[co[c]][2][c] for c in range(len(cg))])
    return x, xl, lam


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, k, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f = fg.make_stitched(4, "13")
    owner = fg.stitched_bus_owner(f, world)
    h = Lopf.setup_part(f, rank, world, bus_owner=owner)                # this rank's maps from liblopf
    _, co, bi = h.part_owner(f.n_bus)
    h.destroy()
    p = oracle.build_problem(f)

    def allreduce(buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        return t.numpy()

    x, xl, lam = _rank_sweeps(p, co, bi, rank, world, k, allreduce)
    q.put((rank, co.tolist(), x.tolist(), xl.tolist(), lam.tolist()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_partitioned_protocol_gloo():
    world, k = 2, 60
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, k, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted([q.get(timeout=240) for _ in range(world)])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    f = fg.make_stitched(4, "13")
    p = oracle.build_problem(f)
    ref = oracle.run_k(p, k)
    co = np.array(got[0][1])
    first = np.asarray(p.dec.seg_copy)[np.asarray(p.dec.seg_ptr)[:-1]]
    x = np.array([got[co[first[g]]][2][g] for g in range(p.n)])
    xl = np.array([got[co[c]][3][c] for c in range(len(co))])
    lam = np.array([got[co[c]][4][c] for c in range(len(co))])
    assert np.array_equal(xl, ref.x_loc) and np.array_equal(lam, ref.lam) and np.array_equal(x, ref.x)
