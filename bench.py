#!/usr/bin/env python
"""Benchmark: ADMM iterations/s and time-to-tolerance of Algorithm 1 (arXiv 2310.09410) on the
8500-bus-shaped synthetic feeder (BASELINE.json configs[2]), one solve per step.

A STEP is one full pass of the hot path over one problem: reset to the initial point (a3) and
sweep (a4-a8) until the paper's stopping criterion — so ms_per_step is the
time-to-tolerance and value = iterations / second.  Under torchrun each rank solves its own
independent feeder instance (seed 8500 + rank): the units are independent problems, no
data-path collective ("scaling": "weak").

`--impl reference` times the CPU oracle (oracle/, plain C, one thread) on the same workload:
each step is a bounded sample of sweeps from the initial point.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADMM iterations/sec and time-to-tolerance (8500-bus); HBM GB/s vs peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class Clocks:
    """Sample nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _ncu_traffic(precision: int = 64, shape: str = "8500"):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary of the SAME
    workload (the summaries are of the 8500-shaped config 3; other shapes report null)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json" if precision == 64 else "ncu_summary_f32.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        if f"{shape}-shaped" not in d.get("workload", ""):
            return None, None
        if "dram_bytes_per_sweep" in d:                   # tools/ncu_json.py summaries
            return d["dram_bytes_per_sweep"] * d["sweeps_per_launch"], d["sweeps_per_launch"]
        return d.get("dram_bytes_per_launch"), d.get("iters_per_launch")
    except Exception:
        return None, None


def cpu_oracle_rate(feeder, sweeps: int, openmp: bool = False, prob=None):
    """Oracle sweeps/s on this host from the initial point; setup excluded.  openmp=False: the parity oracle
    (plain C, one thread); True: the same loop built with -fopenmp on every core of this process
    (SURVEY §8(d) mode (ii), timing only)."""
    import oracle
    from oracle.admm import run_k_omp
    p = prob if prob is not None else oracle.build_problem(feeder)
    x0 = oracle.initial_state(p)
    run = run_k_omp if openmp else oracle.run_k
    run(p, 5, state=x0)                                  # warm the C library / the thread pool
    t = time.perf_counter()
    run(p, sweeps, state=x0)
    dt = time.perf_counter() - t
    return sweeps / dt, dt


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _lp_optimum(feeder, shape):
    """HiGHS optimum of the same LP (tests/golden/lp_optimum.json, written from oracle/ only), or None."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "lp_optimum.json")) as fh:
            g = json.load(fh)["configs"][shape]
        return g["objective"] if g["sha256"] == feeder.sha256() else None
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--shape", default="8500", choices=["13", "123", "8500"])
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32],
                    help="32: the fp32 variant (the paper's GPU precision, PAPER.md:414; streaming/batch kernels)")
    ap.add_argument("--cpu-sweeps", type=int, default=6000, help="oracle sweeps timed for cpu_baseline (~10 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-paper-length", action="store_true", help="skip the fixed-K = 15817 run (PAPER.md:510)")
    ap.add_argument("--ref-sweeps", type=int, default=100, help="oracle sweeps per step for --impl reference")
    ap.add_argument("--config", type=int, default=3, choices=[3, 4, 5],
                    help="3: 8500-shaped single solve (default, the headline); 4: 4096 scenarios of the "
                         "123 shape, sharded; 5: 64 x 8500 stitched feeder, partitioned over the ranks")
    ap.add_argument("--sweeps", type=int, default=500, help="config 5: sweeps per step (fixed K, test off)")
    ap.add_argument("--n-sub", type=int, default=64, help="config 5: stitched subfeeders")
    ap.add_argument("--graph-block", type=int, default=50,
                    help="config 5 under torchrun: sweeps per captured CUDA graph (0 = host-launched sweeps)")
    ap.add_argument("--n-scen", type=int, default=4096, help="config 4: scenarios")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl", "torch"],
                    help="config 5 under torchrun: device-initiated exchange over peer memory (one launch per solve), "
                         "liblopf's NCCL communicator, or torch.distributed's allreduce (per-sweep launches)")
    args = ap.parse_args()
    if args.config == 5:
        return bench_stitched(args)
    if args.config == 4:
        return bench_batch(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    import feedergen as fg
    seed = fg.SEEDS[args.shape] + rank
    feeder = fg.make_feeder(args.shape, seed=seed)
    workload = f"ieee{args.shape}-shaped synthetic radial feeder (seed {fg.SEEDS[args.shape]}+rank), single scenario, " \
               f"solve to the paper's stopping criterion (rho=100, eps_rel=1e-3)"

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle
        p = oracle.build_problem(feeder)
        x0 = oracle.initial_state(p)                     # the oracle's own initial point
        for _ in range(args.warmup):
            oracle.run_k(p, args.ref_sweeps, state=x0)
        t = time.perf_counter()
        for _ in range(args.steps):
            oracle.run_k(p, args.ref_sweeps, state=x0)
        dt = time.perf_counter() - t
        v = args.steps * args.ref_sweeps / dt
        sample = f"{args.ref_sweeps} sweeps from the initial point per step (oracle O6 loop only; setup excluded)"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "shape": args.shape},
            "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2310_09410_b200 import Lopf

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    t0 = time.perf_counter()
    h = Lopf.setup(feeder, kernel=args.kernel, precision=args.precision)
    setup_s = time.perf_counter() - t0
    h.bind(dev)
    sz = h.sizes
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)     # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        h.reset()
        h.solve()
    step_ms, kern_ms, iters = [], [], []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()                                                    # L2 flushed between steps
            ev[i][0].record(stream)
            h.reset()
            h.solve_async(int(h.opts.max_iter), True)
            ev[i][1].record(stream)
            r = h.result_get()
            iters.append(int(r.iters))
            kern_ms.append(float(r.solve_ms))
        barrier()
    for i in range(args.steps):
        step_ms.append(ev[i][0].elapsed_time(ev[i][1]))
    dev_ms = sum(step_ms)
    tot_iters = sum(iters)

    # end to end through the public API with host buffers, stream-ordered (no host synchronisation inside a
    # step): step i uploads the packed problem from its pinned host image (lopf_bind, H2D), solves
    # (lopf_solve_async) and copies the result record and x back into pinned host memory
    # (lopf_fetch_async, D2H).  Two handles on two streams: step i+1's upload runs on the copy engine while
    # step i solves; the host only waits for step i-2's fetch before reusing its buffer.
    e2e_steps = max(3, min(2 * args.steps, 40))
    h2 = Lopf.setup(feeder, kernel=args.kernel, precision=args.precision).bind(dev)
    hs, ss = (h, h2), (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    fb = int(sz.fetch_bytes)
    bufs = [torch.empty(fb, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    pending = [False, False]
    barrier()
    t = time.perf_counter()
    e2e_iters = 0
    for i in range(e2e_steps):
        j = i % 2
        if pending[j]:
            done[j].synchronize()
            e2e_iters += int(Lopf.decode_fetch(bufs[j], int(sz.n), with_x=False)[0].iters)
        with torch.cuda.stream(ss[j]):
            hs[j].bind(dev, stream=ss[j])
            hs[j].solve_async(int(h.opts.max_iter), True, stream=ss[j])
            hs[j].fetch_async(bufs[j], stream=ss[j])
            done[j].record(ss[j])
        pending[j] = True
    for j in range(2):
        if pending[j]:
            done[j].synchronize()
            e2e_iters += int(Lopf.decode_fetch(bufs[j], int(sz.n), with_x=False)[0].iters)
    e2e_s = time.perf_counter() - t
    # breakdown of one step (events on one stream): upload, solve, read-back
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    evs[0].record(stream)
    h.bind(dev, stream=stream)
    evs[1].record(stream)
    h.solve_async(int(h.opts.max_iter), True, stream=stream)
    evs[2].record(stream)
    h.fetch_async(bufs[0], stream=stream)
    evs[3].record(stream)
    torch.cuda.synchronize(dev)
    breakdown = {"h2d_ms": evs[0].elapsed_time(evs[1]), "solve_ms": evs[1].elapsed_time(evs[2]),
                 "d2h_ms": evs[2].elapsed_time(evs[3])}
    r_last, _ = Lopf.decode_fetch(bufs[0], int(sz.n))
    objective = float(r_last.objective)
    # paper-length run (15817 sweeps on IEEE 8500): fixed K with the test off, so the sweep rate
    # and the objective are not those of the early stop of the paper's criterion on this instance
    paper = None
    if args.shape == "8500" and not args.no_paper_length:
        k_paper = 15817
        h.reset()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        h.solve_async(k_paper, False, stream=stream)
        b_.record(stream)
        rp = h.result_get(stream=stream)
        paper = {"sweeps": k_paper, "ms": a_.elapsed_time(b_), "us_per_sweep": 1e3 * a_.elapsed_time(b_) / k_paper,
                 "objective": float(rp.objective)}

    # max over ranks
    vals = torch.tensor([dev_ms, float(tot_iters), e2e_s, float(e2e_iters)], dtype=torch.float64, device=dev)
    if world > 1:
        allv = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(allv, vals)
        allv = torch.stack(allv).cpu().numpy()
    else:
        allv = vals.cpu().numpy()[None, :]
    max_ms = float(allv[:, 0].max())
    all_iters = float(allv[:, 1].sum())
    value = all_iters / (max_ms / 1e3)
    e2e_value = float(allv[:, 3].sum()) / float(allv[:, 2].max())

    if rank == 0:
        peak, peak_src = _peaks()
        mean_kern_ms = statistics.mean(kern_ms)
        mean_iters = statistics.mean(iters)
        achieved = sz.alg_bytes * mean_iters / (mean_kern_ms / 1e3) / 1e9
        dram, ncu_iters = _ncu_traffic(args.precision, args.shape) if sz.kernel == 2 else (None, None)   # resident
        traffic = (dram / ncu_iters * mean_iters) if (dram and ncu_iters) else None
        cpu = cpu_omp = None
        if world == 1 and not args.no_cpu_baseline:
            import oracle
            prob = oracle.build_problem(feeder)
            rate, secs = cpu_oracle_rate(feeder, args.cpu_sweeps, prob=prob)
            cpu = {"value": rate, "unit": "iterations/s", "cores": 1, "kind": "oracle",
                   "sample": f"{args.cpu_sweeps} oracle sweeps (O6 loop, plain C, -O2, one thread) of the same "
                             f"ieee{args.shape}-shaped feeder from the initial point; {secs:.1f} s"}
            rate2, secs2 = cpu_oracle_rate(feeder, args.cpu_sweeps, openmp=True, prob=prob)
            cpu_omp = {"value": rate2, "unit": "iterations/s", "cores": _cores(), "kind": "oracle-openmp",
                       "sample": f"{args.cpu_sweeps} sweeps of the oracle loop built with -fopenmp (static split of each "
                                 f"step over {_cores()} cores, SURVEY 8(d) mode (ii)); {secs2:.1f} s"}
        lp_opt = _lp_optimum(feeder, args.shape)
        out = {
            "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": workload, "shape": args.shape, "S": int(sz.S), "n": int(sz.n),
                       "n_copies": int(sz.n_copies), "iters_to_tolerance": iters[0],
                       "time_to_tolerance_ms": statistics.median(step_ms), "l2": "flushed between steps (512 MiB write)",
                       "kernel": "streaming" if sz.kernel == 1 else "resident", "grid": int(sz.grid),
                       "block": int(sz.block), "setup_s": round(setup_s, 3), "objective": objective,
                       "objective_lp": lp_opt,
                       "objective_gap_vs_lp": None if lp_opt is None else (objective - lp_opt) / abs(lp_opt),
                       "paper_length": None if paper is None else dict(paper, objective_gap_vs_lp=None if lp_opt is None
                                                                       else (paper["objective"] - lp_opt) / abs(lp_opt))},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_src,
                         "kernel": ("admm_resident_kernel" if sz.kernel == 2 else "admm_stream_kernel")
                                   + " (one persistent cooperative launch = one solve)",
                         "alg_bytes_per_sweep": int(sz.alg_bytes), "mean_kernel_ms": mean_kern_ms,
                         "us_per_sweep": 1e3 * mean_kern_ms / mean_iters},
            "cpu_baseline": cpu,
            "cpu_baseline_omp": cpu_omp,
            "e2e": {"value": e2e_value, "unit": "iterations/s", "h2d_bytes_per_step": int(sz.upload_bytes),
                    "d2h_bytes_per_step": int(sz.fetch_bytes), "steps": e2e_steps, "breakdown": breakdown,
                    "pipeline": "2 handles x 2 streams: bind (H2D) / solve_async / fetch_async (D2H), no per-step sync"},
            "clocks": clk.summary(),
            "gpu_launches": 2 * args.steps,
        }
        if sz.kernel == 2:
            out["roofline"]["served_from"] = ("SMEM: the resident kernel keeps operators and iterate on chip, so "
                                              "achieved is algorithmic bytes per second, not DRAM traffic")
            out["roofline"]["dram_bytes_per_sweep"] = None if traffic is None else traffic / mean_iters
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def _dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _max_over_ranks(world, dev, *vals):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        allv = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allv, t)
        return torch.stack(allv).cpu().numpy()
    return t.cpu().numpy()[None, :]


def bench_stitched(args):
    """Config 5 (BASELINE.json configs[4]): the 64 x 8500-shaped stitched feeder (~0.84M buses).
    N = 1: the streaming kernel, one persistent launch of --sweeps sweeps per step.  N > 1: the feeder
    partitioned over the ranks (subfeeders to ranks, feedergen.stitched_bus_owner), one NCCL
    sum-allreduce of the exchange buffer per sweep (paper_2310_09410_b200.partition): strong scaling.
    A step is --sweeps sweeps from the initial point with the test off (fixed K for
    iterations/s); time-to-tolerance is measured once after the timed region."""
    import feedergen as fg
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        import oracle
        p = oracle.build_problem(fg.make_stitched(args.n_sub, "8500"))   # the full instance (setup ~1-2 min, untimed)
        x0 = oracle.initial_state(p)
        k = max(1, args.ref_sweeps // 20)                 # ~0.19 s per sweep: a bounded sample per step
        oracle.run_k(p, 1, state=x0)
        t = time.perf_counter()
        for _ in range(args.steps):
            oracle.run_k(p, k, state=x0)
        dt = time.perf_counter() - t
        v = args.steps * k / dt
        sample = (f"{k} oracle sweeps per step (plain C, one thread) of the full {args.n_sub} x 8500 instance "
                  f"({p.dec.n_copies} copies) from the initial point")
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"stitched {args.n_sub} x 8500-shaped feeder (config 5)"},
            "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    import torch
    import torch.distributed as dist
    from paper_2310_09410_b200 import CONVERGED, Lopf
    from paper_2310_09410_b200.partition import PartitionedSolver

    world, rank, local = _dist_setup()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    feeder = fg.make_stitched(args.n_sub, "8500")
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    if world == 1:
        h = Lopf.setup(feeder, kernel=1, max_iter=100_000, precision=args.precision).bind(dev)
        solver = None
    else:
        solver = PartitionedSolver(feeder, device=dev, bus_owner=fg.stitched_bus_owner(feeder, world), max_iter=100_000,
                                   precision=args.precision, graph_block=args.graph_block if args.exchange != "p2p" else 0,
                                   exchange=args.exchange)
        h = solver.h
    setup_s = time.perf_counter() - t0
    sz = h.sizes
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def step(k):
        h.reset()
        if solver is None:
            h.solve_async(k, False)
        else:
            solver.sweeps(k)

    for _ in range(args.warmup):
        step(args.sweeps)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step(args.sweeps)
            ev[i][1].record(stream)
        barrier()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    # time to tolerance (one solve, after the timed region)
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h.reset()
    a.record(stream)
    if solver is None:
        r = h.solve()
    else:
        r = solver.run(100_000, check_every=200)
    b.record(stream)
    barrier()
    ttt_ms = a.elapsed_time(b)
    k_tol = int(r.iters)
    conv = int(r.outcome) == CONVERGED
    # end to end: upload the packed problem from pinned host memory, --sweeps sweeps, x back.  N = 1: stream-
    # ordered like config 3 -- two handles on two streams, step i+1's upload (lopf_bind) on the copy engine
    # while step i solves (lopf_solve_async, test off), result record + x into pinned host memory
    # (lopf_fetch_async); the host waits only for step i-2's fetch.  N > 1: bind, sweeps, get_x per step.
    e2e_steps = 4 if solver is None else 3
    if solver is None:
        h2 = Lopf.setup(feeder, kernel=1, max_iter=100_000, precision=args.precision).bind(dev)
        hs, ss = (h, h2), (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        fb = int(h.sizes.fetch_bytes)
        bufs = [torch.empty(fb, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        pending = [False, False]
        torch.cuda.synchronize(dev)
        barrier()
        t = time.perf_counter()
        for i in range(e2e_steps):
            j = i % 2
            if pending[j]:
                done[j].synchronize()
                _r, x = Lopf.decode_fetch(bufs[j], int(sz.n))
            with torch.cuda.stream(ss[j]):
                hs[j].bind(dev, stream=ss[j])
                hs[j].solve_async(args.sweeps, False, stream=ss[j])
                hs[j].fetch_async(bufs[j], stream=ss[j])
                done[j].record(ss[j])
            pending[j] = True
        for j in range(2):
            if pending[j]:
                done[j].synchronize()
                _r, x = Lopf.decode_fetch(bufs[j], int(sz.n))
        e2e_s = time.perf_counter() - t
        del h2
    else:
        barrier()
        t = time.perf_counter()
        for _ in range(e2e_steps):
            h.bind(dev)
            solver.sweeps(args.sweeps)
            x = h.get_x()
        torch.cuda.synchronize(dev)
        e2e_s = time.perf_counter() - t
    allv = _max_over_ranks(world, dev, dev_ms, e2e_s, ttt_ms)
    max_ms, e2e_max, ttt_max = float(allv[:, 0].max()), float(allv[:, 1].max()), float(allv[:, 2].max())
    value = args.steps * args.sweeps / (max_ms / 1e3)
    if rank == 0:
        peak, peak_src = _peaks()
        us = 1e3 * max_ms / (args.steps * args.sweeps)
        achieved = sz.alg_bytes / (us * 1e-6) / 1e9 / world            # per GPU (alg bytes of the whole feeder)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            import oracle
            n5 = max(1, args.cpu_sweeps // 50)              # ~0.19 s per oracle sweep of the full instance
            tb = time.perf_counter()
            p = oracle.build_problem(feeder)                # the SAME full instance (oracle setup: ~1-2 min)
            build_s = time.perf_counter() - tb
            x0 = oracle.initial_state(p)
            oracle.run_k(p, 1, state=x0)
            tt = time.perf_counter()
            oracle.run_k(p, n5, state=x0)
            dt = time.perf_counter() - tt
            rate = n5 / dt
            cpu = {"value": rate, "unit": "iterations/s", "cores": 1, "kind": "oracle",
                   "sample": f"{n5} oracle sweeps (O6 loop, plain C, -O2, one thread) of the full {args.n_sub} x 8500 "
                             f"instance from the initial point ({dt:.1f} s; oracle setup {build_s:.0f} s, untimed)"}
        dram = None
        try:
            suffix = "_f32" if args.precision == 32 else ""
            with open(os.path.join(ROOT, "profiles", f"ncu_summary_config5{suffix}.json")) as fh:
                dram = json.load(fh).get("dram_bytes_per_sweep")
        except Exception:
            pass
        out = {
            "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": f"stitched {args.n_sub} x 8500-shaped feeder (BASELINE configs[4]): "
                                   f"{feeder.n_bus} buses, one scenario, {args.sweeps} sweeps per step (test off)",
                       "S": int(sz.S), "n": int(sz.n), "n_copies": int(sz.n_copies),
                       "mode": "streaming kernel" if world == 1 else
                       (f"partitioned over {world} ranks, device-initiated exchange (tagged peer stores, one launch)"
                        if args.exchange == "p2p" else f"partitioned over {world} ranks ({args.exchange} NCCL allreduce)"),
                       "iters_to_tolerance": k_tol, "converged": conv, "time_to_tolerance_ms": ttt_max,
                       "l2": "working set >> L2; flushed between steps anyway", "gen_s": round(gen_s, 1),
                       "setup_s": round(setup_s, 1)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": dram, "peak_source": peak_src, "kernel": "admm_stream_kernel",
                         "alg_bytes_per_sweep": int(sz.alg_bytes), "us_per_sweep": us},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_steps * args.sweeps / e2e_max, "unit": "iterations/s",
                    "h2d_bytes_per_step": int(sz.upload_bytes),
                    "d2h_bytes_per_step": int(sz.fetch_bytes) if world == 1 else int(8 * sz.n), "steps": e2e_steps,
                    "pipeline": ("2 handles x 2 streams: bind (H2D) / solve_async / fetch_async (D2H), no per-step sync"
                                 if world == 1 else "bind, sweeps, get_x per step")},
            "clocks": clk.summary(),
            "gpu_launches": args.steps * (1 if world == 1 or args.exchange == "p2p" else 2 * args.sweeps),
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def bench_batch(args):
    """Config 4 (BASELINE.json configs[3]): --n-scen load scenarios of the 123-shaped feeder (kappa ~ U[0.5, 1.5]
    per load, seed 4096), sharded over the ranks with no collective (paper_2310_09410_b200.dist.shard_range);
    each rank solves its shard with the batch kernel (lane = scenario, per-scenario termination).  A step =
    reset + solve of the shard; value = scenario-sweeps / s summed over ranks (strong scaling: the total
    number of scenarios is fixed)."""
    import numpy as np
    import feedergen as fg
    from paper_2310_09410_b200.dist import shard_range
    f = fg.make_feeder("123")
    scales = fg.scenario_scales(f, args.n_scen, seed=4096)
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        import oracle
        t = time.perf_counter()
        sw = 0
        for i in range(args.steps):
            p = oracle.build_problem(fg.scale_loads(f, scales[i % args.n_scen]))
            x0 = oracle.initial_state(p)
            oracle.run_k(p, args.ref_sweeps * 10, state=x0)
            sw += args.ref_sweeps * 10
        dt = time.perf_counter() - t
        v = sw / dt
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "scenario-iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.n_scen} load scenarios of the 123-shaped feeder (config 4)"},
            "cpu_baseline": {"value": v, "unit": "scenario-iterations/s", "cores": 1, "kind": "oracle",
                             "sample": f"{args.ref_sweeps * 10} oracle sweeps of one scenario per step (setup included)"},
            "e2e": {"value": v, "unit": "scenario-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    import torch
    from paper_2310_09410_b200 import Lopf
    world, rank, local = _dist_setup()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    lo, hi = shard_range(args.n_scen, rank, world)
    t0 = time.perf_counter()
    h = Lopf.setup_batch(f, scales[lo:hi], precision=args.precision).bind(dev)
    setup_s = time.perf_counter() - t0
    sz = h.sizes
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        h.reset()
        h.solve()
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sweeps = 0
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            h.reset()
            h.solve_async(int(h.opts.max_iter), True)
            ev[i][1].record(stream)
            h.result_get()
            sweeps += int(h.get_batch_results()["iters"].sum())
        torch.cuda.synchronize(dev)
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    res = h.get_batch_results()
    e2e_steps = 2
    t = time.perf_counter()
    for _ in range(e2e_steps):
        h.bind(dev)
        h.solve()
        h.get_batch_results()
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t
    allv = _max_over_ranks(world, dev, dev_ms, float(sweeps), e2e_s, float(res["iters"].sum()), float(res["iters"].max()))
    max_ms = float(allv[:, 0].max())
    value = float(allv[:, 1].sum()) / (max_ms / 1e3)
    if rank == 0:
        peak, peak_src = _peaks()
        cpu = None
        if world == 1 and not args.no_cpu_baseline:          # the oracle on a bounded sample: one scenario
            n_cpu = 50 * args.cpu_sweeps
            rate, secs = cpu_oracle_rate(fg.scale_loads(f, scales[0]), n_cpu)
            cpu = {"value": rate, "unit": "scenario-iterations/s", "cores": 1, "kind": "oracle",
                   "sample": f"{n_cpu} oracle sweeps (O6 loop, plain C, -O2, one thread) of scenario 0 from the "
                             f"initial point; {secs:.1f} s; the oracle solves scenarios one after another"}
        batch_sweeps = float(allv[:, 4].max())                 # launch length = slowest scenario
        us_per_batch_sweep = 1e3 * (max_ms / args.steps) / batch_sweeps
        # bytes actually moved: converged scenarios freeze, so a batch sweep carries the active share of the
        # per-scenario bytes (sum of per-scenario K over scenarios x max K); the shared operators are <2%
        active = float(allv[:, 3].sum()) / (args.n_scen * batch_sweeps)
        achieved = sz.alg_bytes * active / (us_per_batch_sweep * 1e-6) / 1e9
        traffic = None                                  # ncu dram bytes per batch sweep (committed summary)
        try:
            suffix = "_f32" if args.precision == 32 else ""
            with open(os.path.join(ROOT, "profiles", f"ncu_summary_config4{suffix}.json")) as fh:
                traffic = json.load(fh).get("dram_bytes_per_sweep")
        except Exception:
            pass
        out = {
            "metric": METRIC, "value": value, "unit": "scenario-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": {"workload": f"{args.n_scen} load scenarios of the 123-shaped feeder (BASELINE configs[3]), "
                                   f"kappa ~ U[0.5,1.5] per load (seed 4096), each solved to the stopping criterion",
                       "scenarios_per_rank": hi - lo, "max_iters": int(allv[:, 4].max()),
                       "mean_iters": float(allv[:, 3].sum()) / args.n_scen, "time_to_tolerance_ms": max_ms / args.steps,
                       "l2": "flushed between steps (512 MiB write)", "setup_s": round(setup_s, 1)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_src,
                         "kernel": "admm_batch_kernel" if args.precision == 32 else "admm_batch_team_kernel",
                         "alg_bytes_per_batch_sweep": int(sz.alg_bytes), "active_fraction": active,
                         "us_per_batch_sweep": us_per_batch_sweep},
            "cpu_baseline": cpu,
            "e2e": {"value": float(allv[:, 3].sum()) * e2e_steps / float(allv[:, 2].max()), "unit": "scenario-iterations/s",
                    "h2d_bytes_per_step": int(sz.upload_bytes), "d2h_bytes_per_step": 64 * (hi - lo), "steps": e2e_steps},
            "clocks": clk.summary(),
            "gpu_launches": 2 * args.steps,
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
