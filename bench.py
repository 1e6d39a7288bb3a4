#!/usr/bin/env python
"""bench.py -- CG iterations/s of the tca hot path on B200 (one JSON line).

A step is one pass of the whole hot path over the
config's synthetic input resident in HBM: operator setup (tca_operator_create),
rhs b = (kron A_d^T) y, the config's CG solve (500 iterations for config 3) and
tca_operator_destroy.  `value` = CG iterations/s of the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--dtype f64]
    python bench.py --impl reference ...     # the CPU oracle, bounded sample

The synthetic input (x_true, noise, y = (kron A_d) x_true + 0.01 noise) is made
on the device by the library's seeded generator before the timed region.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "CG iters/s & operator-apply HBM GB/s (fraction of peak), 4D ~30M unknowns"
UNIT = "CG iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tca", choices=["tca", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--iters", type=int, default=None, help="override CG iterations")
    ap.add_argument("--apply-reps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--solver", default="cg", choices=["cg", "pcg", "cgsr", "jacobi"],
                    help="pcg: CG with the Kronecker-factor preconditioner (tca_pcg_solve); "
                         "cgsr: single-reduction CG (tca_cgsr_solve)")
    ap.add_argument("--rtol", type=float, default=None, help="override the config's stop rule")
    ap.add_argument("--workload", default="fit", choices=["fit", "poisson", "scattered"],
                    help="poisson: Fig. 1c's separable Poisson system 128x129x130 (Eq. 9) with tensor "
                         "Jacobi (--solver jacobi, threshold --rtol, default 1e-4) or CG; scattered: Sec. 4's "
                         "spline reconstruction from 9e6 scattered samples on 128x128x128x16")
    ap.add_argument("--samples", type=int, default=None, help="scattered workload: sample count (default 9e6)")
    ap.add_argument("--cfg4-iters", type=int, default=20,
                    help="CG iterations of the config-4 scaling measurement added to the line (0: skip)")
    ap.add_argument("--small-iters", type=int, default=200,
                    help="CG iterations of the config-0/1 latency measurement added to the line (0: skip)")
    return ap.parse_args()


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def spawn_ranks(nproc, script, script_args, env=None):
    """One process per GPU on this node: re-run `script` under torch.distributed.run
    (rendezvous on 127.0.0.1) with the same arguments; rank 0 prints the line.
    Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", script, *script_args]
    return subprocess.call(cmd, env=env)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_name(cfg, dtype, iters, rtol=None, solver="cg"):
    n = "x".join(map(str, cfg.n))
    m = "x".join(map(str, cfg.m))
    rtol = cfg.rtol if rtol is None else rtol
    name = solver.upper()
    stop = f"{iters} {name} iterations" if rtol <= 0 else f"{name} to rel. residual {rtol:g}"
    return f"config {cfg.index}: {n} unknowns {dtype}, data {m}, lambda {cfg.lam:g}, {stop}"


def fit_config(cfg, dtype, iters, rtol, solver, world):
    """The `config` object of the fit workload's line -- identical in the GPU arm
    and the reference (oracle) arm, which times a bounded sample of the same
    workload (described in its cpu_baseline.sample)."""
    esize = 8 if dtype == "f64" else 4
    return {"workload": workload_name(cfg, dtype, iters, rtol, solver), "solver": solver, "config_index": cfg.index,
            "unknowns": cfg.N, "data_points": cfg.Mdata, "cg_iters_per_step": iters,
            "step": "tca_operator_create + tca_rhs + tca_cg_solve (or tca_pcg_solve) + tca_operator_destroy",
            "l2": ("inputs larger than L2 (each vector %.1f MB, y %.1f MB)" if cfg.N * esize * 5 > 126e6 else
                   "vectors L2-resident (each vector %.1f MB, y %.1f MB; 126 MB L2)") % (
                cfg.N * esize / 2**20, cfg.Mdata * esize / 2**20),
            "parallelism": "single GPU" if world == 1 else
            f"mode-1 sharding over {world} GPUs (NCCL halo + all-reduce)"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.out = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self, window=None):
        """Median SM clock and throttle reasons of the samples inside `window`
        (host wall-clock [t0, t1]; all samples if none fall inside)."""
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = out.strip().splitlines()
        if window is not None:
            import datetime
            inside = []
            for line in lines:
                try:
                    ts = datetime.datetime.strptime(line.split(",")[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if window[0] <= ts <= window[1]:
                    inside.append(line)
            if inside:
                lines = inside
        for line in lines:
            parts = [p.strip() for p in line.split(",")][1:]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------- CPU oracle baseline
def cpu_oracle_sample(cfg, iters_target_s, dtype):
    """Oracle CG iterations on the same config, bounded to ~iters_target_s seconds."""
    import oracle
    A, L = synth.mode_matrices(cfg)
    op = oracle.Operator(A, L, cfg.lam)
    b = synth.random_tensor(cfg.n, seed=1)
    t0 = time.perf_counter()
    op.cg(b, rtol=0.0, max_iters=1)
    t1 = time.perf_counter() - t0
    k = int(max(2, min(cfg.max_iters, iters_target_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    _, it, _, _ = op.cg(b, rtol=0.0, max_iters=k)
    el = time.perf_counter() - t0
    return {"value": it / el, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{it} fp64 CG iterations (Fig. 2) of config {cfg.index} from a seeded b; "
                      f"one iteration = apply + 2 dots + 3 updates; setup/rhs excluded"
                      + ("" if dtype == "f64" else "; oracle is fp64 only"),
            "seconds": el}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    iters = args.iters or cfg.max_iters
    rtol = cfg.rtol if args.rtol is None else args.rtol
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    import oracle
    A, L = synth.mode_matrices(cfg)
    op = oracle.Operator(A, L, cfg.lam)
    b = synth.random_tensor(cfg.n, seed=1)
    # bounded per-step sample so that the whole run finishes in a few minutes
    t0 = time.perf_counter()
    op.cg(b, rtol=0.0, max_iters=1)
    t1 = time.perf_counter() - t0
    budget = 150.0 / max(1, args.steps + args.warmup)
    k = int(max(1, min(iters, budget / max(t1, 1e-6))))
    for _ in range(args.warmup):
        op.cg(b, rtol=0.0, max_iters=1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, it, _, _ = op.cg(b, rtol=0.0, max_iters=k)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = args.steps * k / tot
    sample = (f"each step: {k} fp64 CG iterations (Fig. 2) of config {cfg.index} from a seeded b "
              f"(bounded sample of the {iters}-iteration solve)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",   # the oracle computes in fp64
            "data": "synthetic (seeded; cubic B-spline A_d)",
            "config": fit_config(cfg, args.dtype, iters, rtol, args.solver, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def run_tca(args):
    import torch
    from paper_1001_5460_b200 import tca

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev_index = torch.cuda.current_device()
    cfg = synth.CONFIGS[args.config]
    iters = args.iters or cfg.max_iters
    rtol = cfg.rtol if args.rtol is None else args.rtol
    pcg = args.solver == "pcg"
    solver_fn = {"cg": "cg_solve", "pcg": "pcg_solve", "cgsr": "cgsr_solve"}[args.solver]
    dtype = args.dtype
    tdt = torch.float64 if dtype == "f64" else torch.float32
    esize = 8 if dtype == "f64" else 4
    A, L = synth.mode_matrices(cfg)
    stream = torch.cuda.current_stream()

    # ---- distributed plumbing: torch.distributed for the bootstrap and the
    # timing barrier/max; the library's own NCCL communicator for the halo and
    # dot-product exchanges of the sharded operator (mode 1 split over ranks)
    dist_arg, comm, tdist = None, None, None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", rank=rank, world_size=world,
                                 device_id=torch.device("cuda", local))
        uid = bytearray(tca.NcclComm.unique_id() if rank == 0 else bytes(128))
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        tdist.broadcast(t, 0)
        comm = tca.NcclComm(world, bytes(t.cpu().tolist()), rank)
        dist_arg = comm.dist()

    def barrier():
        if tdist is not None:
            tdist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if tdist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    gen = tca.Operator(A, L, cfg.lam, dtype=dtype, dist=dist_arg)
    ydata = gen.forward_model(None, sigma=synth.NOISE_SIGMA, seed=1)  # resident input (shard-local rows)
    local_n, local_m = gen.local_n, gen.local_m
    gen.close()
    torch.cuda.synchronize()

    state = {}
    retired = []

    def step(timing=False):
        h0 = time.perf_counter()
        op = tca.Operator(A, L, cfg.lam, dtype=dtype, dist=dist_arg)  # a1
        if timing:
            op.set_timing(True)
        h1 = time.perf_counter()
        b = op.rhs(ydata)                                               # a2
        h2 = time.perf_counter()
        x, rep = getattr(op, solver_fn)(b, rtol=rtol, max_iters=iters)  # a3-a7
        h3 = time.perf_counter()
        if timing:   # host-side wall split of each timed step (diagnostics)
            state.setdefault("host_ms", []).append(
                [round(1e3 * (h1 - h0), 2), round(1e3 * (h2 - h1), 2), round(1e3 * (h3 - h2), 2),
                 round(rep["seconds"] * 1e3, 2)])
        if timing:
            ms, cnt = op.get_timing()
            state["apply_ms"] = state.get("apply_ms", 0.0) + ms
            state["apply_cnt"] = state.get("apply_cnt", 0) + cnt
        state["iters"] = state.get("iters", 0) + rep["iterations"]
        state["cg_s"] = state.get("cg_s", 0.0) + rep["seconds"]
        state["last_rep"] = rep
        state["path"] = op.apply_path
        op.close()   # tca_operator_destroy: its workspaces return to the stream-ordered pool
        if timing:
            state["host_ms"][-1].append(round(1e3 * (time.perf_counter() - h3), 2))
        return x

    clocks = ClockSampler(dev_index)   # sampling from before the warm-up: no idle gap before timing
    clocks.start()
    for i in range(args.warmup):   # the last warm-up step also takes the timed path (event-pair graphs)
        step(timing=i == args.warmup - 1)
    state.clear()
    barrier()
    t_wall0 = time.time()
    launches0 = tca.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    gc.disable()   # no collector pauses inside the timed steps
    for _ in range(args.steps):
        step(timing=True)
    ev1.record(stream)
    gc.enable()
    barrier()
    launches = tca.kernel_launches() - launches0
    clk = clocks.stop(window=(t_wall0, time.time()))
    total_ms = max_over_ranks(ev0.elapsed_time(ev1))
    for o_ in retired:
        o_.close()
    retired.clear()
    total_iters = state["iters"]            # iterations of the (global) solve
    value = total_iters / (total_ms * 1e-3)
    hbm, peak_src = peaks()

    # dominant kernel: the operator apply inside CG (event pair around every launch,
    # recorded on the launching stream)
    nloc = int(np.prod(local_n))
    apply_us = 1e3 * state["apply_ms"] / max(1, state["apply_cnt"])
    apply_bytes = 2 * nloc * esize  # read p, write q (algorithmic, this rank's shard)
    # (a whole-solve engine -- tca_tiny.cu / tca_grid.cu, small configs -- has no
    # separate apply launches inside CG: the roofline then uses the standalone apply)
    in_cg = state["apply_cnt"] > 0
    achieved = apply_bytes / (apply_us * 1e-6) / 1e9 if in_cg else 0.0
    traffic = None
    try:   # DRAM bytes per launch from the committed ncu --set full capture (tools/ncu_traffic.py)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(f"{cfg.index}-{dtype}")
        if tr and world == 1:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "kernel": "fused banded operator apply q = M p (band_apply_kernel) inside CG",
                "bytes_per_launch": apply_bytes, "us_per_launch": apply_us,
                "launches_timed": state["apply_cnt"], "peak_source": peak_src,
                "timing": "CUDA event pairs on the launching stream around the applies of every 16th CG "
                          "iteration of each captured graph chunk and every eager one, over the timed region"}

    # phase breakdown of one extra step (outside the timed region)
    barrier()
    t0 = time.perf_counter()
    op = tca.Operator(A, L, cfg.lam, dtype=dtype, dist=dist_arg)
    torch.cuda.synchronize()
    create_ms = 1e3 * (time.perf_counter() - t0)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    b = op.rhs(ydata)
    e1.record(stream)
    x, rep = getattr(op, solver_fn)(b, rtol=rtol, max_iters=iters)
    torch.cuda.synchronize()
    rhs_ms = e0.elapsed_time(e1)
    # standalone apply (operator-apply GB/s, the metric's second half)
    xin = torch.empty(local_n, dtype=tdt, device="cuda")
    tca.generate_normal(xin, seed=3, stream_id=7)
    yout = torch.empty_like(xin)
    for _ in range(3):
        op.apply(xin, yout)
    barrier()
    op.set_timing(True)
    for _ in range(args.apply_reps):
        op.apply(xin, yout)
    barrier()
    ams, acnt = op.get_timing()
    op_engine = op.cg_engine
    op.close()
    a_us = 1e3 * ams / acnt
    apply_info = {"us": a_us, "applies_per_s": 1e6 / a_us,
                  "GBps": apply_bytes / (a_us * 1e-6) / 1e9,
                  "frac_hbm": apply_bytes / (a_us * 1e-6) / 1e9 / hbm}
    phases = {"create_ms": create_ms, "rhs_ms": rhs_ms, "cg_ms": rep["seconds"] * 1e3,
              "cg_us_per_iteration": rep["seconds"] * 1e6 / max(1, rep["iterations"]),
              "apply_us_in_cg": apply_us if in_cg else None}
    if not in_cg:
        roofline.update({"achieved": apply_info["GBps"], "frac": apply_info["frac_hbm"], "us_per_launch": a_us,
                         "launches_timed": acnt,
                         "kernel": "operator apply q = M p, standalone (CG ran as one whole-solve kernel, "
                                   f"engine {op_engine})"})

    # ---- north_star's scaling system (config 4: 256^3 x 32 fp64, mode 1 sharded over
    # the ranks) at this N: ms per CG iteration of the device-resident solve (max
    # over ranks), outside the config-3 timed region.  SCALE runs compare it over N.
    scale4 = None
    if args.cfg4_iters > 0 and args.workload == "fit" and args.solver in ("cg", "cgsr"):
        c4 = synth.CONFIGS[4]
        A4, L4 = synth.mode_matrices(c4)
        op4 = tca.Operator(A4, L4, c4.lam, dtype="f64", dist=dist_arg)
        y4 = op4.forward_model(None, sigma=synth.NOISE_SIGMA, seed=1)
        b4 = op4.rhs(y4)
        del y4
        fn4 = getattr(op4, solver_fn if args.solver != "pcg" else "cg_solve")
        fn4(b4, rtol=0.0, max_iters=min(5, args.cfg4_iters))   # warm-up (graph capture)
        op4.set_timing(True)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x4, rep4 = fn4(b4, rtol=0.0, max_iters=args.cfg4_iters)
        e1.record(stream)
        barrier()
        ms4 = max_over_ranks(e0.elapsed_time(e1))
        ams4, acnt4 = op4.get_timing()
        a4_us = max_over_ranks(1e3 * ams4 / max(1, acnt4))
        scale4 = {"workload": f"config 4: {'x'.join(map(str, c4.n))} unknowns f64, data {'x'.join(map(str, c4.m))}, "
                              f"lambda {c4.lam:g}, {args.solver.upper()} from x0 = 0, mode 1 sharded over {world} GPU(s)",
                  "n_gpus": world, "iterations": rep4["iterations"], "ms": ms4,
                  "ms_per_iteration": ms4 / max(1, rep4["iterations"]),
                  "iters_per_s": rep4["iterations"] / (ms4 * 1e-3),
                  "apply_us_per_rank": a4_us, "local_unknowns": int(np.prod(op4.local_n)),
                  "timing": "CUDA events around one device-resident solve, max over ranks"}
        del x4, b4
        op4.close()
        torch.cuda.empty_cache()

    # ---- configs 0-2 (small systems: launch-latency bound): us per CG iteration
    # of a fixed-iteration solve from x0 = 0, rank 0 only, outside the timed
    # region (config 0 runs the single-block engine of tca_tiny.cu, configs 1-2
    # the cooperative-grid engine of tca_grid.cu).
    small = None
    if args.small_iters > 0 and rank == 0 and args.workload == "fit":
        small = {}
        for ci in (0, 1, 2):
            cs = synth.CONFIGS[ci]
            As, Ls = synth.mode_matrices(cs)
            ops = tca.Operator(As, Ls, cs.lam, dtype="f64")
            bs = ops.rhs(torch.from_numpy(synth.data(As, cs.n, cs.m, seed=1)).cuda())
            ops.cg_solve(bs, rtol=0.0, max_iters=min(10, args.small_iters))   # warm-up (graph capture)
            best = None
            for _ in range(3):
                _, reps_s = ops.cg_solve(bs, rtol=0.0, max_iters=args.small_iters)
                us = reps_s["seconds"] * 1e6 / max(1, reps_s["iterations"])
                best = us if best is None else min(best, us)
            small[f"config{ci}"] = {"n": list(cs.n), "iterations": args.small_iters, "cg_us_per_iteration": best,
                                    "engine": ops.cg_engine}
            ops.close()

    e2e = None
    if not args.no_e2e and args.solver == "cg":   # (tca_solve_host runs plain CG)
        yh = torch.empty(local_m, dtype=tdt, pin_memory=True)
        yh.copy_(ydata.cpu())
        xh = torch.empty(local_n, dtype=tdt, pin_memory=True)
        op = tca.Operator(A, L, cfg.lam, dtype=dtype, dist=dist_arg)
        op.solve_host_batch([yh, yh], [xh, xh], rtol=rtol, max_iters=iters)   # warm-up
        op.close()
        # K steps through the pipelined host API: one operator, K data sets; every
        # step's H2D of y and D2H of x run on a copy stream under its neighbours' compute
        e_steps = max(2, args.steps)
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        op = tca.Operator(A, L, cfg.lam, dtype=dtype, dist=dist_arg)
        reps_e = op.solve_host_batch([yh] * e_steps, [xh] * e_steps, rtol=rtol, max_iters=iters)
        op.close()
        it_sum = sum(r["iterations"] for r in reps_e)
        e1.record(stream)
        barrier()
        for o_ in retired:
            o_.close()
        retired.clear()
        wall = time.perf_counter() - t0
        e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": it_sum / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(np.prod(local_m) * esize) * world,
               "d2h_bytes_per_step": int(nloc * esize) * world,
               "wall_value": it_sum / wall,
               "steps": e_steps,
               "path": "tca_operator_create + tca_solve_host_batch over the steps (pinned host y -> rhs -> CG "
                       "-> host x per step; copies overlap the neighbouring steps' compute) + destroy"}

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        cpu = cpu_oracle_sample(cfg, args.cpu_seconds, dtype)

    rep = state["last_rep"]
    if comm is not None:
        comm.close()
    if rank != 0:
        if tdist is not None:
            tdist.destroy_process_group()
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": dtype, "data": "synthetic (seeded counter RNG on device; cubic B-spline A_d)",
        "config": fit_config(cfg, dtype, iters, rtol, args.solver, world),
        "roofline": roofline,
        "apply": apply_info,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "scaling_config4": scale4,
        "small_configs": small,
        "gpu_launches": int(launches),
        "clocks": clk,
        "time_to_solution_ms": total_ms / args.steps,
        "cg_report": {"iterations": rep["iterations"], "rho0": rep["rho0"],
                      "rho_final": rep["rho_final"], "relres_final": rep["relres_final"],
                      "status": rep["status"]},
        "apply_path": state["path"], "cg_engine": op_engine,
        "phases": phases,
        "step_host_ms": state.get("host_ms"),   # [create, rhs enqueue, solve (synchronous), solve device, destroy] per timed step
    }
    print(json.dumps(line), flush=True)
    if tdist is not None:
        tdist.destroy_process_group()
    return 0


def run_poisson(args):
    """Fig. 1c workload: the separable Poisson operator of
    Eq. 9 on a 128x129x130 grid, tensor Jacobi to R+*R <= 1e-4 (or CG), from a
    seeded N(0,1) right-hand side (rhs.dat is not available; reading Z25).  One
    GPU; a step = create + solve + destroy."""
    import torch
    from paper_1001_5460_b200 import tca
    n = synth.POISSON_SHAPE
    T = [synth.laplacian_1d(k) for k in n]
    dtype = args.dtype
    tdt = torch.float64 if dtype == "f64" else torch.float32
    b = torch.empty(n, dtype=tdt, device="cuda")
    tca.generate_normal(b, seed=1, stream_id=9)
    solver = args.solver if args.solver in ("jacobi", "cg", "cgsr") else "jacobi"
    thr = args.rtol if args.rtol is not None else (1e-4 if solver == "jacobi" else 1e-10)
    iters = args.iters or (200000 if solver == "jacobi" else 5000)
    stream = torch.cuda.current_stream()
    state = {}

    def step(timing=False):
        op = tca.Operator.from_gram(None, T, 1.0, dtype=dtype)
        if timing:
            op.set_timing(True)
        fn = {"jacobi": op.jacobi_solve, "cg": op.cg_solve, "cgsr": op.cgsr_solve}[solver]
        kw = {"threshold": thr} if solver == "jacobi" else {"rtol": thr}
        x, rep = fn(b, max_iters=iters, **kw)
        if timing:
            ms, cnt = op.get_timing()
            state["apply_ms"] = state.get("apply_ms", 0.0) + ms
            state["apply_cnt"] = state.get("apply_cnt", 0) + cnt
        state["iters"] = state.get("iters", 0) + rep["iterations"]
        state["rep"] = rep
        state["path"] = op.apply_path
        op.close()

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    for _ in range(args.warmup):
        step()
    state.clear()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(timing=True)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop(window=(t_wall0, time.time()))
    ms = e0.elapsed_time(e1)
    esize = 8 if dtype == "f64" else 4
    N = int(np.prod(n))
    apply_us = 1e3 * state["apply_ms"] / max(1, state["apply_cnt"])
    hbm, src = peaks()
    rep = state["rep"]
    line = {"metric": f"{solver} iterations/s, Fig. 1c separable Poisson", "clocks": clk, "value": state["iters"] / (ms * 1e-3),
            "unit": "iters/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "time_to_solution_ms": ms / args.steps, "higher_is_better": True,
            "dtype": dtype, "data": "synthetic right-hand side N(0,1), seed 1 (rhs.dat not available)",
            "config": {"workload": "Fig. 1c: 128x129x130 separable Poisson (Eq. 9), tridiag(-1,2,-1) factors",
                       "solver": solver, "stop": (f"R+*R <= {thr:g}" if solver == "jacobi" else f"rtol {thr:g}"),
                       "unknowns": N},
            "roofline": {"bound": "hbm", "achieved": 2 * N * esize / (apply_us * 1e-6) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": 2 * N * esize / (apply_us * 1e-6) / 1e9 / hbm,
                         "us_per_launch": apply_us, "peak_source": src},
            "report": {"iterations": rep["iterations"], "converged": rep["converged"], "rho0": rep["rho0"],
                       "rho_final": rep["rho_final"]},
            "apply_path": state["path"]}
    print(json.dumps(line), flush=True)
    return 0


def run_scattered(args):
    """Sec. 4 workload (reading Z27): spline reconstruction from
    scattered samples on the paper's 128x128x128x16 grid with 9e6 samples
    (uniform synthetic coordinates, y = W x_true + N(0, 0.01^2) formed on the GPU
    by the forward model).  One GPU; a step = create (bucketing + upload of the
    samples) + rhs + CG + destroy."""
    import torch
    from paper_1001_5460_b200 import tca
    n = synth.SCATTER_SHAPE
    K = args.samples or synth.SCATTER_K
    dtype = args.dtype
    t = synth.scattered_positions(n, K, seed=1)
    L = [synth.second_difference(k) for k in n]
    lam = 1e-3
    iters = args.iters or 100
    rtol = args.rtol if args.rtol is not None else 0.0
    op0 = tca.Operator.scattered(n, t, L, lam, dtype=dtype)
    yk = op0.forward_model(None, sigma=synth.NOISE_SIGMA, seed=1)   # y = W x_true + noise
    op0.close()
    stream = torch.cuda.current_stream()
    state = {}

    def step(timing=False):
        h0 = time.perf_counter()
        op = tca.Operator.scattered(n, t, L, lam, dtype=dtype)
        torch.cuda.synchronize()
        state["create_ms"] = state.get("create_ms", 0.0) + 1e3 * (time.perf_counter() - h0)
        if timing:
            op.set_timing(True)
        b = op.rhs(yk)
        x, rep = op.cg_solve(b, rtol=rtol, max_iters=iters)
        if timing:
            ms_, cnt = op.get_timing()
            state["apply_ms"] = state.get("apply_ms", 0.0) + ms_
            state["apply_cnt"] = state.get("apply_cnt", 0) + cnt
        state["iters"] = state.get("iters", 0) + rep["iterations"]
        state["cg_ms"] = state.get("cg_ms", 0.0) + rep["seconds"] * 1e3
        state["rep"] = rep
        op.close()

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    for _ in range(args.warmup):
        step()
    state.clear()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(timing=True)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop(window=(t_wall0, time.time()))
    ms = e0.elapsed_time(e1)
    esize = 8 if dtype == "f64" else 4
    N = int(np.prod(n))
    apply_us = 1e3 * state["apply_ms"] / max(1, state["apply_cnt"])
    hbm, src = peaks()
    abytes = 2 * N * esize + K * (32 + 4 + 16)   # x in, q out; per sample coordinates, index, coefficient scratch
    rep = state["rep"]
    line = {"metric": "CG iterations/s, Sec. 4 scattered-data spline reconstruction", "clocks": clk,
            "value": state["iters"] / (ms * 1e-3),
            "unit": "CG iters/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "dtype": dtype,
            "data": "synthetic: uniform sample coordinates (stream 6), y = W x_true + N(0, 0.01^2) (the paper's "
                    "measurements are not available)",
            "config": {"workload": "Sec. 4: 128x128x128x16 cubic B-spline grid, 9e6 scattered samples, lambda 1e-3, "
                                   "second-difference regulariser", "samples": K, "unknowns": N,
                       "cg_iters_per_step": iters, "step": "create + rhs + CG + destroy"},
            "roofline": {"bound": "hbm", "achieved": abytes / (apply_us * 1e-6) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": abytes / (apply_us * 1e-6) / 1e9 / hbm, "us_per_launch": apply_us,
                         "bytes_per_launch": abytes, "peak_source": src,
                         "note": "instruction-issue bound (shared-memory CAS atomics of the sample scatter); "
                                 "see DESIGN.md 6.6"},
            "apply": {"us": apply_us, "ns_per_sample": 1e3 * apply_us / K, "samples_per_s": K / (apply_us * 1e-6)},
            "phases": {"create_ms": state["create_ms"] / args.steps, "cg_ms": state["cg_ms"] / args.steps,
                       "cg_us_per_iteration": 1e3 * state["cg_ms"] / max(1, state["iters"])},
            "report": {"iterations": rep["iterations"], "converged": rep["converged"], "rho0": rep["rho0"],
                       "rho_final": rep["rho_final"]}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start the N ranks here
        if args.impl == "tca":
            import torch
            if torch.cuda.device_count() < args.gpus:
                print(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} visible CUDA "
                      f"device(s)", file=sys.stderr)
                return 2
        return spawn_ranks(args.gpus, os.path.abspath(__file__), sys.argv[1:])
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "poisson":
        return run_poisson(args)
    if args.workload == "scattered":
        return run_scattered(args)
    return run_tca(args)


if __name__ == "__main__":
    sys.exit(main())
