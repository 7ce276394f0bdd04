#!/usr/bin/env python3
"""Benchmark of the hot path: Q(f,f) evaluations/s at d=3 N=64 N̄=8 (fp64),
BASELINE.json's metric, on config c5 (512 spatial cells of perturbed
Maxwellians, batched dvm_collide_batched calls).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c1|c2|c3|c4|c5] [--scaling strong|weak]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

c5 (default): a step = one full evaluation of the 512 cells (all 2017
directions).  Multi-GPU: the 512 cells are sharded into contiguous blocks of
512/N per rank (--scaling strong, the default, BASELINE c5: "cells sharded
across 1/2/4/8 GPUs"; no data-path collective); --scaling weak gives every rank
512 cells of a global batch of 512 N.  Timed on the device between barriers,
max over ranks.  Inputs (1 GiB at N = 1) exceed the 126 MB L2.

c1-c4 (--workload): one grid per step.  c1, c3, c4: one evaluation; with N > 1
direction-sharded (2D: whole pair units) with one fp64 NCCL all-reduce inside
the timed region.  c2: one evaluation + 100 explicit Euler steps dt = 0.01
(BASELINE c2; 101 evaluations per step, one rank's trajectory; N > 1 runs
independent replicas).

`--impl reference` times the CPU oracle (oracle/, the slow direct pair sum)
on a bounded sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Q(f,f) evals/sec at d=3 N=64 N̄=8, fp64; achieved HBM GB/s vs peak"
UNIT = "evals/s"
D, NGRID, NBAR, L = 3, 64, 8, 8.0
CELLS_PER_RANK = 512


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                      "-i", str(self.idx)], capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, n in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


_NPAIRS = {}


def _oracle_sample(name: str, seconds: float, seed: int, k_fixed: int | None = None):
    """Time the oracle (oracle/dvm_oracle.c as it stands) on a bounded sample of
    workload `name`: whole-grid evaluations when the grid is small, otherwise a
    seeded set of nodes of one cell sized for ~`seconds` of host work.  The
    oracle hands out blocks of 16 nodes per thread (OpenMP dynamic), so the
    sample is a multiple of 16 x threads nodes and every thread is busy.
    k_fixed: a sample size (in blocks of 16 x threads nodes) from an earlier
    call, skipping the calibration.
    Returns (evals/s, busy threads, sample description, seconds, k)."""
    import dvm_inputs
    from oracle import oracle
    cfg = dvm_inputs.CONFIGS[name]
    nodes = cfg.N ** cfg.d
    Nt = oracle.ntilde_rule(cfg.N, cfg.Nbar)
    f = dvm_inputs.make(name, cells=1)[0]
    threads = os.cpu_count() or 1
    block = 16 * threads
    if name not in _NPAIRS:
        _NPAIRS[name] = oracle.pairs(cfg.d, Nt, cfg.Nbar, 1.0)[2].size
    npairs = _NPAIRS[name]
    if nodes <= 4 * block:
        t0 = time.perf_counter()
        oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, diagnostics=False)
        dt = time.perf_counter() - t0
        reps = max(1, min(200, int(seconds / max(dt, 1e-4))))
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, diagnostics=False)
        dt = time.perf_counter() - t0
        busy = min(threads, -(-nodes // 16))
        return reps / dt, busy, (f"{reps} whole-grid evaluations of {name} ({nodes} nodes, {npairs} pairs/node), "
                                 f"{dt:.1f} s"), dt, None
    rng = np.random.default_rng(seed)
    if k_fixed is None:
        # per-call fixed cost (the oracle builds its pair list on every call) and the
        # per-block cost, so the sample is sized on the node work
        t0 = time.perf_counter()
        oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, points=np.zeros(1, np.int64), diagnostics=False)
        t_fix = time.perf_counter() - t0
        pts = np.sort(rng.choice(nodes, size=block, replace=False)).astype(np.int64)
        t0 = time.perf_counter()
        oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, points=pts, diagnostics=False)
        t_blk = max(time.perf_counter() - t0 - t_fix, 1e-3)
        k = int(max(4, min(nodes // block, seconds / t_blk)))  # >= 4 blocks per thread: the pair list is amortised
    else:
        k = k_fixed
    pts = np.sort(rng.choice(nodes, size=k * block, replace=False)).astype(np.int64)
    t0 = time.perf_counter()
    oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, points=pts, diagnostics=False)
    dt = time.perf_counter() - t0
    return ((pts.size / dt) / nodes, threads,
            f"{pts.size} seeded nodes of one {name} cell (of {nodes}), direct pair sum ({npairs} pairs/node), "
            f"{dt:.1f} s; evals/s = nodes/s / {nodes}", dt, k)


def cpu_baseline(name: str = "c5", seconds: float = 15.0):
    value, busy, sample, _, _ = _oracle_sample(name, seconds, 0)
    return {"value": value, "unit": UNIT, "cores": busy, "kind": "oracle", "sample": sample}


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    name = args.workload
    per_step_s = float(os.environ.get("REF_SECONDS_PER_STEP", "3"))
    # calibrate the per-step sample once (warm-up), then time every step on it
    kfix = None
    for w in range(max(1, args.warmup)):
        _, _, _, _, kk = _oracle_sample(name, per_step_s if w == 0 else 0.2, 99, kfix)
        kfix = kk if kfix is None else kfix
    vals, secs = [], 0.0
    busy, sample = 0, ""
    for k in range(args.steps):
        v, busy, sample, dt, _ = _oracle_sample(name, per_step_s, 1 + k, kfix)
        vals.append(v)
        secs += dt
    value = float(np.mean(vals))
    import dvm_inputs
    cfg = dvm_inputs.CONFIGS[name]
    evals_per_step = (cfg.cells if name == "c5" else 101 if name == "c2" else 1)
    ms_per_step = evals_per_step / value * 1e3  # extrapolated: one full step of the workload
    line = {"impl": "reference", "metric": METRIC if name == "c5" else f"Q(f,f) evals/sec, {name}",
            "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded, dvm_inputs {name})",
            "config": {"workload": WORKLOADS[name], "sample_per_step": sample,
                       "timed_host_seconds": secs,
                       "ms_per_step_note": "extrapolated from the timed sample to one full step of the workload "
                                           "(the full oracle step is far longer than the driver's run)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": busy, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


WORKLOADS = {
    "c1": "c1: d=2 Maxwell, N=16, Nbar=4, Ntilde=4, L=8, one grid",
    "c2": "c2: d=2 Maxwell, N=64, Nbar=8, Ntilde=14, L=8, one evaluation + 100 Euler steps dt=0.01",
    "c3": "c3: d=2 Maxwell, N=256, Nbar=16, Ntilde=57, L=8, one grid",
    "c4": "c4: d=3 hard spheres, N=32, Nbar=4, Ntilde=7, L=8, one grid",
    "c5": "c5: d=3 hard spheres, N=64, Nbar=8, Ntilde=14, L=8, 512 batched cells",
}


def _kernel_metrics(name: str):
    """ncu evidence for the dominant kernel, measured on bench.py's own launch
    (profiles/kernel_metrics.json, written from an ncu capture; see profiles/r02)."""
    path = os.path.join(ROOT, "profiles", "kernel_metrics.json")
    try:
        return json.load(open(path)).get(name)
    except Exception:
        return None


# what limits the dominant kernel (ncu evidence in profiles/r02/SUMMARY.md)
BINDING = {
    "k_fg2": "SM L1/shared data pipe (~70%, shared by both warp roles: four register re-arrangements of every "
             "point per step plus misaligned tap loads) and latency (16 warps per SM); fp64 pipe ~29%, issue ~37%; "
             "see DESIGN.md 6 (data-movement floor) and profiles/r02/SUMMARY.md",
    "k_gain3d": "SM L1/shared-memory pipe (sliding-program loads + scattered frame gather/store); "
                "see profiles/r01/SUMMARY.md",
}


def _roofline(prof, psteps, bytes_per_eval, evals_per_step, cells=None, workload=None):
    """roofline object for the dominant kernel: algorithmic (streaming-
    formulation) bytes of the evaluations one launch covers / its CUDA-event
    launch time, against the measured HBM copy bandwidth."""
    total = sum(v[0] for v in prof.values() if v[1]) or 1.0
    top_name, (top_ms, top_n) = max(prof.items(), key=lambda kv: kv[1][0])
    share = top_ms / total
    if share >= 0.9:
        # one kernel is the evaluation: its launches carry the step's algorithmic bytes
        launches_per_step = max(1, top_n // psteps)
        alg_bytes = bytes_per_eval * evals_per_step / launches_per_step
        avg_launch_s = top_ms / top_n / 1e3
        basis = "dominant kernel"
    else:
        # the evaluation is split over several kernels: charge the bytes to the
        # summed device time of all of them (per step), not to the largest one
        alg_bytes = bytes_per_eval * evals_per_step
        avg_launch_s = total / psteps / 1e3
        basis = f"all kernels of the step (largest: {top_name}, {100 * share:.0f}%)"
    peak, peak_src = _peaks()
    achieved = alg_bytes / avg_launch_s / 1e9
    km = _kernel_metrics(top_name) or {}
    if km and km.get("cells") is not None and km.get("cells") != cells:
        km = {}  # the ncu capture was of another launch size: not this launch's counters
    traffic = km.get("dram_bytes_per_launch")
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": traffic, "kernel": top_name, "kernel_share_of_step": top_ms / total,
         "kernel_avg_launch_ms": top_ms / top_n, "algorithmic_bytes_per_launch": alg_bytes,
         "time_basis": basis,
         "peak_source": peak_src,
         "note": "streaming-formulation bytes (A+2)*8*N^d per cell-evaluation (SURVEY.md 8(d)); "
                 "effective, not DRAM traffic",
         "binding_resource": BINDING.get(top_name, "see profiles/r02/SUMMARY.md")}
    if km:
        # SURVEY 8(d)'s other two numbers, from the ncu capture of the same launch
        if traffic:
            r["dram_GBps"] = traffic / avg_launch_s / 1e9
        r["fp64_pipe_pct"] = km.get("fp64_pipe_pct")
        r["l1tex_pct"] = km.get("l1tex_pct")
        r["ncu_source"] = km.get("source")
    elif workload is not None and _kernel_metrics("workload:" + workload):
        # c1-c4: the ncu totals of one whole evaluation (every kernel of it) against
        # this run's per-evaluation device time (libdvm's per-launch events)
        wm = _kernel_metrics("workload:" + workload)
        step_s = total / psteps / 1e3
        r["dram_GBps"] = wm["dram_bytes_per_eval"] * evals_per_step / step_s / 1e9
        r["fp64_pipe_pct"] = round(wm["fp64_pipe_pct"], 2)
        r["l1tex_pct"] = round(wm["l1tex_pct"], 2)
        r["ncu_source"] = wm.get("source")
    return r


def run_ours(args):
    import torch
    import torch.distributed as dist

    import dvm_inputs
    from paper_1201_3986_b200 import Plan
    from paper_1201_3986_b200.parallel import cell_range

    world, rank, local = _dist()
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    nodes = NGRID ** D
    if args.scaling == "strong":
        global_cells = args.cells
        first, cells = cell_range(global_cells, rank, world)
    else:
        global_cells = args.cells * world
        first, cells = rank * args.cells, args.cells
    f_host = dvm_inputs.make("c5", cells=cells, first_cell=first)
    f = torch.from_numpy(f_host).cuda()
    Q = torch.empty_like(f)
    plan = Plan(D, NGRID, NBAR)
    A = plan.A
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        plan.collide(f, Q)
    torch.cuda.synchronize()
    mass_rel = float((Q.sum(dim=1).abs() / Q.abs().sum(dim=1)).max()) if cells else 0.0

    # ---- headline: device-resident inputs, K steps between barriers, CUDA events
    launches0 = plan.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            plan.collide(f, Q)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = plan.launches() - launches0
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = global_cells * args.steps / (ms_total / 1e3)

    # ---- dominant kernel: per-launch CUDA events inside libdvm on the same stream
    plan.profile(True)
    psteps = max(1, min(args.steps, 2))
    for _ in range(psteps):
        plan.collide(f, Q)
    prof = plan.profile_read()
    plan.profile(False)
    roofline = _roofline(prof, psteps, (A + 2) * 8.0 * nodes, cells, cells=cells)
    eff_step_gbs = value / world * (A + 2) * 8.0 * nodes / 1e9

    # ---- e2e through the C ABI with host buffers (pinned), copies inside the timed region
    fh = torch.from_numpy(f_host).pin_memory()
    qh = torch.empty_like(fh).pin_memory()
    plan.collide_host_ptr(fh.data_ptr(), qh.data_ptr(), cells)  # warm (allocates staging)
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.collide_host_ptr(fh.data_ptr(), qh.data_ptr(), cells)
    t1 = time.perf_counter()
    e2e_ms = (t1 - t0) * 1e3
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = global_cells * e2e_steps / (e2e_ms / 1e3)
    # the host variant evaluates large batches in 4 pipelined chunks: equal to the
    # device-resident call up to fp64 summation order (direction chunking)
    qd = Q.cpu()
    e2e_rel = float((qh - qd).abs().max() / qd.abs().max()) if cells else 0.0

    clocks = clk.summary()
    if rank == 0:
        cpu = cpu_baseline("c5") if (world == 1 and not args.no_cpu_baseline) else None
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded c5 Maxwellian cells, dvm_inputs)",
                "config": {"workload": WORKLOADS["c5"], "global_cells": global_cells, "cells_rank0": cells,
                           "directions": A, "parallelism": f"cell-sharded x{world} ({args.scaling})",
                           "l2_flush": "inputs 1 GiB (N=1) > 126 MB L2",
                           "effective_streaming_GBps_per_gpu": eff_step_gbs},
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(fh.numel() * 8),
                        "d2h_bytes_per_step": int(qh.numel() * 8), "max_rel_diff_vs_device": e2e_rel,
                        "pipelined": "4 chunks, copies on 2 streams" if cells >= 256 else "one shot"},
                "gpu_launches": int(launches), "clocks": clocks,
                "checks": {"mass_rel_max": mass_rel},
                "kernel_profile_ms": {k: v[0] / psteps for k, v in prof.items() if v[1]}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_grid(args):
    """c1-c4: one grid per step.  c1/c3/c4: one evaluation (N > 1: direction-
    sharded, 2D by pair units, + one fp64 NCCL sum all-reduce inside the timed
    region); c2: one evaluation + 100 Euler steps on the
    device (CUDA-graph replay), per rank (N > 1: independent replicas)."""
    import torch
    import torch.distributed as dist

    import dvm_inputs
    from paper_1201_3986_b200 import Plan
    from paper_1201_3986_b200.parallel import DirectionSharded, PeerDirectionSharded

    name = args.workload
    cfg = dvm_inputs.CONFIGS[name]
    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    f0 = dvm_inputs.make(name)
    nodes = cfg.N ** cfg.d
    f = torch.from_numpy(f0).cuda()
    q = torch.empty_like(f)
    c2 = name == "c2"
    if c2:
        ev = None
        plan = Plan(cfg.d, cfg.N, cfg.Nbar)
        fw = f.clone()

        def step():
            fw.copy_(f)
            plan.collide(fw, q)
            plan.euler(fw, 0.01, 100)
        evals = 101
    else:
        # --reduce peer: the partials are pushed into every rank's peer window over
        # NVLink and added in rank order (dvm_collide_push / dvm_peer_reduce)
        ev = (PeerDirectionSharded(cfg.d, cfg.N, cfg.Nbar, ncells=1) if args.reduce == "peer"
              else DirectionSharded(cfg.d, cfg.N, cfg.Nbar))
        plan = ev.plan

        def step():
            ev(f, q)
        evals = 1
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    reps = max(20, args.steps) if not c2 else max(3, args.steps)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # the grids fit L2: a 256 MiB write (> the 126 MB L2) before every timed step,
    # outside its event pair, so each step starts with a cold L2
    flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    launches0 = plan.launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with ClockSampler(local) as clk:
        for i in range(reps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    launches = (plan.launches() - launches0) // reps
    ms = sum(a.elapsed_time(b) for a, b in evs) / reps
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = (world if c2 else 1) * evals * 1e3 / ms
    A = plan.A
    # per-launch events inside libdvm; c2's Euler steps 2..100 replay a CUDA graph
    # (no per-launch events), so its roofline is taken on profiled evaluations
    plan.profile(True)
    psteps = 2
    for _ in range(psteps):
        if c2:
            plan.collide(f, q)
        else:
            step()
    prof = plan.profile_read()
    plan.profile(False)
    roofline = _roofline(prof, psteps, (A + 2) * 8.0 * nodes, 1, cells=1, workload=name)
    # e2e with host buffers through the C ABI: f in, Q (and for c2 the final f) out
    fh = torch.from_numpy(f0.copy()).pin_memory()
    qh = torch.empty_like(fh).pin_memory()
    if c2:
        def e2e():
            fw.copy_(fh, non_blocking=True)
            plan.collide(fw, q)
            plan.euler(fw, 0.01, 100)
            qh.copy_(q, non_blocking=True)
            fh.copy_(fw, non_blocking=True)
            torch.cuda.synchronize()
            fh.copy_(torch.from_numpy(f0))
        h2d, d2h = fh.numel() * 8, 2 * fh.numel() * 8
    else:
        def e2e():
            if world > 1:
                f.copy_(fh, non_blocking=True)
                ev(f, q)
                qh.copy_(q, non_blocking=True)
                torch.cuda.synchronize()
            else:
                plan.collide_host_ptr(fh.data_ptr(), qh.data_ptr(), 1)
        h2d, d2h = fh.numel() * 8, fh.numel() * 8
    e2e()
    torch.cuda.synchronize()
    e2e_ms = 0.0
    for i in range(reps):
        flush.fill_(float(i))  # cold L2 for every step, outside the timed call
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e()
        e2e_ms += (time.perf_counter() - t0) * 1e3
    e2e_ms /= reps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    if rank == 0:
        cpu = cpu_baseline(name, 8.0) if (world == 1 and not args.no_cpu_baseline) else None
        red = "one-shot peer-memory reduction" if args.reduce == "peer" else "NCCL all-reduce"
        par = ("replicas" if c2 else f"direction-sharded (2D: pair units) + {red}") + f" x{world}"
        line = {"metric": f"Q(f,f) evals/sec, {name}", "value": value, "unit": UNIT, "n_gpus": world,
                "steps": reps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak" if c2 else "strong", "vs_baseline": None, "dtype": "f64",
                "data": f"synthetic (seeded {name}, dvm_inputs)",
                "config": {"workload": WORKLOADS[name], "evals_per_step": evals, "directions": A,
                           "directions_rank0": plan.info()["A_local"], "parallelism": par,
                           "l2_flush": "256 MiB write before every timed step, outside its timing (per-step CUDA "
                                       "events; e2e: per-call host clock)"},
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": (world if c2 else 1) * evals * 1e3 / e2e_ms, "unit": UNIT,
                        "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
                "gpu_launches": int(launches), "clocks": clk.summary(),
                "kernel_profile_ms": {k: v[0] / psteps for k, v in prof.items() if v[1]}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_dry(args):
    """CPU / gloo rehearsal of the N > 1 plumbing (no GPU): the same sharding
    (c5: cell_range blocks, strong or weak; c1-c4: LPT direction shards, 2D by
    pair units), barrier + max-over-ranks timing and the rank-0 JSON line, with
    the CPU oracle on a few nodes standing in for the kernel (test
    infrastructure; numbers are not measurements)."""
    import torch
    import torch.distributed as dist

    import dvm_inputs
    from oracle import oracle
    from paper_1201_3986_b200 import parallel

    world, rank, _ = _dist()
    if world > 1:
        dist.init_process_group("gloo")
    name = args.workload
    cfg = dvm_inputs.CONFIGS[name]
    Nt = oracle.ntilde_rule(cfg.N, cfg.Nbar)
    nodes = cfg.N ** cfg.d
    pts = np.arange(0, nodes, max(1, nodes // 4))[:4]
    if name == "c5":
        if args.scaling == "strong":
            first, cells = parallel.cell_range(args.cells, rank, world)
            global_cells = args.cells
        else:
            first, cells = rank * args.cells, args.cells
            global_cells = args.cells * world
        f = dvm_inputs.make("c5", cells=min(cells, 2), first_cell=first) if cells else None
        mine = None
    else:
        first, cells, global_cells = 0, 1, 1
        f = dvm_inputs.make(name)
        dirs = oracle.directions(cfg.d, cfg.Nbar)
        M = Nt // np.abs(dirs).max(axis=1)
        owner = parallel.owners_2d(dirs, M, world) if cfg.d == 2 else parallel.lpt_assign(M + 1, world)
        mine = dirs[owner == rank]

    def step():
        if f is None:
            return torch.zeros(len(pts), dtype=torch.float64)
        q, _, _ = oracle.collide(f[:1], cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, points=pts, dirs=mine,
                                 nthreads=1, diagnostics=False)
        q = torch.from_numpy(q[0])
        if name != "c5" and world > 1:
            dist.all_reduce(q, op=dist.ReduceOp.SUM)  # the direction-sharded sum
        return q

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        q = step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got, torch.tensor([first, cells]))
        spans = [g.tolist() for g in got]
    else:
        spans = [[first, cells]]
    if rank == 0:
        print(json.dumps({"dry_run": True, "workload": name, "n_ranks": world, "scaling": args.scaling,
                          "global_cells": global_cells, "rank_spans": spans, "ms_per_step_max": ms,
                          "q_sample": [float(x) for x in q.tolist()]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=CELLS_PER_RANK,
                    help="c5: global cells (strong) or cells per rank (weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reduce", default="nccl", choices=["nccl", "peer"],
                    help="c1/c3/c4 direction shards: NCCL all-reduce or the peer-window push + reduce")
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c5 (default, the BASELINE metric) or one of the single-grid configs")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo rehearsal of the multi-rank plumbing (oracle stand-in, no GPU; not a measurement)")
    args = ap.parse_args()
    if args.dry_run:
        return run_dry(args)
    if args.warmup < 3 and args.impl == "ours":
        print("note: --warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "c5":
        return run_grid(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
