#!/usr/bin/env python
"""Benchmark of the B200 GaBP hot path (BASELINE.json metric: GaBP edge-message updates/s and
achieved HBM GB/s; time to residual 1e-8).

Default workload = BASELINE.json config 2: poisson5(2048, 2048), b ~ U[-1,1] seed 1, synchronous
(flood) GaBP solve with the reference's stop rule (rel. residual 1e-8, 20000-sweep cap).  One
"step" = one solve iteration exactly as GabpEngine::solve runs it (gabp.cpp:187-218): a flood sweep,
the residual check ||b - A x||_inf and the stop test.  value = edge-message updates/s over the
whole job = n_gpus * E * K / (max over ranks of the device time of K steps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload mg]

With --impl reference, rank 0 times the reference's own CPU implementation (oracle/_ref, the
reference sources compiled here; else the restatement) on the same workload and prints the same
line with "impl": "reference"; other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GaBP edge-message updates/sec"
UNIT = "edge-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.1)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


SHARED_GPU = False  # ranks share a GPU (more ranks than visible GPUs): gloo, host-barrier shard steps


def dist_setup():
    """One process per GPU over NCCL.  With more ranks than visible GPUs (a plumbing check of the
    multi-GPU mode on one device) the ranks share the GPUs round-robin, torch.distributed runs on
    gloo, and the sharded solve uses host barriers instead of device-side waits between processes."""
    global SHARED_GPU
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        ndev = torch.cuda.device_count()
        if ndev < world:
            SHARED_GPU = True
            local = local % max(ndev, 1)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world, device="cuda"):
    """Every rank gets the slowest rank's value (device time of its K steps)."""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if SHARED_GPU else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------------
# CPU baseline: the reference's own GabpEngine::solve on the host cores
# ------------------------------------------------------------------------------------------------
def oracle_config2():
    """Config 2's input generated by the oracle itself (poisson5 + mt19937 seed 1, the restated
    proj/tests/oracles.hpp:126-152 generators), so the reference arm loads nothing from the package."""
    from oracle.oracle import Oracle
    o = Oracle.reference()
    kind = "reference"
    if o is None:
        o, kind = Oracle.restatement(), "port"
    gen = Oracle.restatement()
    A = gen.poisson5(2048, 2048)
    b = gen.rng(1).vector(A.n)
    return o, kind, A, b


def cpu_reference_rate(o, kind, A, b, iters, warmup=1, windows=3):
    """Best of `windows` timed windows of `iters` iterations of the reference's own solve loop
    (GabpEngine::solve: flood sweep + residual + stop test, gabp.cpp:187-218) on the full system,
    after `warmup` untimed iterations (BM_SweepFlood method, sweep_bench.cpp:37-48)."""
    from oracle.oracle import Schedule as OSched
    eng = o.engine(A)
    E = eng.num_edges
    tol = 1e-8 * float(np.abs(b).max())
    eng.solve(b, OSched.parallel_flood(), tol=tol, max_iter=max(1, warmup))  # warm-up (page-in, allocator)
    best = float("inf")
    for _ in range(windows):
        t0 = time.perf_counter()
        rep = eng.solve(b, OSched.parallel_flood(), tol=tol, max_iter=iters)
        best = min(best, time.perf_counter() - t0)
        assert rep.iterations == iters
    return {"value": E * iters / best, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{iters} solve iterations (flood sweep + residual, gabp.cpp:187-218) of the full {A.n}-unknown "
                      f"system per window, best of {windows} windows after {max(1, warmup)} warm-up iteration(s); "
                      "1 thread (the reference is single-threaded)",
            "seconds": best, "windows": windows, "cpu": _cpu_name(), "nproc": os.cpu_count()}


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _cpu_baseline_fields(cb):
    return {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "nproc", "cpu")}


def run_reference_arm(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref: the reference sources compiled by
    oracle/Makefile) on the workload's system, input from the oracle's generators; the package is
    not loaded.  --full-solve adds the configuration's own run (config 3: to rel. residual 1e-8;
    config 4: 300 sweeps) as time to solution."""
    if rank != 0:
        return
    if args.config not in (2, 3, 4):
        print(json.dumps({"impl": "reference", "unavailable": f"no CPU reference arm for workload {args.workload}"}),
              flush=True)
        return
    from oracle.oracle import Oracle
    if args.config == 2:
        o, kind, A, b = oracle_config2()
    else:
        o = Oracle.reference()
        kind = "reference"
        if o is None:
            o, kind = Oracle.restatement(), "port"
        A, b = Oracle.restatement().config_problem(args.config)
    iters = max(1, min(args.steps, args.ref_iters if args.config != 4 else 2))
    cb = cpu_reference_rate(o, kind, A, b, iters, min(max(1, args.warmup), 3) if args.config != 4 else 1,
                            windows=3 if args.config != 4 else 1)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": iters, "warmup": max(1, args.warmup), "ms_per_step": cb["seconds"] * 1e3 / iters,
            "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 and args.scaling == "strong" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": DATA[args.config],
            "config": workload_config(A.n, A.nnz, args),
            "cpu_baseline": _cpu_baseline_fields(cb),
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.full_solve and args.config in (3, 4):
        from oracle.oracle import Schedule as OSched
        eng = o.engine(A)
        tol = 0.0 if args.config == 4 else 1e-8 * float(np.abs(b).max())
        cap = 300 if args.config == 4 else 20000
        t0 = time.perf_counter()
        rep = eng.solve(b, OSched.parallel_flood(), tol=tol, max_iter=cap)
        dt = time.perf_counter() - t0
        line["solve"] = {"status": ["Converged", "Diverged", "MaxIter"][rep.status], "iterations": rep.iterations,
                         "seconds": dt, "final_rel_residual": float(rep.residual_history[-1] / np.abs(b).max()),
                         "how": "the reference's GabpEngine::solve, 1 thread, host arrays (no setup)"}
    print(json.dumps(line), flush=True)


WORKLOADS = {
    2: "config2: poisson5 2048x2048, flood GaBP solve loop (sweep + residual + stop test per step)",
    3: "config3: upwind convection-diffusion 1024x1024 (cell Peclet 2, theta 0.3), nonsymmetric flood GaBP solve loop",
    4: "config4: 3D anisotropic lognormal diffusion 256^3 7-point, flood GaBP, fixed 300 sweeps",
    "csr7": "general-sparsity path: the config-4 system (256^3 7-point lognormal diffusion) on the SELL layout "
            "(DIA disabled), flood GaBP solve loop",
    "csr_random": "general-sparsity path: random symmetric diagonally dominant matrix, 4194304 unknowns, 6 random "
                  "neighbours drawn per node (seed 7), SELL layout, flood GaBP solve loop",
}


def random_dd(n, draws, seed):
    """Random symmetric strictly diagonally dominant CSR (canonical: sorted columns, duplicates
    summed): every node draws `draws` random neighbours, off-diagonals U[-1, 0), diagonal =
    1 + sum |off|.  numpy / scipy on the host (input generation only)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(n, dtype=np.int64), draws)
    c = rng.integers(0, n, size=n * draws)
    keep = r != c
    r, c = r[keep], c[keep]
    v = -rng.random(r.size)
    M = sp.coo_matrix((np.concatenate([v, v]), (np.concatenate([r, c]), np.concatenate([c, r]))), shape=(n, n)).tocsr()
    M.sum_duplicates()
    M.sort_indices()
    d = 1.0 + np.asarray(abs(M).sum(axis=1)).ravel()
    M = (M + sp.diags(d)).tocsr()
    M.sort_indices()
    b = rng.uniform(-1.0, 1.0, n)
    return M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data.astype(np.float64), b


def load_workload(g, args):
    """(A, b, layout, nx) of the bench workload."""
    if args.workload == "csr7":
        P = g.config_problem(4)
        return P.A, P.b, g.Layout.Csr, P.nx
    if args.workload == "csr_random":
        n = 1 << 22
        ro, ci, v, b = random_dd(n, 6, 7)
        return g.SparseMatrix(n, ro, ci, v), b, g.Layout.Csr, 0
    P = g.config_problem(args.config)
    return P.A, P.b, g.Layout.Auto, P.nx


DATA = {2: "synthetic (BASELINE.json config 2: b ~ U[-1,1], seed 1)", 3: "synthetic (BASELINE.json config 3)",
        4: "synthetic (BASELINE.json config 4)", "csr7": "synthetic (BASELINE.json config 4 system)",
        "csr_random": "synthetic (random diagonally dominant graph, seed 7)"}


def workload_config(n, nnz, args):
    """The workload description; identical on both arms (the layout the GPU picked is reported
    outside `config`)."""
    E = int(nnz - n)
    return {"workload": WORKLOADS[args.wkey],
            "n": int(n), "nnz": int(nnz), "edges": E, "tol": "1e-8*||b||_inf",
            "max_iter": 300 if args.config == 4 else 20000,
            "l2": "inputs larger than L2: %.0f MB (SURVEY B_sweep) per step vs 126 MB L2; no flush needed" % (
                (40 * E + 24 * n) / 1e6),
            "parallelism": (f"{args.gpus} row-block shards of one system (peer-memory halos over NVLink, CUDA IPC, "
                            "device-side step flags)" if args.gpus > 1 and args.scaling == "strong" else
                            f"{args.gpus} independent replicas (one system per GPU)")}


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def run_gpu(args, world, rank, local):
    import torch

    import paper_1904_04093_b200 as g
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    A_in, b_in, layout, nx_in = load_workload(g, args)
    n = A_in.n
    eng = g.GabpEngine(A_in, layout)
    E = eng.num_edges
    info = eng.info
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)
    b_host = torch.from_numpy(b_in).pin_memory()
    b_dev = b_host.to(dev)
    # the general-sparsity workloads time a fixed number of sweeps (the random system converges
    # in ~60): no stop test can end the timed loop
    tol = 0.0 if args.config == 0 else 1e-8 * float(np.abs(b_in).max())
    max_iter = max(20000, args.warmup + 2 * args.steps + 4)
    opt = g.GabpOptions(tol=tol, max_iter=max_iter)
    sched = g.Schedule.parallel_flood()

    # ---- headline: K solve iterations with b resident in HBM -----------------------------------
    eng.solve_device_begin(b_dev.data_ptr(), sched, opt)
    eng.solve_device_steps(args.warmup)
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        eng.solve_device_steps(args.steps)
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
    barrier(world)
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world)
    value = world * E * args.steps / (ms_max / 1e3)

    # ---- dominant kernel: the fused sweep+residual launch of the same loop, CUDA events around
    # every launch on the engine's stream (the loop continues the solve above, no graphs) --------
    hot_ms = eng.solve_device_steps_timed(args.steps)
    t_sweep = hot_ms / args.steps / 1e3
    status, its, _, _ = eng.solve_device_end()
    assert int(status) == 2 and its >= args.warmup + 2 * args.steps - 2, (status, its)  # never stopped early
    # algorithmic bytes of one fused launch: the sweep's 40E + 24n plus the residual's own reads,
    # x(t-2) (8n; A and b are the sweep's, shared when A is symmetric) -- SURVEY.md 8(d)
    bytes_sweep = float(info["bytes_per_sweep"]) + 8.0 * n + (0.0 if info["symmetric_values"] else 8.0 * E)
    peak, peak_src = peaks()
    achieved = bytes_sweep / t_sweep / 1e9
    # a constant-coefficient stencil (config 2) runs the variant with the coefficients and the
    # diagonal as kernel parameters: it moves 32E + 28n, less than the SURVEY formula counts
    kernel_bytes = 32.0 * E + 28.0 * n if info.get("uniform_coefficients") else bytes_sweep
    if info["layout"] == 1 and not info["symmetric_values"]:
        # nonsymmetric stencils: the out-edge coefficient A_kj is read from row k's own entry (a line
        # node k fetches for its residual), so only one coefficient array comes from DRAM
        kernel_bytes = bytes_sweep - 8.0 * E
    traffic = None
    tp = os.path.join(ROOT, "profiles", "flood_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the public C-ABI with host buffers -----------------------------------
    e2e_sweeps = args.e2e_sweeps
    e2e_opt = g.GabpOptions(tol=tol, max_iter=e2e_sweeps)
    b_np = b_host.numpy()
    x_pin = torch.empty(n, dtype=torch.float64).pin_memory().numpy()  # pinned result buffer
    eng.solve(b_np, sched, g.GabpOptions(tol=tol, max_iter=2), x_out=x_pin)  # warm path
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    reps = []
    for _ in range(args.e2e_calls):
        reps.append(eng.solve(b_np, sched, e2e_opt, x_out=x_pin))
    t_e2e = max_over_ranks(time.perf_counter() - t0, world)
    assert all(r.iterations == e2e_sweeps for r in reps)
    e2e_value = world * E * e2e_sweeps * args.e2e_calls / t_e2e
    h2d = 8 * n  # b per solve call
    d2h = 8 * n + 8 * (e2e_sweeps + 1)  # x + residual history per call

    # ---- the other schedules on the same system: solve iterations per ms, device-resident -------
    schedules = {}
    if args.config == 2 and info["num_slots"] == 4 and not args.no_schedules:
        nxg = nx_in
        for name, sch, k in (("red_black", g.Schedule.red_black_grid(nxg, nxg), 128),
                             ("sequential_pipelined", g.Schedule.sequential(), 2048)):
            eng.solve_device_begin(b_dev.data_ptr(), sch, g.GabpOptions(tol=0.0, max_iter=k + 8))
            eng.solve_device_steps(4)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.solve_device_steps(k)
            e1.record(stream)
            e1.synchronize()
            st_, its_, _, _ = eng.solve_device_end()
            assert its_ == k + 4, (name, st_, its_)
            schedules[name] = {"ms_per_iteration": e0.elapsed_time(e1) / k, "iterations_timed": k,
                               "edge_updates_per_s": E * k / (e0.elapsed_time(e1) / 1e3)}
        schedules["flood"] = {"ms_per_iteration": ms_max / args.steps}

    # ---- the configuration's own run: solve to 1e-8 (cap 20000) or the fixed 300 sweeps ---------
    cap = 300 if args.config == 4 else 20000
    tts = None
    if args.config in (3, 4) or args.full_solve:
        full_opt = g.GabpOptions(tol=0.0 if args.config == 4 else tol, max_iter=cap)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = eng.solve(b_np, sched, full_opt)
        t_full = time.perf_counter() - t0
        tts = {"status": rep.status.name, "iterations": rep.iterations, "seconds": t_full,
               "final_rel_residual": float(rep.residual_history[-1] / np.abs(b_in).max()),
               "how": "one bgabp_solve call with host buffers (H2D b, D2H x + history included)"}

    kernel_name = "k_flood_solve_dia<%d> (K1 flood sweep + K4 residual, fused)" % info["num_slots"]
    if (info["layout"] == 1 and info.get("uniform_coefficients") and n % 64 == 0
            and os.environ.get("BGABP_DIA_TMA", "1") != "0"):
        kernel_name = ("k_flood_solve_dia_tma<%d> (K1 flood sweep + K4 residual, fused; in-slot messages, mask and b "
                       "staged by bulk async copies)" % info["num_slots"])
    formula = (("32*E + 28*n: messages 16 B/edge in + 16 B/edge out; b, x(t-2) read, x(t-1) write, mask per node "
                "(coefficients are kernel parameters)") if info.get("uniform_coefficients") else
               "40*E + 24*n (B_sweep, SURVEY.md 8(d)) + 8*n (x read of the fused residual)"
               + ("" if info["symmetric_values"] else " (the out-edge coefficients come from the neighbours' row "
                  "entries through L1/L2, not DRAM; SURVEY's figure adds 8*E for them)"))
    extra = {}
    if info["layout"] == 2:
        # general sparsity: 44*E + 28*n counts 4 B of index per edge and per node
        kernel_name = "k_flood_solve_sell (SELL layout: flood sweep + residual, fused)"
        kernel_bytes = 44.0 * E + 28.0 * n
        formula = ("44*E + 28*n (SURVEY.md 8(d) general CSR: 40 B/edge of messages and coefficient + 4 B/edge "
                   "index; b, A_jj, x, 4 B index per node)")
        slots = float(info["sell_slots"])
        moved = slots * (8.0 + 16.0 + 8.0 + (0.0 if info["symmetric_values"] else 8.0)) + 16.0 * E + 36.0 * n
        extra = {"sell_slots": int(slots), "sell_slots_per_edge": slots / max(float(E), 1.0),
                 "sell_bytes_per_launch": moved, "sell_frac": moved / t_sweep / 1e9 / peaks()[0],
                 "sell_bytes_formula": "slots * (rev 4 + nbr 4 + message 16 + coefficient 8 [+ row coefficient 8]) "
                                       "+ 16 B/edge message store + 36 B/node; x gathers of the residual excluded "
                                       "(L2-resident)"}
    kernel_achieved = kernel_bytes / t_sweep / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": DATA[args.wkey],
            "config": workload_config(n, A_in.nnz, args),
            "layout": {1: "DIA", 2: "CSR"}[info["layout"]],
            "roofline": {"bound": "hbm", "kernel": kernel_name,
                         # lead: the bytes this kernel variant must move per launch (messages in/out,
                         # the per-node vectors, and the coefficients only where it reads them)
                         "achieved": kernel_achieved, "peak": peak, "unit": "GB/s", "frac": kernel_achieved / peak,
                         "traffic": traffic, "peak_source": peak_src, "bytes_per_launch": kernel_bytes,
                         "bytes_formula": formula,
                         "us_per_launch": t_sweep * 1e6, "frac_of_8TBs": kernel_achieved / 8000.0,
                         "share_of_step": t_sweep * 1e3 / (ms_max / args.steps),
                         # SURVEY.md 8(d)'s conservative formula, which also counts coefficient and
                         # diagonal reads the constant-stencil variant never issues (can exceed 1)
                         "survey_bytes_per_launch": bytes_sweep, "survey_achieved": achieved,
                         "survey_frac": achieved / peak,
                         "traffic_over_bytes": (traffic / kernel_bytes) if traffic else None},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_sweeps,
                    "d2h_bytes_per_step": d2h / e2e_sweeps,
                    "how": f"{args.e2e_calls} x bgabp_solve(pinned host b and x, max_iter={e2e_sweeps}) incl. H2D b, "
                           "D2H x + residual history"},
            "gpu_launches": 2 * args.steps, "clocks": clk.summary()}
    line["roofline"].update(extra)
    if tts is not None:
        line["solve"] = tts
    if args.config == 2 and not args.no_tts and rank == 0:
        # after the headline (its buffers are fresh allocations; the configs' setups below reuse
        # the engine's cached device blocks once it is gone)
        del eng
        torch.cuda.synchronize()
        line["time_to_solution"] = time_to_solution(g, torch, args)
    if schedules:
        line["schedules"] = schedules  # same system, sweep + residual + stop test per iteration
    if args.config != 2:
        line["roofline"]["traffic"] = None
        line["roofline"]["traffic_over_bytes"] = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Csr, Oracle
            if args.config == 2:
                o, kind, A, b = oracle_config2()
            else:
                o = Oracle.reference()
                kind = "reference"
                if o is None:
                    o, kind = Oracle.restatement(), "port"
                A, b = Csr(A_in.n, A_in.row_offsets, A_in.col_indices, A_in.values), b_in
            cb = cpu_reference_rate(o, kind, A, b, args.cpu_iters if args.config != 4 else 2)
            line["cpu_baseline"] = _cpu_baseline_fields(cb)
        except Exception as ex:  # the oracle is test infrastructure; its absence must not hide the GPU number
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "unavailable", "sample": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_sharded(args, world, rank, local):
    """N > 1 GPUs, strong scaling of ONE system: the workload's matrix split into N contiguous
    row blocks (grid rows), one shard per rank/GPU; every iteration the fused step stores the
    halo messages, the ghost x and the stop words straight into the neighbours' memory over
    NVLink (CUDA IPC mappings) and the decision waits on the peers' step flags on the device --
    no collective and no host synchronisation inside the timed loop."""
    import torch

    import paper_1904_04093_b200 as g
    from paper_1904_04093_b200 import shard as sh
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    A_in, b_in, _, nx_in = load_workload(g, args)
    n = A_in.n
    E = int(A_in.nnz - n)
    halo = sh.dia_halo(A_in)
    layouts = sh.ShardLayout.partition(n, halo, world, align=max(nx_in, 1))
    L = layouts[rank]
    shard = sh.GpuShard(sh.local_matrix(A_in, L), L, b_in[L.glo:L.ghi], device=f"cuda:{local}")
    solver = sh.IpcSolve(shard, layouts, host_barrier=SHARED_GPU)
    solver.connect()
    b_inf = float(np.abs(b_in).max())
    tol = 0.0 if args.config == 0 else 1e-8 * b_inf
    opt = g.GabpOptions(tol=tol, max_iter=max(20000, args.warmup + 2 * args.steps + 8))
    stream = shard.stream
    solver.begin(opt, b_inf)
    solver.steps(args.warmup)
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        solver.steps(args.steps)
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    done = solver.done()
    status, its, detail, _, _ = solver.end()
    value = E * args.steps / (ms / 1e3)  # the whole system's edges: total work fixed (strong scaling)
    # end to end: b from pinned host memory into each shard, e2e_sweeps iterations, x and the
    # residual history back, every rank
    b_loc = torch.from_numpy(np.ascontiguousarray(b_in[L.glo:L.ghi])).pin_memory()
    e2e_opt = g.GabpOptions(tol=tol, max_iter=args.e2e_sweeps)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.e2e_calls):
        shard.b.copy_(b_loc, non_blocking=True)
        solver.begin(e2e_opt, b_inf)
        solver.steps(args.e2e_sweeps + 2)
        _st, _its, _d, x_own, _hist = solver.end()
    t_e2e = max_over_ranks(time.perf_counter() - t0, world)
    e2e_value = E * args.e2e_sweeps * args.e2e_calls / t_e2e
    solver.close()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": DATA[args.wkey],
                "config": workload_config(n, A_in.nnz, args),
                "solve_state": {"status_after_timing": int(status), "iterations": its, "stopped_early": bool(done),
                                "detail": detail},
                "e2e": {"value": e2e_value, "unit": UNIT,
                        "h2d_bytes_per_step": 8.0 * n / args.e2e_sweeps,
                        "d2h_bytes_per_step": (8.0 * n + 8.0 * world * (args.e2e_sweeps + 1)) / args.e2e_sweeps,
                        "how": f"{args.e2e_calls} sharded solves of {args.e2e_sweeps} iterations: pinned host b per "
                               "shard in, owned x and history out"},
                "gpu_launches": 3 * args.steps, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def time_to_solution(g, torch, args):
    """The metric's 'time to residual 1e-8' on the configs that reach it, through the public API
    with host buffers, setup (engine / hierarchy build from host CSR) included:
    config 3 (nonsymmetric GaBP, bgabp_solve) and config 5 (V(2,2) red-black GaBP, bgmg_solve).
    Config 2's flood solve needs ~6.7M sweeps and stops at the 20000 cap."""
    out = {}
    P3 = g.config_problem(3)
    tol3 = 1e-8 * float(np.abs(P3.b).max())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e3 = g.GabpEngine(P3.A)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep = e3.solve(P3.b, g.Schedule.parallel_flood(), g.GabpOptions(tol=tol3, max_iter=20000))
    dt = time.perf_counter() - t0
    out["config3_nonsymmetric_gabp"] = {
        "status": rep.status.name, "iterations": rep.iterations, "setup_seconds": setup, "solve_seconds": dt,
        "time_to_solution_seconds": setup + dt,
        "final_rel_residual": float(rep.residual_history[-1] / np.abs(P3.b).max())}
    del e3
    smoothers = (("gabp_red_black", g.MgSmoother.GabpRedBlack), ("gs_red_black", g.MgSmoother.GsRedBlack),
                 ("gabp_flood", g.MgSmoother.GabpFlood))
    # warm-up: one small hierarchy and solve per smoother, so that the one-time costs of a process (the
    # CUDA modules of the multigrid kernels load on first use: 0.1-1 s) are not charged to the first
    # timed configuration
    wl, wb = _mg_levels(g, 7, 1.0)
    for _name, sm in smoothers:
        wh = g.Hierarchy.from_levels([p.A for p in wl], [p.nx for p in wl], sm)
        g.mg_solve(wh, g.CycleSpec(2, 2, sm), wb, g.MgSolveOptions(tol=1e-8 * float(np.abs(wb).max()), max_cycles=5))
        del wh
    torch.cuda.synchronize()
    for sigma in (1.0, 2.0):
        levels, b = _mg_levels(g, args.mg_J, sigma)
        tol = 1e-8 * float(np.abs(b).max())
        for name, sm in smoothers:
            cap = args.mg_cycles if sm != g.MgSmoother.GabpFlood else min(args.mg_cycles, 40)  # flood stalls
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], sm)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            t0 = time.perf_counter()
            rep = g.mg_solve(h, g.CycleSpec(2, 2, sm), b, g.MgSolveOptions(tol=tol, max_cycles=cap))
            dt = time.perf_counter() - t0
            out[f"config5_mg_v22_{name}_sigma{sigma:g}"] = {
                "status": rep.status.name, "cycles": rep.iterations, "levels": h.num_levels(), "setup_seconds": setup,
                "solve_seconds": dt, "time_to_solution_seconds": setup + dt, "max_cycles": cap,
                "final_rel_residual": float(rep.residual_history[-1] / np.abs(b).max()),
                "flop_estimate": rep.flop_estimate,
                "note": ("as specified (sigma 2); coarse K by arithmetic full weighting, the only rediscretisation "
                         "rule with which the reference's V-cycle converges (DESIGN.md 6, tools/config5_coarse_rules.py)"
                         if sigma == 2.0 else "sigma 1: same recipe with milder contrast")}
            del h
        del levels
    return out


# ------------------------------------------------------------------------------------------------
# config 5: multigrid V(2,2) time to 1e-8 (secondary line, --workload mg)
# ------------------------------------------------------------------------------------------------
def _mg_levels(g, J, sigma):
    levels = [g.config5_level(J, k, sigma=sigma) for k in range(J - 4)]  # down to 31 x 31 (J = 5)
    return levels, levels[0].b


def run_mg(args, world, rank, local):
    """Config 5: V(2,2) with red-black GaBP / flood GaBP / red-black GS to rel. residual 1e-8."""
    import torch

    import paper_1904_04093_b200 as g
    torch.cuda.set_device(local)
    J = args.mg_J
    out = {"metric": "multigrid V(2,2) time to rel. residual 1e-8", "unit": "s", "higher_is_better": False,
           "dtype": "f64", "data": "synthetic (BASELINE.json config 5 recipe, seed 4)",
           "config": {"workload": f"config5: 2D -div(K grad u), {(1 << J) - 1}^2 vertices, {J - 4} levels to 31^2, "
                                  "K = exp(N(0, sigma^2)) per unknown, harmonic faces, rediscretised levels "
                                  "(K coarsened by arithmetic full weighting), rows scaled 1/h^2"},
           "gpu": {}, "cpu_reference": {}}
    # warm-up (module loads of the multigrid kernels, see time_to_solution)
    wl, wb = _mg_levels(g, 7, 1.0)
    for sm in (g.MgSmoother.GabpRedBlack, g.MgSmoother.GsRedBlack, g.MgSmoother.GabpFlood):
        wh = g.Hierarchy.from_levels([p.A for p in wl], [p.nx for p in wl], sm)
        g.mg_solve(wh, g.CycleSpec(2, 2, sm), wb, g.MgSolveOptions(tol=1e-8 * float(np.abs(wb).max()), max_cycles=5))
        del wh
    torch.cuda.synchronize()
    for sigma in args.mg_sigmas:
        levels, b = _mg_levels(g, J, sigma)
        bd = torch.tensor(b, device="cuda")
        xd = torch.zeros_like(bd)
        tol = 1e-8 * float(np.abs(b).max())
        for name, sm in (("gabp_red_black", g.MgSmoother.GabpRedBlack), ("gs_red_black", g.MgSmoother.GsRedBlack),
                         ("gabp_flood", g.MgSmoother.GabpFlood)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = g.Hierarchy.from_levels([p.A for p in levels], [p.nx for p in levels], sm)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            spec = g.CycleSpec(2, 2, sm)
            cap = args.mg_cycles if sm != g.MgSmoother.GabpFlood else min(args.mg_cycles, 40)
            # cold: the first solve on a fresh hierarchy (records the smoother's cold-start
            # precisions per level, captures the V-cycle graph); warm: the same solve again
            t0 = time.perf_counter()
            g.mg_solve_device(h, spec, bd.data_ptr(), xd.data_ptr(), g.MgSolveOptions(tol=tol, max_cycles=cap))
            torch.cuda.synchronize()
            cold = time.perf_counter() - t0
            t0 = time.perf_counter()
            rep = g.mg_solve_device(h, spec, bd.data_ptr(), xd.data_ptr(), g.MgSolveOptions(tol=tol, max_cycles=cap))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            out["gpu"][f"sigma{sigma}/{name}"] = {
                "status": rep.status.name, "cycles": rep.iterations, "seconds": dt,
                "ms_per_cycle": 1e3 * dt / max(rep.iterations, 1), "setup_seconds": setup,
                "cold_solve_seconds": cold, "time_to_solution_seconds": setup + cold, "levels": h.num_levels(),
                "final_rel_residual": float(rep.residual_history[-1] / np.abs(b).max()), "detail": rep.detail}
            del h
    # the reference's V-cycle on the host (Eigen-free restatement of multigrid.cpp over the
    # reference's own compiled GabpEngine), on a bounded sample: the same recipe at J = mg_cpu_J
    if rank == 0 and not args.no_cpu_baseline:
        from oracle.oracle import Oracle
        o = Oracle.reference() or Oracle.restatement()
        gen = Oracle.restatement()  # the oracle's own config-5 generator (pinned to the product's)
        for sigma in args.mg_sigmas:
            cpu_levels = [gen.config5_level(args.mg_cpu_J, k, sigma=sigma) for k in range(args.mg_cpu_J - 4)]
            b = cpu_levels[0][1]
            tol = 1e-8 * float(np.abs(b).max())
            for name, sm in (("gabp_red_black", 1), ("gs_red_black", 7)):
                if name not in args.mg_cpu_smoothers:
                    continue
                t0 = time.perf_counter()
                oh = o.hierarchy([A for A, _ in cpu_levels], [int(round(np.sqrt(A.n))) for A, _ in cpu_levels], sm)
                setup = time.perf_counter() - t0
                t0 = time.perf_counter()
                rep = oh.solve(2, 2, b, tol=tol, max_cycles=args.mg_cycles)
                dt = time.perf_counter() - t0
                out["cpu_reference"][f"J{args.mg_cpu_J}/sigma{sigma}/{name}"] = {
                    "status": ["Converged", "Diverged", "MaxIter"][rep.status], "cycles": rep.iterations,
                    "seconds": dt, "ms_per_cycle": 1e3 * dt / max(rep.iterations, 1), "setup_seconds": setup,
                    "time_to_solution_seconds": setup + dt, "cores": 1, "kind": "reference" if o is Oracle.reference() else "port"}
            if args.mg_cpu_J == J:
                continue
            # the GPU at the CPU's size too, for a like-for-like time-to-solution
            lv2, b2 = _mg_levels(g, args.mg_cpu_J, sigma)
            bd2 = torch.tensor(b2, device="cuda")
            xd2 = torch.zeros_like(bd2)
            for name, sm in (("gabp_red_black", g.MgSmoother.GabpRedBlack), ("gs_red_black", g.MgSmoother.GsRedBlack)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                h = g.Hierarchy.from_levels([p.A for p in lv2], [p.nx for p in lv2], sm)
                torch.cuda.synchronize()
                setup = time.perf_counter() - t0
                tol2 = 1e-8 * float(np.abs(b2).max())
                t0 = time.perf_counter()
                rep = g.mg_solve_device(h, g.CycleSpec(2, 2, sm), bd2.data_ptr(), xd2.data_ptr(),
                                        g.MgSolveOptions(tol=tol2, max_cycles=args.mg_cycles))
                torch.cuda.synchronize()
                cold = time.perf_counter() - t0
                out["gpu"][f"J{args.mg_cpu_J}/sigma{sigma}/{name}"] = {
                    "status": rep.status.name, "cycles": rep.iterations, "setup_seconds": setup,
                    "cold_solve_seconds": cold, "time_to_solution_seconds": setup + cold}
                del h
    if rank == 0:
        print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2", choices=["config2", "config3", "config4", "csr7", "csr_random",
                                                              "mg"])
    ap.add_argument("--full-solve", action="store_true", help="config 2: also run the capped 20000-sweep solve")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: one system sharded over the GPUs (strong) or one replica per GPU (weak)")
    ap.add_argument("--e2e-sweeps", type=int, default=500)
    ap.add_argument("--e2e-calls", type=int, default=3)
    ap.add_argument("--ref-iters", type=int, default=20, help="reference arm: iterations per timed window")
    ap.add_argument("--cpu-iters", type=int, default=10, help="cpu_baseline: iterations per timed window")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-schedules", action="store_true", help="skip the red-black / sequential timings")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-1e-8 runs (configs 3 and 5)")
    ap.add_argument("--mg-J", type=int, default=12)
    ap.add_argument("--mg-cycles", type=int, default=1000)
    ap.add_argument("--mg-cpu-J", type=int, default=9)
    ap.add_argument("--mg-cpu-smoothers", nargs="+", default=["gabp_red_black", "gs_red_black"])
    ap.add_argument("--mg-sigmas", type=float, nargs="+", default=[2.0, 1.0])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.config = int(args.workload[-1]) if args.workload.startswith("config") else (
        0 if args.workload.startswith("csr") else 2)
    args.wkey = args.config if args.config else args.workload
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, world, rank)
        return
    world, rank, local = dist_setup()
    if args.workload == "mg":
        run_mg(args, world, rank, local)
    elif world > 1 and args.scaling == "strong":
        run_sharded(args, world, rank, local)
    else:
        run_gpu(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
