#!/usr/bin/env python
"""Benchmark of the B200 T^2S^2 hot path.

Default workload (--workload march): implicit time steps/s of the d=6 + time
march (BASELINE.json configs[2]: n=33 nodes per dim, eps=1e-3, translating
Gaussian, backward Euler dt=1e-3, TT rounding tolerance 1e-12).  A "step" is
one implicit step: rhs assembly and rounding, the alternating TT solve with
its local direct/Krylov solves, and re-truncation.  Steps are a sequential
chain (step k starts from state k-1), so K timed steps are steps W+1..W+K of
one march.  Multi-GPU: the march does not shard, so each rank runs an
independent replica ("replicas only", weak scaling); value = all ranks'
steps / max-over-ranks time.

--workload sweep: BASELINE.json configs[4], the batched parameter sweep of
independent d=6 steady solves (n=33, seeded eps and b).  A "step" is one
solve capped at --sweep-sweeps ALS sweeps; rank r of N takes seeds r, r+N,
... of the 64 (sweep.shard), cycling, with no data-path collective;
solves/s, weak scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload march|sweep]

Defaults: 3 warm-up steps, then steps 4..23 of the config-2 march timed
(--steps 97: the whole 100-step march); 16 solves after 1 warm-up solve for
the sweep.

--impl b200 (default): the CUDA engine through its C ABI.  One JSON line with
value (inputs resident in HBM), e2e (public API with pinned host buffers:
per-step H2D of the step's inputs, D2H of its result), the roofline of the
dominant kernel family, launch counts, clocks and the reference CPU baseline.

--impl reference: the reference itself — ttss from baseline/_ref, its own
tt_apply / tt_add / tt_round / tt_solver.solve in the loop of
time_integration._march (time_integration.py:164-177) with the per-step
forcing — on this host's cores, rank 0 only, on the same steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MARCH = dict(metric="implicit_time_steps_per_s", unit="steps/s", index=2)
SWEEP = dict(metric="steady_solves_per_s", unit="solves/s", index=4)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps; default 20 (march: steps 4..23; --steps 97 times the rest "
                         "of BASELINE config 2's 100-step march), 16 solves (sweep)")
    ap.add_argument("--warmup", type=int, default=None, help="default 3 (march), 1 (sweep)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="march", choices=["march", "sweep"])
    ap.add_argument("--sweep-sweeps", type=int, default=6,
                    help="ALS sweeps per config-4 solve (fixed budget)")
    ap.add_argument("--sweep-partitions", type=int, default=4,
                    help="run the timed solves on P disjoint SM partitions (green contexts)")
    ap.add_argument("--residual-tol", type=float, default=None,
                    help="march: inner residual target (default: the reference's MarchConfig "
                         "1e-10); 1e-12 reads BASELINE's 'TT tolerance' as the residual target")
    ap.add_argument("--cpu-sample-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup is None:
        args.warmup = 3 if args.workload == "march" else 1
    if args.steps is None:
        args.steps = 20 if args.workload == "march" else 16
    return args


def march_config(recipe, extra=None):
    cfg = {
        "workload": "BASELINE configs[2]: d=6+time implicit march",
        "dims": recipe.dims, "nodes_per_dim": recipe.degree + 1, "eps": recipe.eps,
        "dt": recipe.dt, "scheme": "backward_euler",
        "tt_rounding_tol": recipe.solver.get("rounding_tol"), "step_tol": recipe.step_tol,
        "residual_tol": recipe.solver.get("residual_tol"),
        "tolerances": "rounding_tol 1e-12 (BASELINE 'TT tolerance'); residual_tol and the step "
                      "re-truncation are the reference's MarchConfig defaults "
                      "(time_integration.py:54-60), identical in both arms",
        "solution": "translating Gaussian exp(-|x-b t|^2/0.05), b seeded unit vector",
    }
    if extra:
        cfg.update(extra)
    return cfg


def sweep_config(args, world, extra=None):
    cfg = {
        "workload": "BASELINE configs[4]: batched sweep of d=6 steady solves",
        "dims": 6, "nodes_per_dim": 33, "seeds": 64, "sweeps_per_solve": args.sweep_sweeps,
        "eps": "log-uniform [1e-12, 1e-1] per seed", "solution": "separable boundary layer",
        "tt_rounding_tol": 1e-12, "residual_tol": 1e-10,
        "sharding": f"rank r of {world} takes seeds r, r+{world}, ... (cycling)",
    }
    if extra:
        cfg.update(extra)
    return cfg


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


# -- the reference's own CPU path (ttss) -------------------------------------------


def ttss_step(rtt, rsol, left, right, state, bc, src, step_tol, cfg):
    """One implicit step exactly as time_integration._march takes it
    (time_integration.py:164-177), in the reference's own functions."""
    rhs = rtt.tt_add(rtt.tt_add(rtt.tt_apply(right, state), bc), src)
    rhs = rtt.tt_round(rhs, 0.01 * step_tol)
    new, rep = rsol.solve(left, rhs, x0=state, cfg=cfg)
    return rtt.tt_round(new, step_tol), rep


def ttss_march(recipe, problem, state, first, count):
    """Steps first..first+count-1 with ttss; forcing sampled outside the
    timed region (it is the step's input).  Returns (seconds, state)."""
    from paper_2506_04732_b200.reference import module

    rtt, rsol = module("tensor_train"), module("tt_solver")
    left, right, _, forcing, _, _ = problem
    cfg = rsol.SolverConfig(**recipe.solver)
    forc = {k: forcing(k) for k in range(first, first + count)}
    t0 = time.perf_counter()
    for k in range(first, first + count):
        state, _ = ttss_step(rtt, rsol, left, right, state, *forc[k], recipe.step_tol, cfg)
    return time.perf_counter() - t0, state


def march_recipe(args):
    from paper_2506_04732_b200 import workloads as wl

    recipe = wl.config(MARCH["index"])
    if args.residual_tol is not None:
        recipe.solver = dict(recipe.solver, residual_tol=args.residual_tol)
    return recipe


def sweep_seeds(rank, world, count):
    from paper_2506_04732_b200.sweep import shard

    mine = shard(64, rank, world)
    return [mine[i % len(mine)] for i in range(count)]


def ttss_sweep(args, seeds):
    """Config-4 solves with ttss.tt_solver.solve at the fixed sweep budget."""
    from paper_2506_04732_b200 import workloads as wl
    from paper_2506_04732_b200.reference import module

    rsol = module("tt_solver")
    recipes = wl.sweep_recipes()
    probs = {i: wl.steady_problem(recipes[i]) for i in set(seeds)}
    total = 0.0
    for i in seeds:
        a, b, _, _ = probs[i]
        cfg = rsol.SolverConfig(**recipes[i].solver, max_sweeps=args.sweep_sweeps)
        t0 = time.perf_counter()
        rsol.solve(a, b, cfg=cfg)
        total += time.perf_counter() - t0
    return total


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2506_04732_b200 import workloads as wl

    W, K = args.warmup, args.steps
    cores = blas_threads()
    if args.workload == "march":
        w = MARCH
        recipe = march_recipe(args)
        problem = wl.march_problem(recipe)
        _, state = ttss_march(recipe, problem, problem[2], 1, W)
        elapsed, _ = ttss_march(recipe, problem, state, W + 1, K)
        config = march_config(recipe, {"parallelism": "cpu", "timed_steps": f"{W + 1}..{W + K}"})
        sample = (f"steps {W + 1}..{W + K} of the config-2 march after {W} untimed steps: "
                  "ttss (baseline/_ref) tt_apply/tt_add/tt_round/tt_solver.solve, numpy/OpenBLAS")
    else:
        w = SWEEP
        allseeds = sweep_seeds(0, 1, W + K)  # the GPU arm's seeds: W warm-up, then K timed
        seeds = allseeds[W:]
        ttss_sweep(args, allseeds[:min(W, 1)])  # untimed warm-up solve
        elapsed = ttss_sweep(args, seeds)
        config = sweep_config(args, 1, {"parallelism": "cpu", "timed_seeds": seeds})
        sample = (f"{K} config-4 solves (seeds {seeds}), {args.sweep_sweeps} sweeps each: "
                  "ttss.tt_solver.solve (baseline/_ref), numpy/OpenBLAS")
    value = K / elapsed
    line = {
        "impl": "reference", "metric": w["metric"], "value": value, "unit": w["unit"],
        "n_gpus": args.gpus, "steps": K, "warmup": W, "ms_per_step": 1e3 * elapsed / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded manufactured solutions)", "config": config,
        "cpu_baseline": {"value": value, "unit": w["unit"], "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": w["unit"], "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -- GPU leg --------------------------------------------------------------------------


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.gpu = gpu

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None, "reasons": sorted(reasons),
                "samples": len(sms)}


def fp64_gemm_peak_tflops(torch):
    """cuBLAS DGEMM throughput on this device (FP64 tensor cores): the
    roofline denominator for fp64 kernels (MEASURED_PEAKS.json has none)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = max(best, 2.0 * n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    del a, b
    return best


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def roofline(torch, prof):
    """Roofline of the dominant kernel family from the per-family CUDA-event
    times of a profiled replay (algorithmic flops/bytes counted at each
    launch site, csrc LaunchScope)."""
    name, st = max(prof.items(), key=lambda kv: kv[1]["device_ms"])
    peak64 = fp64_gemm_peak_tflops(torch)
    peaks = measured_peaks()
    flop_bound = st["flops"] > 0 and (st["flops"] / max(st["bytes"], 1.0)) > 2.0
    per_launch_ms = st["device_ms"] / max(st["launches"], 1)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(name)
    except Exception:
        pass
    common = {"traffic": traffic, "kernel": name, "avg_launch_ms": per_launch_ms,
              "launches": st["launches"]}
    if flop_bound:
        achieved = st["flops"] / (st["device_ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak64, "unit": "TFLOP/s",
                "frac": achieved / peak64,
                "peak_source": "cuBLAS DGEMM 8192^3 fp64 measured in this run "
                               "(MEASURED_PEAKS.json has no fp64 figure)",
                "algorithmic_per_launch": st["flops"] / max(st["launches"], 1),
                "algorithmic_unit": "flop (dense solve: 2/3 N^3 + 2 N^2)"
                if name.startswith("gj") or name.startswith("lu") else "flop"}
    else:
        hbm = peaks.get("hbm_gbs", 6650.0)
        achieved = st["bytes"] / (st["device_ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
                else "fallback 6650 GB/s (B200_PROFILING.md)",
                "algorithmic_per_launch": st["bytes"] / max(st["launches"], 1)}
    roof.update(common)
    tot = sum(v["device_ms"] for v in prof.values())
    kernels = {k: {"launches": v["launches"], "device_ms": round(v["device_ms"], 3),
                   "share": round(v["device_ms"] / tot, 4) if tot else 0.0,
                   "gflop": round(v["flops"] / 1e9, 4)}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["device_ms"])}
    return roof, kernels


class Dist:
    def __init__(self, torch):
        self.torch = torch
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        torch.cuda.set_device(self.local)
        os.environ["T2S2_DEVICE"] = str(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            dist.init_process_group("nccl")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x):
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


def pin(torch, cores):
    flat = np.concatenate([np.ascontiguousarray(c).ravel() for c in cores])
    t = torch.empty(flat.size, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = flat
    return t


def run_b200_march(args, torch, dd):
    from paper_2506_04732_b200 import _native, workloads as wl
    from paper_2506_04732_b200.march import march_device
    from paper_2506_04732_b200.solver import SolverConfig
    from paper_2506_04732_b200.tt import from_device, to_device

    recipe = march_recipe(args)
    W, K = args.warmup, args.steps
    problem = wl.march_problem(recipe)
    left, right, state0, forcing, exact, _ = problem
    forc = [forcing(k) for k in range(1, W + K + 1)]
    cfg = SolverConfig(**recipe.solver)
    ctx = _native.context()
    eng_stream = torch.cuda.ExternalStream(_native.lib().t2s2_stream(ctx))
    hl, hr = to_device(left), to_device(right)
    hbc = [to_device(b) for b, _ in forc]
    hsrc = [to_device(s) for _, s in forc]
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def one_step(state, k, bc=None, src=None):
        stored, rows = march_device(hl, hr, state, 1, [bc or hbc[k - 1]], [src or hsrc[k - 1]],
                                    recipe.step_tol, cfg, store_stride=1)
        return stored[1], rows[0]

    def l2_flush():
        _native.synchronize()
        flush.fill_(1.0)
        torch.cuda.synchronize()

    # warm-up steps 1..W
    state = to_device(state0)
    for k in range(1, W + 1):
        nxt, _ = one_step(state, k)
        state.free()
        state = nxt
    warm_state = state
    _native.synchronize()

    # timed steps W+1..W+K, L2 flushed between steps (flush not timed)
    dd.barrier()
    torch.cuda.synchronize()
    _native.stats_reset(profile_events=False)
    rows, total_ms, state = [], 0.0, warm_state
    with Clocks(dd.local) as clk:
        t_wall = time.perf_counter()
        for k in range(W + 1, W + K + 1):
            l2_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng_stream)
            nxt, row = one_step(state, k)
            e1.record(eng_stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            rows.append(row)
            if state is not warm_state:
                state.free()
            state = nxt
        t_wall = time.perf_counter() - t_wall
    torch.cuda.synchronize()
    gpu_launches = sum(v["launches"] for k, v in _native.stats_read().items() if k != "copy")  # kernels; "copy" = copy-engine nodes
    elapsed = dd.max(total_ms / 1e3)
    dd.barrier()
    value = dd.world * K / elapsed

    # accuracy of the timed march against the analytic solution
    fin = from_device(state)
    ex = exact((W + K) * recipe.dt)
    from oracle import tt_ops as ot  # checker only: error of the result, not timed

    exact_err = float(ot.tt_norm(ot.tt_add(fin.cores, ot.tt_scale(ex.cores, -1.0)))
                      / ot.tt_norm(ex.cores))
    state.free()

    # profiled replay of the same K steps (identical inputs, same warm state):
    # per-family CUDA-event time on the engine stream -> roofline
    _native.stats_reset(profile_events=True)
    state = warm_state
    for k in range(W + 1, W + K + 1):
        nxt, _ = one_step(state, k)
        if state is not warm_state:
            state.free()
        state = nxt
    state.free()
    prof = _native.stats_read()
    _native.stats_reset(profile_events=False)

    # e2e: public API with pinned host buffers; per step H2D of the step's
    # forcing trains and D2H of the new state, the same steps replayed from
    # the same warm state, L2 flushed between steps like the device-timed run
    h2d = d2h = 0
    e2e_ms = 0.0
    host_state = warm_state
    pinned = {k: (pin(torch, forc[k - 1][0].cores), pin(torch, forc[k - 1][1].cores))
              for k in range(W + 1, W + K + 1)}
    out_buf = torch.empty(4 * 1024 * 1024, dtype=torch.float64, pin_memory=True)
    for k in range(W + 1, W + K + 1):
        pb, ps = pinned[k]
        b, s = forc[k - 1]
        l2_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng_stream)
        db = _native.DeviceTrain.upload_flat(pb.data_ptr(), b.mode_sizes, None, b.ranks)
        ds = _native.DeviceTrain.upload_flat(ps.data_ptr(), s.mode_sizes, None, s.ranks)
        nxt, _ = one_step(host_state, k, db, ds)
        _, _, _, total = nxt.shape()
        nxt.download_into(out_buf.data_ptr(), out_buf.numel())
        e1.record(eng_stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        h2d += 8 * (pb.numel() + ps.numel())
        d2h += 8 * total
        db.free()
        ds.free()
        if host_state is not warm_state:
            host_state.free()
        host_state = nxt
    host_state.free()
    warm_cores = from_device(warm_state)
    warm_state.free()
    e2e_elapsed = dd.max(e2e_ms / 1e3)
    if dd.rank != 0:
        return None

    roof, kernels = roofline(torch, prof)
    cpu = None
    if not args.no_cpu_baseline and args.cpu_sample_steps > 0:
        # the reference's own step loop on this host, from the device's step-W state
        S = args.cpu_sample_steps
        el, _ = ttss_march(recipe, problem, warm_cores, W + 1, S)
        cpu = {"value": S / el, "unit": MARCH["unit"], "cores": blas_threads(),
               "kind": "reference",
               "sample": f"steps {W + 1}..{W + S} of the same config-2 march from the device's "
                         f"step-{W} state: ttss (baseline/_ref) on this host, numpy/OpenBLAS"}
    return {
        "metric": MARCH["metric"], "value": value, "unit": MARCH["unit"], "n_gpus": dd.world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * elapsed / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (manufactured translating Gaussian, seeded)",
        "config": march_config(recipe, {
            "parallelism": f"replicas x{dd.world}" if dd.world > 1 else "single GPU",
            "l2": "256 MiB write between timed steps (not timed)",
            "timed_steps": f"{W + 1}..{W + K}",
            "max_rank_seen": max(r[1] for r in rows),
            "sweeps_per_step": [r[4] for r in rows],
            "exact_rel_error_final": exact_err,
        }),
        "roofline": roof, "kernels": kernels, "gpu_launches": gpu_launches,
        "e2e": {"value": dd.world * K / e2e_elapsed, "unit": MARCH["unit"],
                "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K},
        "cpu_baseline": cpu, "clocks": clk.summary(), "wall_s_timed": t_wall,
    }


def partitioned_sweep(args, seeds, probs, recipes, e2e=False):
    """The same solves on P disjoint SM partitions of this GPU (green
    contexts), one host thread each pulling from a shared queue; returns the
    batch makespan in seconds from the device's global timer (first start to
    last end over all partitions), the partition sizes, and the bytes moved
    per solve.  e2e: each solve's operator, right-hand side and initial guess
    are uploaded from host memory and its solution downloaded inside the
    timed region (the public API path)."""
    import threading

    from paper_2506_04732_b200 import _native
    from paper_2506_04732_b200.solver import SolverConfig, _default_initial_guess, solve_device
    from paper_2506_04732_b200.tt import to_device

    P = args.sweep_partitions
    sms = _native.sm_partitions(P)
    queue = list(seeds)
    lock = threading.Lock()
    ready = threading.Barrier(P + 1)
    go = threading.Event()
    starts, ends, errors = [], [], []
    moved = [0, 0]

    def cfg_of(i):
        return SolverConfig(**recipes[i].solver, max_sweeps=args.sweep_sweeps)

    def worker(t):
        mine = {}
        try:
            _native.use_partition(t)
            for i in set(seeds):
                a, b = probs[i][0], probs[i][1]
                mine[i] = (to_device(a), to_device(b),
                           to_device(_default_initial_guess(b, None, np.random.default_rng(0))))
            i0 = seeds[0]  # warm-up: module load and shared-memory limits in this context
            h, _ = solve_device(*mine[i0], SolverConfig(**recipes[i0].solver, max_sweeps=1))
            h.free()
            _native.synchronize()
        except Exception as exc:
            errors.append(exc)
        ready.wait()
        go.wait()
        try:
            if not errors:
                t0 = _native.device_clock_ns()
                while True:
                    with lock:
                        if not queue:
                            break
                        i = queue.pop(0)
                    if e2e:
                        a, b = probs[i][0], probs[i][1]
                        x0 = _default_initial_guess(b, None, np.random.default_rng(0))
                        ups = [_native.DeviceTrain.upload(t.cores, t.cores[0].ndim == 4)
                               for t in (a, b, x0)]
                        h, _ = solve_device(*ups, cfg_of(i))
                        cores, _ = h.download()
                        for u in ups:
                            u.free()
                        with lock:
                            moved[0] += 8 * sum(c.size for t in (a, b, x0) for c in t.cores)
                            moved[1] += 8 * sum(c.size for c in cores)
                    else:
                        h, _ = solve_device(*mine[i], cfg_of(i))
                    h.free()
                t1 = _native.device_clock_ns()
                with lock:
                    starts.append(t0)
                    ends.append(t1)
        except Exception as exc:
            errors.append(exc)
        for hs in mine.values():
            for h in hs:
                h.free()

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(P)]
    for th in threads:
        th.start()
    ready.wait()
    go.set()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    n = max(len(seeds), 1)
    return (max(ends) - min(starts)) * 1e-9, sms, (moved[0] // n, moved[1] // n)


def run_b200_sweep(args, torch, dd):
    from paper_2506_04732_b200 import _native, workloads as wl
    from paper_2506_04732_b200.solver import SolverConfig, solve_device
    from paper_2506_04732_b200.tt import to_device

    W, K = args.warmup, args.steps
    seeds = sweep_seeds(dd.rank, dd.world, W + K)
    recipes = wl.sweep_recipes()
    probs = {i: wl.steady_problem(recipes[i]) for i in set(seeds)}
    ctx = _native.context()
    eng_stream = torch.cuda.ExternalStream(_native.lib().t2s2_stream(ctx))
    dev = {i: (to_device(p[0]), to_device(p[1])) for i, p in probs.items()}
    x0 = {}
    from paper_2506_04732_b200.solver import _default_initial_guess

    for i, p in probs.items():
        x0[i] = to_device(_default_initial_guess(p[1], None, np.random.default_rng(0)))

    def cfg_of(i):
        return SolverConfig(**recipes[i].solver, max_sweeps=args.sweep_sweeps)

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def l2_flush():
        _native.synchronize()
        flush.fill_(1.0)
        torch.cuda.synchronize()

    for i in seeds[:W]:
        h, _ = solve_device(dev[i][0], dev[i][1], x0[i], cfg_of(i))
        h.free()
    _native.synchronize()
    dd.barrier()
    torch.cuda.synchronize()
    _native.stats_reset(profile_events=False)
    total_ms, sweeps, reports = 0.0, 0, []
    with Clocks(dd.local) as clk:
        for i in seeds[W:]:
            l2_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng_stream)
            h, rep = solve_device(dev[i][0], dev[i][1], x0[i], cfg_of(i))
            e1.record(eng_stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            sweeps += len(rep.residual_history)
            reports.append((i, rep.residual_history[-1], rep.rank_history[-1]))
            h.free()
    gpu_launches = sum(v["launches"] for k, v in _native.stats_read().items() if k != "copy")  # kernels; "copy" = copy-engine nodes
    elapsed = dd.max(total_ms / 1e3)
    value = dd.world * K / elapsed
    serial = None
    if args.sweep_partitions > 1:
        # headline = the partitioned run; the one-stream run above is kept
        l2_flush()
        with Clocks(dd.local) as clk:  # the headline's timed region
            p_s, sms, _ = partitioned_sweep(args, seeds[W:], probs, recipes)
        p_s = dd.max(p_s)
        serial = {"value": value, "ms_per_step": 1e3 * elapsed / K,
                  "how": "one engine context on all 148 SMs, solves one after another, "
                         "CUDA events per solve"}
        elapsed = p_s
        value = dd.world * K / elapsed
    _native.stats_reset(profile_events=True)
    for i in seeds[W:]:
        h, _ = solve_device(dev[i][0], dev[i][1], x0[i], cfg_of(i))
        h.free()
    prof = _native.stats_read()
    _native.stats_reset(profile_events=False)

    # e2e: operator, rhs and initial guess uploaded from pinned host memory and
    # the solution downloaded, every solve
    e2e_ms, h2d, d2h = 0.0, 0, 0
    out_buf = torch.empty(16 * 1024 * 1024, dtype=torch.float64, pin_memory=True)
    for i in seeds[W:]:
        a, b = probs[i][0], probs[i][1]
        xh = _default_initial_guess(b, None, np.random.default_rng(0))
        pa, pb, px = pin(torch, a.cores), pin(torch, b.cores), pin(torch, xh.cores)
        l2_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng_stream)
        da = _native.DeviceTrain.upload_flat(pa.data_ptr(), a.row_sizes, a.col_sizes, a.ranks)
        db = _native.DeviceTrain.upload_flat(pb.data_ptr(), b.mode_sizes, None, b.ranks)
        dx = _native.DeviceTrain.upload_flat(px.data_ptr(), xh.mode_sizes, None, xh.ranks)
        h, _ = solve_device(da, db, dx, cfg_of(i))
        total = h.shape()[3]
        h.download_into(out_buf.data_ptr(), out_buf.numel())
        e1.record(eng_stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        h2d += 8 * (pa.numel() + pb.numel() + px.numel())
        d2h += 8 * total
        for t in (da, db, dx, h):
            t.free()
    e2e_elapsed = dd.max(e2e_ms / 1e3)
    e2e_serial = None
    if args.sweep_partitions > 1:
        # the headline e2e uses the same SM partitions as the headline value
        e2e_serial = {"value": dd.world * K / e2e_elapsed, "unit": SWEEP["unit"],
                      "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K}
        l2_flush()
        p_s, _, (h2d, d2h) = partitioned_sweep(args, seeds[W:], probs, recipes, e2e=True)
        e2e_elapsed = dd.max(p_s)
        h2d, d2h = h2d * K, d2h * K
    if dd.rank != 0:
        return None
    roof, kernels = roofline(torch, prof)
    cpu = None
    if not args.no_cpu_baseline and args.cpu_sample_steps > 0:
        S = min(args.cpu_sample_steps, 2)
        sample = seeds[W:W + S]
        el = ttss_sweep(args, sample)
        cpu = {"value": S / el, "unit": SWEEP["unit"], "cores": blas_threads(),
               "kind": "reference",
               "sample": f"{S} of the timed solves (seeds {sample}), {args.sweep_sweeps} sweeps "
                         "each: ttss.tt_solver.solve (baseline/_ref) on this host"}
    return {
        "metric": SWEEP["metric"], "value": value, "unit": SWEEP["unit"], "n_gpus": dd.world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * elapsed / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded boundary-layer manufactured solutions)",
        "config": sweep_config(args, dd.world, {
            "parallelism": f"sharded x{dd.world}" if dd.world > 1 else "single GPU",
            "l2": "256 MiB write between timed solves (not timed)",
            "rank0_timed": [{"seed": i, "residual": r, "max_rank": m} for i, r, m in reports],
            "sweeps_timed_rank0": sweeps,
            "sm_partitions": (f"{args.sweep_partitions} green contexts of "
                              f"{sms} SMs, one host thread each, shared queue; makespan from "
                              "the device global timer" if args.sweep_partitions > 1 else None),
        }),
        "serial": serial,
        "roofline": roof, "kernels": kernels, "gpu_launches": gpu_launches,
        "e2e": {"value": dd.world * K / e2e_elapsed, "unit": SWEEP["unit"],
                "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K},
        "cpu_baseline": cpu, "clocks": clk.summary(), "e2e_serial": e2e_serial,
    }


def run_b200(args):
    import torch

    dd = Dist(torch)
    line = (run_b200_march if args.workload == "march" else run_b200_sweep)(args, torch, dd)
    if line is not None:
        print(json.dumps(line), flush=True)
    dd.close()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
