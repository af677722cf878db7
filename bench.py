#!/usr/bin/env python
"""Benchmark of the B200 T^2S^2 hot path: implicit time steps/s of the
d=6 + time march (BASELINE.json configs[2]: n=33 nodes per dim, eps=1e-3,
translating Gaussian, backward Euler dt=1e-3, TT tolerance 1e-12).

A "step" is one implicit step: rhs assembly and rounding, the alternating
TT solve with its local direct/Krylov solves, and re-truncation.  Steps are
a sequential chain (step k starts from state k-1), so K timed steps are
steps W+1..W+K of one march.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl b200 (default): the CUDA engine through its C ABI.  Prints one JSON
line with value (inputs resident in HBM), e2e (public API with pinned host
buffers, per-step H2D of the forcing and D2H of the new state), the roofline
of the dominant kernel family, launch counts, clocks and the CPU oracle
baseline.  Multi-GPU: the march does not shard, so each rank runs an
independent replica ("replicas only", weak scaling); value = all ranks'
steps / max-over-ranks time.

--impl reference: the reference's CPU algorithm (the oracle port in
oracle/, pinned to the reference's outputs) on this host's cores, rank 0
only.
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

METRIC = "implicit_time_steps_per_s"
UNIT = "steps/s"
CONFIG_INDEX = 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload_config(recipe, extra=None):
    cfg = {
        "workload": "BASELINE configs[2]: d=6+time implicit march",
        "dims": recipe.dims, "nodes_per_dim": recipe.degree + 1, "eps": recipe.eps,
        "dt": recipe.dt, "scheme": "backward_euler", "tt_rounding_tol": recipe.solver.get("rounding_tol"),
        "step_tol": recipe.step_tol,
        "residual_tol": recipe.solver.get("residual_tol"),
        "solution": "translating Gaussian exp(-|x-b t|^2/0.05), b seeded unit vector",
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


# -- CPU legs (oracle = the reference's algorithm, pinned to its outputs) ----------


def cpu_backend():
    """Setup numerics on the CPU oracle (no GPU needed): a context manager."""
    from oracle import tt_ops as ot
    from paper_2506_04732_b200 import assembly, tt

    def rnd(v, tol, max_rank=None):
        if isinstance(v, tt.TTOperator):
            rows, cols = v.row_sizes, v.col_sizes
            return tt.TTOperator(ot.as_operator(ot.tt_round(ot.as_vector(v.cores), tol, max_rank),
                                                rows, cols))
        return tt.TTVector(ot.tt_round(v.cores, tol, max_rank))

    def add(a, b):
        return type(a)(ot.tt_add(a.cores, b.cores))

    def app(op, v):
        return tt.TTVector(ot.tt_apply(op.cores, v.cores))

    return assembly.setup_backend(round=rnd, add=add, apply=app)


def oracle_problem(recipe):
    """The workload's trains built with the oracle doing the setup numerics."""
    from paper_2506_04732_b200 import workloads as wl

    with cpu_backend():
        return wl.march_problem(recipe)


def cpu_march(recipe, n_steps, start_step=1, state=None, problem=None):
    from oracle import als_solver as als
    from oracle import march as om

    left, right, state0, forcing, _, _ = problem or oracle_problem(recipe)
    st = state if state is not None else state0.cores
    cfg = als.Config(**recipe.solver)
    with cpu_backend():
        forc = {k: forcing(k) for k in range(start_step, start_step + n_steps)}
    t0 = time.perf_counter()
    for k in range(start_step, start_step + n_steps):
        bc, src = forc[k]
        st, _, _ = om.step(left.cores, right.cores, st, bc.cores, src.cores, recipe.step_tol, cfg,
                           index=k)
    return time.perf_counter() - t0, st


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2506_04732_b200 import workloads as wl

    recipe = wl.config(CONFIG_INDEX)
    problem = oracle_problem(recipe)
    _, state = cpu_march(recipe, args.warmup, problem=problem)
    elapsed, _ = cpu_march(recipe, args.steps, start_step=args.warmup + 1, state=state,
                           problem=problem)
    value = args.steps / elapsed
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(recipe, {"parallelism": "cpu"}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} timed steps after {args.warmup} warm-up "
                                   "steps of the config-2 march (oracle port of "
                                   "pkg/src/ttss, numpy/BLAS)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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


def run_b200(args):
    import torch

    from paper_2506_04732_b200 import _native, workloads as wl
    from paper_2506_04732_b200.march import march_device
    from paper_2506_04732_b200.solver import SolverConfig
    from paper_2506_04732_b200.tt import to_device

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(local)
    os.environ["T2S2_DEVICE"] = str(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")

    recipe = wl.config(CONFIG_INDEX)
    W, K = args.warmup, args.steps
    left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
    forc = [forcing(k) for k in range(1, W + K + 1)]
    cfg = SolverConfig(**recipe.solver)
    ctx = _native.context()
    eng_stream = torch.cuda.ExternalStream(_native.lib().t2s2_stream(ctx))
    hl, hr = to_device(left), to_device(right)
    hbc = [to_device(b) for b, _ in forc]
    hsrc = [to_device(s) for _, s in forc]
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def one_step(state, k):
        stored, rows = march_device(hl, hr, state, 1, [hbc[k - 1]], [hsrc[k - 1]],
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
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    _native.stats_reset(profile_events=False)
    rows = []
    total_ms = 0.0
    state = warm_state
    with Clocks(local) as clk:
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
    launch_stats = _native.stats_read()
    gpu_launches = sum(v["launches"] for v in launch_stats.values())
    final_state = state
    elapsed = total_ms / 1e3
    if dist:
        t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        dist.barrier()
    value = world * K / elapsed

    # accuracy of the timed march against the analytic solution
    from paper_2506_04732_b200.tt import from_device, tt_add, tt_norm, tt_scale

    fin = from_device(final_state)
    ex = exact((W + K) * recipe.dt)
    exact_err = float(tt_norm(tt_add(fin, tt_scale(ex, -1.0))) / tt_norm(ex))
    final_state.free()

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

    # e2e: public API, pinned host buffers; per step H2D of the step's
    # forcing trains and D2H of the new state; the same steps W+1 .. W+K
    # replayed from the same warm state, L2 flushed between steps like the
    # device-timed run
    h2d = d2h = 0
    e2e_ms = 0.0
    host_state = warm_state
    pinned = {}

    def pin(cores):
        flat = np.concatenate([c.ravel() for c in cores])
        t = torch.empty(flat.size, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = flat
        return t

    for k in range(W + 1, W + K + 1):
        b, s = forc[k - 1]
        pinned[k] = (pin(b.cores), pin(s.cores), b, s)
    out_buf = torch.empty(4 * 1024 * 1024, dtype=torch.float64, pin_memory=True)
    for k in range(W + 1, W + K + 1):
        pb, ps, b, s = pinned[k]
        l2_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng_stream)
        db = _native.DeviceTrain.upload_flat(pb.data_ptr(), b.mode_sizes, None, b.ranks)
        ds = _native.DeviceTrain.upload_flat(ps.data_ptr(), s.mode_sizes, None, s.ranks)
        stored, _ = march_device(hl, hr, host_state, 1, [db], [ds], recipe.step_tol, cfg,
                                 store_stride=1)
        nxt = stored[1]
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
    warm_state.free()
    e2e_elapsed = e2e_ms / 1e3
    if dist:
        t = torch.tensor([e2e_elapsed], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_elapsed = float(t.item())

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel family
    fam = max(prof.items(), key=lambda kv: kv[1]["device_ms"])
    name, st = fam
    peak64 = fp64_gemm_peak_tflops(torch)
    peaks = measured_peaks()
    flop_bound = st["flops"] > 0 and (st["flops"] / max(st["bytes"], 1.0)) > 2.0
    per_launch_ms = st["device_ms"] / max(st["launches"], 1)
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(name)
    except Exception:
        pass
    if flop_bound:
        achieved = st["flops"] / (st["device_ms"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak64, "unit": "TFLOP/s",
                "frac": achieved / peak64, "traffic": traffic, "kernel": name,
                "peak_source": "cuBLAS DGEMM 8192^3 fp64 measured in this run "
                               "(MEASURED_PEAKS.json has no fp64 figure)",
                "algorithmic_per_launch": st["flops"] / max(st["launches"], 1),
                "avg_launch_ms": per_launch_ms, "launches": st["launches"]}
    else:
        hbm = peaks.get("hbm_gbs", 6650.0)
        achieved = st["bytes"] / (st["device_ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "kernel": name,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
                else "fallback 6650 GB/s (B200_PROFILING.md)",
                "algorithmic_per_launch": st["bytes"] / max(st["launches"], 1),
                "avg_launch_ms": per_launch_ms, "launches": st["launches"]}
    tot_prof = sum(v["device_ms"] for v in prof.values())
    kernels = {k: {"launches": v["launches"], "device_ms": round(v["device_ms"], 3),
                   "share": round(v["device_ms"] / tot_prof, 4) if tot_prof else 0.0,
                   "gflop": round(v["flops"] / 1e9, 4)}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["device_ms"])}

    cpu = None
    if not args.no_cpu_baseline and args.cpu_sample_steps > 0:
        problem = oracle_problem(recipe)
        _, st = cpu_march(recipe, W, problem=problem)          # untimed warm-up steps
        el, _ = cpu_march(recipe, args.cpu_sample_steps, start_step=W + 1, state=st,
                          problem=problem)
        cpu = {"value": args.cpu_sample_steps / el, "unit": UNIT, "cores": blas_threads(),
               "kind": "port",
               "sample": f"steps {W + 1}..{W + args.cpu_sample_steps} of the same config-2 "
                         f"march after {W} untimed steps, oracle port (numpy/BLAS) on this host"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": 1e3 * elapsed / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (manufactured translating Gaussian, seeded)",
        "config": workload_config(recipe, {
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "l2": "256 MiB write between timed steps (not timed)",
            "timed_steps": f"{W + 1}..{W + K}",
            "max_rank_seen": max(r[1] for r in rows),
            "sweeps_per_step": [r[4] for r in rows],
            "exact_rel_error_final": exact_err,
        }),
        "roofline": roof,
        "kernels": kernels,
        "gpu_launches": gpu_launches,
        "e2e": {"value": world * K / e2e_elapsed, "unit": UNIT, "h2d_bytes_per_step": h2d // K,
                "d2h_bytes_per_step": d2h // K},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "wall_s_timed": t_wall,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
