"""Run a full BASELINE march (config 2: 100 steps, config 3: 200 steps) on the
device and report time, ranks and the error against the manufactured
solution; optionally compare with the CPU oracle run on the same inputs.

    python tools/full_march.py <config> [--oracle] [--steps N]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--oracle", action="store_true")
args = ap.parse_args()

from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import from_device, to_device, tt_add, tt_norm, tt_scale

recipe = wl.config(args.config)
n = args.steps or recipe.n_steps
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
forc = [forcing(k) for k in range(1, n + 1)]
hl, hr, hs = to_device(left), to_device(right), to_device(state0)
bcs = [to_device(b) for b, _ in forc]
srcs = [to_device(s) for _, s in forc]
cfg = SolverConfig(**recipe.solver)
_native.synchronize()
t0 = time.perf_counter()
stored, rows = march_device(hl, hr, hs, n, bcs, srcs, recipe.step_tol, cfg, store_stride=n)
_native.synchronize()
wall = time.perf_counter() - t0
final = from_device(stored[n])
ex = exact(n * recipe.dt)
err = tt_norm(tt_add(final, tt_scale(ex, -1.0))) / tt_norm(ex)
out = {"config": args.config, "steps": n, "wall_s": wall, "steps_per_s": n / wall,
       "final_ranks": list(final.ranks), "max_rank": max(r[1] for r in rows),
       "sweeps_total": sum(r[4] for r in rows), "exact_rel_error": err}
if args.oracle:
    from oracle import als_solver as als, march as om, tt_ops as ot
    t1 = time.perf_counter()
    st = state0.cores
    ocfg = als.Config(**recipe.solver)
    for k in range(1, n + 1):
        b, s = forc[k - 1]
        st, rep, _ = om.step(left.cores, right.cores, st, b.cores, s.cores, recipe.step_tol, ocfg, k)
    out["oracle_wall_s"] = time.perf_counter() - t1
    out["oracle_final_ranks"] = list(ot.ranks_of(st))
    out["oracle_exact_rel_error"] = ot.tt_norm(ot.tt_add(st, ot.tt_scale(ex.cores, -1.0))) / ot.tt_norm(ex.cores)
    fa = ot.tt_full(final.cores) if np.prod(final.mode_sizes) <= 2e6 else None
    rng = np.random.default_rng(0)
    idx = np.column_stack([rng.integers(0, m, 100000) for m in final.mode_sizes])
    def samp(cores):
        o = np.ones((idx.shape[0], 1))
        for l, c in enumerate(cores):
            o = np.einsum("ka,akb->kb", o, c[:, idx[:, l], :])
        return o[:, 0]
    a, b = samp(final.cores), samp(st)
    out["rel_diff_vs_oracle_1e5_samples"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
print(json.dumps(out), flush=True)
