"""Step-by-step trace of a BASELINE march on the device (development tool):
per step wall time, max rank, sweeps, final residual."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import to_device
idx = int(sys.argv[1]); n = int(sys.argv[2])
over = {}
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    over[k] = float(v) if "." in v or "e" in v else int(v)
recipe = wl.config(idx)
solver_kw = dict(recipe.solver)
step_tol = over.pop("step_tol", recipe.step_tol)
solver_kw.update(over)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
hl, hr, hs = to_device(left), to_device(right), to_device(state0)
cfg = SolverConfig(**solver_kw)
print("solver", solver_kw, "step_tol", step_tol, flush=True)
state = hs
t_all = time.perf_counter()
for k in range(1, n + 1):
    b, s = forcing(k)
    hb, hsrc = to_device(b), to_device(s)
    t0 = time.perf_counter()
    try:
        stored, rows = march_device(hl, hr, state, 1, [hb], [hsrc], step_tol, cfg, store_stride=1)
    except Exception as e:
        print("step", k, "FAILED", e, flush=True)
        break
    _native.synchronize()
    dt = time.perf_counter() - t0
    state = stored[1]
    r = rows[0]
    print(f"step {k:3d} {dt*1e3:8.1f} ms rank {r[1]:3d} sweeps {r[4]:2d} res {r[3]:.2e} ranks {state.ranks}", flush=True)
print("total", time.perf_counter() - t_all)
