"""Quick device timing of the config-2 march (development helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t0 = time.time()
recipe = wl.config(idx)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
fs = [forcing(k) for k in range(1, steps + 1)]
print("setup", time.time() - t0, "left ranks", left.ranks, flush=True)
hl, hr, hs = to_device(left), to_device(right), to_device(state0)
bcs = [to_device(b) for b, _ in fs]; srcs = [to_device(s) for _, s in fs]
cfg = SolverConfig(**recipe.solver)
_native.check(_native.lib().t2s2_synchronize(_native.context()))
t0 = time.time()
stored, rows = march_device(hl, hr, hs, steps, bcs, srcs, recipe.step_tol, cfg)
_native.check(_native.lib().t2s2_synchronize(_native.context()))
dt = time.time() - t0
print(f"{steps} steps in {dt:.3f}s -> {steps/dt:.2f} steps/s")
for r in rows: print(r)
