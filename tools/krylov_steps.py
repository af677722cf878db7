import os, sys
sys.path.insert(0, '/root/repo')
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import to_device
import time
recipe = wl.config(2)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
hl, hr, state = to_device(left), to_device(right), to_device(state0)
cfg = SolverConfig(**recipe.solver)
tot = 0
for k in range(1, 101):
    bc, src = (to_device(t) for t in forcing(k))
    _native.stats_reset()
    _native.synchronize(); t0 = time.perf_counter()
    stored, rows = march_device(hl, hr, state, 1, [bc], [src], recipe.step_tol, cfg, store_stride=1)
    _native.synchronize(); dt = time.perf_counter() - t0
    state = stored[1]
    st = _native.stats_read()
    g = st.get("gmres", {}).get("launches", 0); c = st.get("cg", {}).get("launches", 0); lu = st.get("lu_fused", {}).get("launches", 0)
    tot += dt
    if g or dt > 0.02:
        print(f"step {k}: {dt*1e3:6.1f} ms sweeps {rows[0][4]} gmres launches {g} cg {c} lu {lu} gj {st.get('gj_nopivot',{}).get('launches',0)}")
print("total", tot)
