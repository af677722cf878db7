"""Determinism probe: every step of the config-2 march runs twice from the
same input state; the second run compares each device->host read with the
first run's (t2s2_read_trace mode 3) and the resulting states bit for bit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import from_device, to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
recipe = wl.config(idx)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
fs = [forcing(k) for k in range(1, steps + 1)]
hl, hr, state = to_device(left), to_device(right), to_device(state0)
bcs = [to_device(b) for b, _ in fs]
srcs = [to_device(s) for _, s in fs]
cfg = SolverConfig(**recipe.solver)
_native.context()
for k in range(steps):
    _native.read_trace(1)
    _native.stats_reset()
    a, rows = march_device(hl, hr, state, 1, [bcs[k]], [srcs[k]], recipe.step_tol, cfg, store_stride=1)
    st = {n: v["launches"] for n, v in _native.stats_read().items() if v["launches"]}
    n = _native.read_trace(3)
    b, _ = march_device(hl, hr, state, 1, [bcs[k]], [srcs[k]], recipe.step_tol, cfg, store_stride=1)
    _native.read_trace(0)
    same = all(np.array_equal(x, y) for x, y in zip(from_device(a[1]).cores, from_device(b[1]).cores))
    print(f"step {k+1}: sweeps {rows[0][4]} reads {n} identical {same} cg {st.get('cg',0)} gmres {st.get('gmres',0)} lu {st.get('lu_fused',0)}", flush=True)
    state = a[1]
