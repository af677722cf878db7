"""Launch sequence of one config-2 march step (step 14, one sweep): family tag and
CUDA-event microseconds per launch, in launch order (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import to_device
recipe = wl.config(2)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
hl, hr, state = to_device(left), to_device(right), to_device(state0)
cfg = SolverConfig(**recipe.solver)
for k in range(1, 15):
    bc, src = (to_device(t) for t in forcing(k))
    if k == 14:
        _native.stats_reset(profile_events=True)
    stored, rows = march_device(hl, hr, state, 1, [bc], [src], recipe.step_tol, cfg, store_stride=1)
    state = stored[1]
recs = _native.launch_log()
print(rows, len(recs))
line = []
for name, fl, by, ms in recs:
    tag = {"gj_nopivot": "GJ", "gemm": "g", "vector": "v", "permute": "p", "reduce": "r", "svd_jacobi": "S", "qr": "Q", "galerkin_build": "B", "lu_fused": "LU", "check": "c"}.get(name, name)
    line.append(f"{tag}{ms*1e3:.0f}")
print(" ".join(line))
