"""Config-4 seed solved by the engine and by ttss (and the oracle) at a
scaled size, residual histories side by side (development aid).

    python tools/c4_scaled.py SEED DIMS DEGREE MAX_RANK SWEEPS
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import workloads as wl  # noqa: E402
from paper_2506_04732_b200.reference import module  # noqa: E402

seed, dims, degree, max_rank, sweeps = (int(v) for v in sys.argv[1:6])
r = wl.sweep_recipes(dims=dims, degree=degree)[seed]
a, b, exact, _ = wl.steady_problem(r)
rsol = module("tt_solver")
kw = dict(r.solver, max_rank=max_rank, max_sweeps=sweeps)
out = {}
t0 = time.time()
from paper_2506_04732_b200 import solver as dsol  # noqa: E402

xd, rd = dsol.solve(a, b, cfg=dsol.SolverConfig(**kw))
out["b200"] = (rd.residual_history, time.time() - t0)
t0 = time.time()
xr, rr = rsol.solve(a, b, cfg=rsol.SolverConfig(**kw))
out["ttss"] = (rr.residual_history, time.time() - t0)
if len(sys.argv) > 6:
    from oracle import als_solver as als
    t0 = time.time()
    xo, ro = als.solve(a.cores, b.cores, cfg=als.Config(**kw))
    out["oracle"] = (ro.residual_history, time.time() - t0)
print(f"seed {seed} eps {r.eps:.3e} d={dims} n={degree + 1} cap {max_rank}")
for k, (h, t) in out.items():
    print(f"{k:7s} {t:7.1f}s", " ".join(f"{v:.3e}" for v in h))
print("choices b200 (per core visit, 0 old / 1 Galerkin / 2 LS):")
