import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import als_solver as als
from paper_2506_04732_b200 import workloads as wl
from paper_2506_04732_b200.solver import solve, SolverConfig
idx = int(sys.argv[1]); sweeps = int(sys.argv[2])
r = wl.sweep_recipes()[idx]
a, b, exact, _ = wl.steady_problem(r)
kw = dict(r.solver); kw["max_sweeps"] = sweeps
choices = []
orig = als.Sweep.update if hasattr(als, "Sweep") else None
xo, repo = als.solve(a.cores, b.cores, cfg=als.Config(**kw))
print("oracle", os.environ.get("OPENBLAS_NUM_THREADS"), repo.residual_history, [c.shape for c in xo][:3])
if len(sys.argv) > 3:
    x, rep = solve(a, b, cfg=SolverConfig(**kw))
    print("device", rep.residual_history, [c.shape for c in x.cores][:3])
