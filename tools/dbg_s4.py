"""Debug: golden solver case s4 with forced Krylov local solves, device vs
oracle residual histories (development helper)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from oracle import als_solver as als  # noqa: E402
from paper_2506_04732_b200 import solver, tt  # noqa: E402

z = dict(np.load(os.path.join(ROOT, "tests/golden/solve_small.npz")))
tag = sys.argv[1] if len(sys.argv) > 1 else "s4"


def get(name):
    n = int(z[f"{name}_d"])
    return [z[f"{name}_{l}"] for l in range(n)]


from golden_io import get_train  # noqa: E402

a, b, x0 = get_train(z, f"{tag}_a"), get_train(z, f"{tag}_b"), get_train(z, f"{tag}_x0")
kw = {k[len(tag) + 5:]: z[k].item() for k in z if k.startswith(f"{tag}_cfg_")}
kw["local_solver"] = sys.argv[2] if len(sys.argv) > 2 else "iterative"
print(kw)
x, rep = solver.solve(tt.TTOperator(a), tt.TTVector(b), x0=tt.TTVector(x0), cfg=solver.SolverConfig(**kw))
xo, repo = als.solve(a, b, x0=x0, cfg=als.Config(**kw))
print("device", [f"{r:.3e}" for r in rep.residual_history], rep.converged, rep.rank_history)
print("oracle", [f"{r:.3e}" for r in repo.residual_history], repo.converged, repo.rank_history)
print("device choices", getattr(rep, "choices", None))
print("oracle choices", repo.choices)
