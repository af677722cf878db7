"""Debug: config 1 full size, residual history and manufactured-solution
error (development helper; reads the committed fixture)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from golden_io import get_train  # noqa: E402
from oracle import tt_ops as ot  # noqa: E402
from paper_2506_04732_b200 import solver, tt, workloads as wl  # noqa: E402

z = dict(np.load(os.path.join(ROOT, "tests/golden/config1.npz")))
recipe = wl.config(1)
cfg = solver.SolverConfig(**recipe.solver)
x, rep = solver.solve(tt.TTOperator(get_train(z, "a")), tt.TTVector(get_train(z, "b")),
                      x0=tt.TTVector(get_train(z, "x0")), cfg=cfg)
a, b, exact, opset = wl.steady_problem(recipe)
err = ot.tt_norm(ot.tt_add(x.cores, ot.tt_scale(exact.cores, -1.0))) / ot.tt_norm(exact.cores)
print("device res", " ".join(f"{r:.2e}" for r in rep.residual_history))
print("ranks", rep.rank_history)
print("ref    res", " ".join(f"{r:.2e}" for r in z["res"]))
print("err", err, "ref err", float(z["exact_err"]))
