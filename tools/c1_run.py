"""Config-1 full-size solve through the device path beside the reference's
golden history (development helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
from golden_io import get_train  # noqa: E402
from oracle import tt_ops as ot  # noqa: E402
from paper_2506_04732_b200 import solver, tt, workloads as wl  # noqa: E402

z = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "config1.npz")))
recipe = wl.config(1)
kw = dict(recipe.solver)
if len(sys.argv) > 1:
    kw["max_sweeps"] = int(sys.argv[1])
x, rep = solver.solve(tt.TTOperator(get_train(z, "a")), tt.TTVector(get_train(z, "b")),
                      x0=tt.TTVector(get_train(z, "x0")), cfg=solver.SolverConfig(**kw))
a, b, exact, _ = wl.steady_problem(recipe)
err = ot.tt_norm(ot.tt_add(x.cores, ot.tt_scale(exact.cores, -1.0))) / ot.tt_norm(exact.cores)
print("device   ", " ".join("%.2e" % v for v in rep.residual_history), "ranks", x.ranks, "err %.3e" % err)
print("reference", " ".join("%.2e" % v for v in z["res"]), "err %.3e" % float(z["exact_err"]))
print("wall", rep.wall_time)
