import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
from golden_io import get_train
from paper_2506_04732_b200 import tt, solver, workloads as wl
z = dict(np.load('/root/repo/tests/golden/config1.npz'))
recipe = wl.config(1)
x, rep = solver.solve(tt.TTOperator(get_train(z, "a")), tt.TTVector(get_train(z, "b")), x0=tt.TTVector(get_train(z, "x0")), cfg=solver.SolverConfig(**recipe.solver, max_sweeps=int(sys.argv[1]) if len(sys.argv) > 1 else 40))
print(rep.residual_history, x.ranks)
