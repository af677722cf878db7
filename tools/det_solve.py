"""Determinism of a steady solve: the same config-4 solve (or config-1) twice
in one process, compared read by read (t2s2_read_trace mode 3) and bit by bit.
    python tools/det_solve.py [seed_index] [max_sweeps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.solver import SolverConfig, solve

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
r = wl.sweep_recipes()[idx]
a, b, exact, _ = wl.steady_problem(r)
cfg = dict(r.solver)
cfg["max_sweeps"] = sweeps
_native.context()
_native.read_trace(1)
x1, rep1 = solve(a, b, cfg=SolverConfig(**cfg))
n = _native.read_trace(3)
x2, rep2 = solve(a, b, cfg=SolverConfig(**cfg))
_native.read_trace(0)
same = all(np.array_equal(p, q) for p, q in zip(x1.cores, x2.cores))
print(f"seed {idx} eps {r.eps:.2e} sweeps {len(rep1.residual_history)} reads {n} ranks {rep1.rank_history} identical {same}")
print("  residuals", ["%.3e" % v for v in rep1.residual_history])
