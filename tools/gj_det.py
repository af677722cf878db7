"""Determinism stress test of the no-pivot Gauss-Jordan solve (diagonally dominant systems; DET_SIZES="1953 2000" are the sizes that exposed the hand-off race fixed in round 2):
the same systems solved repeatedly must give bit-identical results."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native  # noqa: E402

if os.environ.get('T2S2_LIB'):
    _native.load_library(os.environ['T2S2_LIB'])

if os.environ.get('BUDGET'):
    _native.context()
    _native.set_thread_sm_budget(int(os.environ['BUDGET']))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(3)
for n in [int(x) for x in os.environ.get('DET_SIZES', '66 264 792 1188 1848').split()]:
    a = rng.standard_normal((n, n))
    a += np.diag(np.abs(a).sum(0))
    b = rng.standard_normal(n)
    ref = _native.dense_solve(a, b)
    bad = 0
    for _ in range(reps):
        x = _native.dense_solve(a, b)
        if not np.array_equal(x, ref):
            bad += 1
    print(f"N={n}: {bad}/{reps} runs differ", flush=True)
