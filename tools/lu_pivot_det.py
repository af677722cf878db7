"""Repeated pivoted dense solves of the same system must agree bit for bit
(DET_SIZES="..." sizes, BUDGET=<CTAs> caps the cooperative grid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2506_04732_b200 import _native
_native.context()
if os.environ.get("BUDGET"):
    _native.set_thread_sm_budget(int(os.environ["BUDGET"]))
rng = np.random.default_rng(1)
for n in [int(x) for x in os.environ.get("DET_SIZES", "264 792 1188 1617 1848").split()]:
    a = rng.standard_normal((n, n)) + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    outs = [_native.dense_solve(a, b) for _ in range(40)]
    ref = np.linalg.solve(a, b)
    ndiff = sum(not np.array_equal(outs[0], o) for o in outs)
    print(n, "runs differing from the first:", ndiff, "rel err", np.abs(outs[0] - ref).max() / np.abs(ref).max(), flush=True)
