"""One verified no-pivot Gauss-Jordan solve per size (for ncu captures):
python tools/gj_profile.py [N ...]   (default 792 1155 1848)"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native
_native.context()
for n in [int(v) for v in sys.argv[1:]] or [792, 1155, 1848]:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    a += np.diag(np.abs(a).sum(0))
    b = rng.standard_normal(n)
    x = _native.dense_solve(a, b)
    print(n, "residual", np.linalg.norm(a @ x - b) / np.linalg.norm(b), flush=True)
