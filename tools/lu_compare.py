"""Dense local-solve timing: the engine's fused LU (t2s2_dense_solve, device
time from the launch accounting) beside cuSOLVER through torch.linalg.solve
on the same matrices (development comparison, not a product path).

    python tools/lu_compare.py [N ...]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native  # noqa: E402

sizes = [int(s) for s in sys.argv[1:]] or [165, 825, 1188, 1617, 1980]
rng = np.random.default_rng(0)
for n in sizes:
    a = rng.standard_normal((n, n))
    if os.environ.get("LU_DOMINANT", "1") == "1":  # no interchanges: the no-pivot path
        a += np.diag(np.abs(a).sum(0))
    b = rng.standard_normal(n)
    _native.dense_solve(a, b)  # warm
    _native.stats_reset(profile_events=True)
    reps = 10
    for _ in range(reps):
        x = _native.dense_solve(a, b)
    st = _native.stats_read()
    fams = [k for k in ("gj_nopivot", "lu_nopivot", "lu_fused") if st.get(k, {}).get("launches", 0)]
    fam = "+".join(fams)
    lu_ms = sum(st[k]["device_ms"] for k in fams) / reps
    err = np.linalg.norm(a @ x - b) / np.linalg.norm(b)
    line = f"N={n:5d} {fam} {lu_ms * 1e3:8.1f} us  resid {err:.1e}"
    try:
        import torch

        ta = torch.tensor(a, device="cuda")
        tb = torch.tensor(b, device="cuda")
        torch.linalg.solve(ta, tb)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            torch.linalg.solve(ta, tb)
        e1.record()
        torch.cuda.synchronize()
        line += f" | cusolver(torch.linalg.solve) {e0.elapsed_time(e1) / reps * 1e3:8.1f} us"
        f0 = time.perf_counter()
        for _ in range(reps):
            torch.linalg.lu_factor(ta)
        torch.cuda.synchronize()
        line += f" | lu_factor wall {(time.perf_counter() - f0) / reps * 1e6:8.1f} us"
    except Exception as exc:  # noqa: BLE001
        line += f" | torch: {exc}"
    print(line, flush=True)
