"""Add the reference-equivalent envelope to tests/golden/config4_full_<i>.npz:
the same complete solve by ttss with another BLAS thread count
(tools/make_golden_full.py cfg4 with OPENBLAS_NUM_THREADS=1 and
T2S2_GOLDEN_OUT=<dir>) and by the numpy oracle (tools/oracle_config4.py).
Rank-capped config-4 solves end on a path-dependent plateau: ttss itself
moves its final residual by 2.6x between 1 and 2 threads (seed 0).

    python tools/config4_envelope.py <other-ttss-dir> <oracle-json-dir> SEED...
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
other, odir = sys.argv[1], sys.argv[2]
for seed in (int(s) for s in sys.argv[3:]):
    path = os.path.join(ROOT, "tests", "golden", f"config4_full_{seed}.npz")
    z = dict(np.load(path))
    res, err, src = [float(z["res"][-1])], [float(z["exact_err"])], [f"ttss {int(z['blas_threads'])} threads"]
    o = os.path.join(other, f"config4_full_{seed}.npz")
    if os.path.exists(o):
        w = np.load(o)
        res.append(float(w["res"][-1]))
        err.append(float(w["exact_err"]))
        src.append(f"ttss {int(w['blas_threads'])} threads")
    j = os.path.join(odir, f"oracle_c4_{seed}.json")
    if os.path.exists(j):
        d = json.load(open(j))
        res.append(float(d["res"][-1]))
        err.append(float(d["err"]))
        src.append("numpy oracle (oracle/als_solver.py)")
    z["env_res"], z["env_err"], z["env_src"] = np.array(res), np.array(err), np.array(src)
    np.savez_compressed(path, **z)
    print(seed, dict(zip(src, zip(res, err))))
