"""Throughput of the config-4 parameter sweep (solves/s) on one GPU, with
k concurrent engine contexts.  Scaled by default (development tool):

    python tools/bench_sweep.py [count] [dims] [degree] [max_sweeps] [concurrency...]
"""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import sweep, workloads as wl

count = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dims = int(sys.argv[2]) if len(sys.argv) > 2 else 6
degree = int(sys.argv[3]) if len(sys.argv) > 3 else 32
sweeps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
conc = [int(c) for c in sys.argv[5:]] or [1, 4]
recipes = wl.sweep_recipes(count=count, dims=dims, degree=degree)
for k in conc:
    t0 = time.perf_counter()
    res = sweep.run_sweep(recipes, overrides={"max_sweeps": sweeps}, concurrency=k)
    el = time.perf_counter() - t0
    print(json.dumps({"concurrency": k, "solves": count, "dims": dims, "nodes": degree + 1,
                      "max_sweeps": sweeps, "wall_s": el, "solves_per_s": count / el,
                      "final_residuals": [res[i]["residuals"][-1] for i in range(count)],
                      "max_ranks": [max(res[i]["ranks"]) for i in range(count)]}), flush=True)
