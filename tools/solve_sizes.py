"""Per-launch profile of config-2 march steps (development/measurement aid).

    python tools/solve_sizes.py [first_step] [count]

Runs steps 1..first_step-1 unprofiled, then profiles `count` steps with the
engine's per-launch log (CUDA events around every launch, t2s2_launch_log)
and prints: the dense local solves by size N (recovered from their
algorithmic flop count 2/3 N^3 + 2 N^2) with their device times, and the
per-family totals.
"""
import collections
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native, workloads as wl  # noqa: E402
from paper_2506_04732_b200.march import march_device  # noqa: E402
from paper_2506_04732_b200.solver import SolverConfig  # noqa: E402
from paper_2506_04732_b200.tt import to_device  # noqa: E402


def solve_n(flops):
    n = round((1.5 * flops) ** (1.0 / 3.0))
    for c in range(max(1, n - 3), n + 4):
        if abs(2.0 / 3.0 * c ** 3 + 2.0 * c * c - flops) < 0.5:
            return c
    return n


def main(first=4, count=20):
    recipe = wl.config(2)
    left, right, state0, forcing, _, _ = wl.march_problem(recipe)
    cfg = SolverConfig(**recipe.solver)
    hl, hr, state = to_device(left), to_device(right), to_device(state0)
    recs = []
    for k in range(1, first + count):
        bc, src = forcing(k)
        hb, hs = to_device(bc), to_device(src)
        if k == first:
            _native.stats_reset(profile_events=True)
        stored, _ = march_device(hl, hr, state, 1, [hb], [hs], recipe.step_tol, cfg,
                                 store_stride=1)
        state.free()
        state = stored[1]
        hb.free()
        hs.free()
    recs = _native.launch_log()
    fam = collections.defaultdict(lambda: [0, 0.0])
    solves = collections.defaultdict(list)
    for name, fl, by, ms in recs:
        fam[name][0] += 1
        fam[name][1] += ms
        if name in ("gj_nopivot", "lu_fused"):
            solves[(name, solve_n(fl))].append(ms)
    tot = sum(v[1] for v in fam.values())
    print(f"{count} steps, {len(recs)} launches, {tot:.2f} ms event-timed kernel time")
    for name, (n, ms) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"  {name:16s} {n:6d} launches {ms:9.3f} ms {100 * ms / tot:5.1f}%")
    print("dense solves by size:")
    rows = []
    for (name, n), v in sorted(solves.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        rows.append({"kernel": name, "N": n, "count": len(v), "avg_us": 1e3 * float(np.mean(v)),
                     "total_ms": float(np.sum(v))})
        print(f"  {name:12s} N={n:5d} x{len(v):4d} avg {1e3 * np.mean(v):8.1f} us "
              f"total {np.sum(v):8.3f} ms")
    # GEMM programs by duration class
    g = [ms for name, fl, by, ms in recs if name == "gemm"]
    if g:
        g = np.array(g) * 1e3
        print("gemm programs by event-timed duration (us): count, total ms")
        edges = [0, 6, 8, 10, 15, 20, 30, 50, 100, 1e9]
        for lo, hi in zip(edges[:-1], edges[1:]):
            m = (g >= lo) & (g < hi)
            print(f"  [{lo:5.0f}, {hi:5.0f})  x{int(m.sum()):5d}  {g[m].sum() / 1e3:8.3f} ms")
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "solve_sizes.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump({"steps": count, "first": first, "families": dict(fam), "solves": rows},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:3]))
