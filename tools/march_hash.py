"""Bit-level fingerprint of a march: SHA-1 of every stored state's cores, the
sweeps and the launch count per step.  Two builds whose kernels perform the
same arithmetic print the same hashes (used to check that launch fusions and
layout changes leave the trajectory bit-identical).

    python tools/march_hash.py <config> [--steps N] [--out file.json]
"""
import argparse, hashlib, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--steps", type=int, default=25)
ap.add_argument("--out", default="")
args = ap.parse_args()

from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import from_device, to_device

recipe = wl.config(args.config)
n = args.steps
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
forc = [forcing(k) for k in range(1, n + 1)]
hl, hr, hs = to_device(left), to_device(right), to_device(state0)
bcs = [to_device(b) for b, _ in forc]
srcs = [to_device(s) for _, s in forc]
cfg = SolverConfig(**recipe.solver)
walls = []
for rep in range(3):  # the last run is the one fingerprinted; its wall time is warm
    _native.synchronize()
    _native.stats_reset(profile_events=False)
    t0 = time.perf_counter()
    stored, rows = march_device(hl, hr, hs, n, bcs, srcs, recipe.step_tol, cfg, store_stride=1)
    _native.synchronize()
    walls.append(round(time.perf_counter() - t0, 4))
    if rep < 2:
        for h in stored.values():
            h.free()
wall = min(walls)
launches = sum(v["launches"] for v in _native.stats_read().values())
steps = []
for k in range(1, n + 1):
    t = from_device(stored[k])
    h = hashlib.sha1()
    for c in t.cores:
        h.update(np.ascontiguousarray(c).tobytes())
    steps.append({"step": k, "sha1": h.hexdigest()[:16], "ranks": list(t.ranks), "sweeps": int(rows[k - 1][4])})
out = {"config": args.config, "steps": n, "wall_s": wall, "walls": walls, "launches": launches,
       "sweeps_total": sum(s["sweeps"] for s in steps), "states": steps}
print(json.dumps({k: v for k, v in out.items() if k != "states"}))
print(" ".join(s["sha1"][:6] for s in steps))
if args.out:
    json.dump(out, open(args.out, "w"), indent=0)
