"""Per-family device time of one config-4 steady solve (development helper).

    python tools/profile_solve.py [recipe_index] [max_sweeps] [prof]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native, workloads as wl  # noqa: E402
from paper_2506_04732_b200.solver import solve  # noqa: E402
from paper_2506_04732_b200.solver import SolverConfig  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prof = len(sys.argv) > 3 and sys.argv[3] == "prof"
recipes = wl.sweep_recipes()
r = recipes[idx]
a, b, exact, _ = wl.steady_problem(r)
cfg = dict(r.solver)
cfg["max_sweeps"] = sweeps
_native.context()
_native.stats_reset(profile_events=prof)
t0 = time.perf_counter()
x, rep = solve(a, b, cfg=SolverConfig(**cfg))
el = time.perf_counter() - t0
print(f"recipe {idx} eps={r.eps:.3e} sweeps={len(rep.residual_history)} wall {el:.2f}s")
print("  residuals", ["%.2e" % v for v in rep.residual_history])
print("  ranks", rep.rank_history)
st = _native.stats_read()
tot = sum(v["device_ms"] for v in st.values()) or 1.0
for name, v in sorted(st.items(), key=lambda kv: -kv[1]["device_ms"] if prof else -kv[1]["launches"]):
    print(f"    {name:16s} n={v['launches']:8d} ms={v['device_ms']:10.2f} ({100 * v['device_ms'] / tot:4.1f}%)"
          f" gflop={v['flops'] / 1e9:10.3f} tflops={v['flops'] / max(v['device_ms'], 1e-9) / 1e9:6.2f}")
if prof and len(sys.argv) > 4:
    # the GEMM programs grouped by algorithmic flops (one group ~ one program shape)
    import collections

    groups = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for fam, fl, by, ms in _native.launch_log():
        if fam == "gemm":
            g = groups[round(fl / 1e3)]
            g[0] += 1
            g[1] += ms
            g[2] = fl
    tot = sum(v[1] for v in groups.values())
    print("  GEMM programs by flop count (top 12 by time):")
    for key, (n, ms, fl) in sorted(groups.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"    {fl / 1e6:10.2f} MFLOP x{n:6d}  {ms:9.1f} ms ({100 * ms / tot:4.1f}%)  "
              f"{1e3 * ms / n:7.1f} us/launch  {fl / (ms / n) / 1e9:6.2f} TF")
