"""Quick device timing of the config-2 march (development helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t0 = time.time()
recipe = wl.config(idx)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
fs = [forcing(k) for k in range(1, steps + 1)]
print("setup", time.time() - t0, "left ranks", left.ranks, flush=True)
hl, hr, hs = to_device(left), to_device(right), to_device(state0)
bcs = [to_device(b) for b, _ in fs]; srcs = [to_device(s) for _, s in fs]
cfg = SolverConfig(**recipe.solver)
_native.check(_native.lib().t2s2_synchronize(_native.context()))
prof = len(sys.argv) > 3 and sys.argv[3] == "prof"
# T2S2_PROFILE_FROM=k: cudaProfilerStart before step k (ncu --profile-from-start off)
prof_from = int(os.environ.get("T2S2_PROFILE_FROM", "-1"))
state = hs
tot = 0.0
for k in range(steps):
    if k == prof_from:
        import ctypes
        ctypes.CDLL("libcudart.so.12").cudaProfilerStart()
    _native.stats_reset(profile_events=prof)
    t0 = time.time()
    stored, rows = march_device(hl, hr, state, 1, [bcs[k]], [srcs[k]], recipe.step_tol, cfg, store_stride=1)
    _native.synchronize()
    dt = time.time() - t0
    tot += dt
    state = stored[1]
    st = _native.stats_read()
    top = sorted(st.items(), key=lambda kv: -kv[1]["device_ms"] if prof else -kv[1]["launches"])[:8]
    print(f"step {k+1}: {dt*1e3:.1f} ms", rows[0], "launches", sum(v["launches"] for v in st.values()))
    for name, v in top:
        print(f"    {name:16s} n={v['launches']:6d} ms={v['device_ms']:9.3f} gflop={v['flops']/1e9:8.4f}")
print(f"{steps} steps in {tot:.3f}s -> {steps/tot:.2f} steps/s")
