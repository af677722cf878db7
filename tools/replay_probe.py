"""What do the synchronising host reads of a step cost?  Each step of the
config-2 march runs twice from the same input state: once recording every
device->host read that steers the host, once with the recorded values handed
back without synchronising (the host runs ahead of the device, as a
device-decided or graph-replayed step would).  Same kernels, same results;
the time difference is the idle time the reads cause."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_04732_b200 import _native, workloads as wl
from paper_2506_04732_b200.march import march_device
from paper_2506_04732_b200.solver import SolverConfig
from paper_2506_04732_b200.tt import from_device, to_device

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 23
first = int(sys.argv[3]) if len(sys.argv) > 3 else 4
recipe = wl.config(idx)
left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
fs = [forcing(k) for k in range(1, steps + 1)]
hl, hr, state = to_device(left), to_device(right), to_device(state0)
bcs = [to_device(b) for b, _ in fs]
srcs = [to_device(s) for _, s in fs]
cfg = SolverConfig(**recipe.solver)
ctx = _native.context()
stream = torch.cuda.ExternalStream(_native.lib().t2s2_stream(ctx))


def timed(k, st):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _native.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    stored, rows = march_device(hl, hr, st, 1, [bcs[k]], [srcs[k]], recipe.step_tol, cfg, store_stride=1)
    t_host = time.perf_counter() - t0
    e1.record(stream)
    e1.synchronize()
    return stored[1], rows[0], e0.elapsed_time(e1), 1e3 * t_host


tot = [0.0, 0.0]
for k in range(steps):
    if k + 1 < first:
        nxt, _, _, _ = timed(k, state)
        state = nxt
        continue
    _native.read_trace(1)  # record (the determinism probes' buffers join the trace: not timed)
    r, _, _, _ = timed(k, state)
    r.free()
    _native.read_trace(0)
    a, row, ms_sync, host_sync = timed(k, state)  # the plain, synchronising run
    nreads = _native.read_trace(2)
    b, _, ms_free, host_free = timed(k, state)
    _native.read_trace(0)
    ca, cb = from_device(a).cores, from_device(b).cores
    same = all(np.array_equal(x, y) for x, y in zip(ca, cb))
    tot[0] += ms_sync
    tot[1] += ms_free
    print(f"step {k+1}: sweeps {row[4]} trace entries {nreads}  synchronising {ms_sync:7.2f} ms  "
          f"read-free {ms_free:7.2f} ms (host enqueue {host_free:6.2f} ms)  identical {same}", flush=True)
    state = a
print(f"steps {first}..{steps}: synchronising {tot[0]:.1f} ms, read-free {tot[1]:.1f} ms, ratio {tot[0]/tot[1]:.3f}")
