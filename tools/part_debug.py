"""Debug aid: config-4 solves on SM partitions with progress prints and a
stack dump watchdog.  python tools/part_debug.py P SWEEPS COUNT"""
import faulthandler
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(150, exit=True)
from paper_2506_04732_b200 import _native, workloads as wl  # noqa: E402
from paper_2506_04732_b200.solver import SolverConfig, _default_initial_guess, solve_device  # noqa: E402
from paper_2506_04732_b200.tt import to_device  # noqa: E402

P, S, C = (int(v) for v in sys.argv[1:4])
recipes = wl.sweep_recipes()
probs = {i: wl.steady_problem(recipes[i]) for i in range(C)}
print("partitions", _native.sm_partitions(P), flush=True)
queue = list(range(C))
lock = threading.Lock()


def worker(t):
    _native.use_partition(t)
    while True:
        with lock:
            if not queue:
                return
            i = queue.pop(0)
        a, b = to_device(probs[i][0]), to_device(probs[i][1])
        x0 = to_device(_default_initial_guess(probs[i][1], None, np.random.default_rng(0)))
        t0 = time.time()
        print(f"  part {t} solve {i} start", flush=True)
        h, rep = solve_device(a, b, x0, SolverConfig(**recipes[i].solver, max_sweeps=S))
        print(f"  part {t} solve {i} done {time.time() - t0:.2f}s res {rep.residual_history[-1]:.3e}",
              flush=True)
        for x in (h, a, b, x0):
            x.free()


ths = [threading.Thread(target=worker, args=(t,)) for t in range(P)]
for th in ths:
    th.start()
for th in ths:
    th.join()
print("ok", flush=True)
