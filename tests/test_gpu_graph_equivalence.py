"""The Jacobi-PCG local solves replay a captured CUDA graph of whole
iterations (csrc/iterative.cu, pcg); with T2S2_NO_GRAPH=1 the same
iterations are launched eagerly.  Same kernels, same parameters, same
order: the two solves must agree bit for bit (config 1, d=3 n=33
eps=1e-6, whose local least-squares solves go through PCG)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, os, sys
sys.path.insert(0, os.environ["ROOT"])
sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np
from golden_io import get_train
from paper_2506_04732_b200 import _native, solver, tt, workloads as wl
z = dict(np.load(os.path.join(os.environ["ROOT"], "tests", "golden", "config1.npz")))
kw = dict(wl.config(1).solver)
kw["max_sweeps"] = 4
x, rep = solver.solve(tt.TTOperator(get_train(z, "a")), tt.TTVector(get_train(z, "b")),
                      x0=tt.TTVector(get_train(z, "x0")), cfg=solver.SolverConfig(**kw))
st = _native.stats_read()
h = hashlib.sha256()
for c in x.cores:
    h.update(np.ascontiguousarray(c, dtype=np.float64).tobytes())
print("RESULT", h.hexdigest(), repr(list(rep.residual_history)), st.get("cg", {}).get("launches", 0))
"""


def _run(no_graph):
    env = dict(os.environ, ROOT=ROOT)
    env.pop("T2S2_NO_GRAPH", None)
    if no_graph:
        env["T2S2_NO_GRAPH"] = "1"
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")][-1]
    return line.split(" ", 1)[1]


@pytest.mark.gpu
def test_pcg_graph_replay_is_bit_identical_to_eager_launches():
    graph, eager = _run(False), _run(True)
    assert graph.rsplit(" ", 1)[0] == eager.rsplit(" ", 1)[0]
    # the replayed graphs count their kernels like eager launches
    assert int(graph.rsplit(" ", 1)[1]) == int(eager.rsplit(" ", 1)[1]) > 0
