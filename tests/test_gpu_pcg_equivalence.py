"""The Jacobi-PCG local solves run their whole iteration loop in one
cooperative kernel with the matvec program inside it (csrc/iterative.cu,
pcg).  Operators whose matvec does not fit one program get the matvec as a
separate launch per iteration and the same kernel for the vector part;
T2S2_PCG_EXTERNAL_MATVEC=1 forces that form.  Same arithmetic in the same
order, grid barriers instead of launch boundaries: the two solves must agree
bit for bit (config 1, d=3 n=33 eps=1e-6, whose local least-squares solves
go through PCG)."""
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


def _run(external):
    env = dict(os.environ, ROOT=ROOT)
    env.pop("T2S2_PCG_EXTERNAL_MATVEC", None)
    if external:
        env["T2S2_PCG_EXTERNAL_MATVEC"] = "1"
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")][-1]
    return line.split(" ", 1)[1]


@pytest.mark.gpu
def test_pcg_loop_kernel_is_bit_identical_to_per_iteration_launches():
    fused, external = _run(False), _run(True)
    assert fused.rsplit(" ", 1)[0] == external.rsplit(" ", 1)[0]
    # one launch per local solve against one per iteration (plus the top)
    assert 0 < int(fused.rsplit(" ", 1)[1]) < int(external.rsplit(" ", 1)[1])
