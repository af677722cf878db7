"""The Krylov local solves run their iteration loops on the device
(csrc/iterative.cu): Jacobi-PCG as one cooperative kernel for the whole loop,
GMRES as one per restart cycle, each with the matvec program inside.
Operators whose matvec does not fit one program get the matvec as a separate
launch per iteration and the same kernels for the vector part;
T2S2_KRYLOV_EXTERNAL_MATVEC=1 forces that form.  Same arithmetic in the same
order, grid barriers instead of launch boundaries: the two solves must agree
bit for bit (config 1, d=3 n=33 eps=1e-6: local systems beyond the direct
size, least-squares candidates by PCG; and three steps of the config-2 march,
whose enriched cores take the GMRES path)."""
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
h = hashlib.sha256()
for c in x.cores:
    h.update(np.ascontiguousarray(c, dtype=np.float64).tobytes())
# three steps of the config-2 march: enriched cores cross the direct-solve
# size in steps 2 and 3 (GMRES for the Galerkin candidates)
from paper_2506_04732_b200.march import march_device
recipe = wl.config(2)
left, right, state0, forcing, _, _ = wl.march_problem(recipe)
hl, hr, state = tt.to_device(left), tt.to_device(right), tt.to_device(state0)
for k in range(1, 4):
    bc, src = (tt.to_device(t) for t in forcing(k))
    stored, _ = march_device(hl, hr, state, 1, [bc], [src], recipe.step_tol,
                             solver.SolverConfig(**recipe.solver), store_stride=1)
    state = stored[1]
for c in tt.from_device(state).cores:
    h.update(np.ascontiguousarray(c, dtype=np.float64).tobytes())
st = _native.stats_read()
print("RESULT", h.hexdigest(), repr(list(rep.residual_history)),
      "%d/%d" % (st.get("cg", {}).get("launches", 0), st.get("gmres", {}).get("launches", 0)))
"""


def _run(external):
    env = dict(os.environ, ROOT=ROOT)
    env.pop("T2S2_KRYLOV_EXTERNAL_MATVEC", None)
    if external:
        env["T2S2_KRYLOV_EXTERNAL_MATVEC"] = "1"
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")][-1]
    return line.split(" ", 1)[1]


@pytest.mark.gpu
def test_krylov_loop_kernels_are_bit_identical_to_per_iteration_launches():
    fused, external = _run(False), _run(True)
    assert fused.rsplit(" ", 1)[0] == external.rsplit(" ", 1)[0]
    # one launch per solve / restart cycle against one per iteration
    (fc, fg), (ec, eg) = ([int(v) for v in r.rsplit(" ", 1)[1].split("/")] for r in (fused, external))
    assert 0 < fc < ec and 0 < fg < eg
