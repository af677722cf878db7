"""Run-to-run determinism of the engine, and the read trace itself.

Every device->host read that steers the host goes through host_read
(csrc/api.cu); t2s2_read_trace records them, replays them to an identical
run without synchronising, or compares a second run against the record.
The hand-offs inside the kernels (arrival counters, named barriers, grid
barriers in the Krylov loops) must not let timing reach the numbers: the
same step run twice gives the same bits.  (This probe is what found the
Gauss-Jordan hand-off race fixed in round 2: step 4 of the march, a local
system of N = 1980.)"""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def pk():
    from paper_2506_04732_b200 import _native

    _native.context()  # fail loudly if the engine cannot start
    return _native


def _march_steps(pk, steps, second):
    """Steps 1..steps of the config-2 march, each run twice from the same
    state: recorded, then under read-trace mode ``second``."""
    from paper_2506_04732_b200 import _native, workloads as wl
    from paper_2506_04732_b200.march import march_device
    from paper_2506_04732_b200.solver import SolverConfig
    from paper_2506_04732_b200.tt import from_device, to_device

    recipe = wl.config(2)
    left, right, state0, forcing, _, _ = wl.march_problem(recipe)
    hl, hr, state = to_device(left), to_device(right), to_device(state0)
    cfg = SolverConfig(**recipe.solver)
    out = []
    for k in range(1, steps + 1):
        bc, src = (to_device(t) for t in forcing(k))
        _native.read_trace(1)
        a, rows = march_device(hl, hr, state, 1, [bc], [src], recipe.step_tol, cfg, store_stride=1)
        n = _native.read_trace(second)
        try:
            b, _ = march_device(hl, hr, state, 1, [bc], [src], recipe.step_tol, cfg, store_stride=1)
        finally:
            _native.read_trace(0)
        same = all(np.array_equal(x, y)
                   for x, y in zip(from_device(a[1]).cores, from_device(b[1]).cores))
        out.append((k, rows[0][4], n, same))
        state = a[1]
    return out


@pytest.mark.gpu
def test_march_steps_are_bit_reproducible(pk):
    # steps 2-4 cross the direct-solve size (GMRES, PCG) and use the pivoting
    # fallback; step 4 has the N = 1980 Gauss-Jordan solve
    for k, sweeps, reads, same in _march_steps(pk, 6, 3):
        assert reads > 20 and same, (k, sweeps, reads)


@pytest.mark.gpu
def test_replayed_reads_give_the_same_step_without_synchronising(pk):
    for k, sweeps, reads, same in _march_steps(pk, 3, 2):
        assert same, (k, sweeps, reads)


@pytest.mark.gpu
def test_replay_rejects_a_different_run(pk):
    from paper_2506_04732_b200 import _native, tt

    rng = np.random.default_rng(0)
    x = tt.TTVector([rng.standard_normal((1, 9, 3)), rng.standard_normal((3, 9, 1))])
    _native.read_trace(1)
    tt.tt_norm(x)
    assert _native.read_trace(2) >= 1
    try:
        tt.tt_norm(x)  # consumes the recorded read
        with pytest.raises(Exception):
            tt.tt_round(x, 1e-10)  # asks for reads that were never recorded
    finally:
        _native.read_trace(0)
