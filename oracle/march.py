"""CPU oracle: implicit step-and-truncate time marching (numpy).

TEST INFRASTRUCTURE ONLY (see oracle/tt_ops.py for the import rule).

Restates the step loop of ``pkg/src/ttss/time_integration.py:149-191``:

    rhs_k   = round(right @ state + bc_k + src_k, 0.01 * step_tol)
    state'  = solve(left, rhs_k, x0=state)
    state   = round(state', step_tol)

The reference samples the boundary term ``bc = (I - M) g`` and the source
``src = dt * M b`` once (time-independent data).  Manufactured solutions with
time-dependent data (BASELINE configs 2-3) supply them per step; passing the
same pair for every step is exactly the reference loop.
"""

from __future__ import annotations

import numpy as np

from .als_solver import Config, solve
from .tt_ops import compression_ratio, ranks_of, tt_add, tt_apply, tt_round


class StepFailure(RuntimeError):
    def __init__(self, step, message):
        super().__init__(f"step {step}: {message}")
        self.step = step


def step(left, right, state, bc, src, step_tol, solver_cfg, index=1):
    """One implicit step; returns (new state, solver report, rounded rhs)."""
    rhs = tt_apply(right, state)
    if bc is not None:
        rhs = tt_add(rhs, bc)
    if src is not None:
        rhs = tt_add(rhs, src)
    rhs = tt_round(rhs, 0.01 * step_tol)
    new, rep = solve(left, rhs, x0=state, cfg=solver_cfg)
    achieved = min(rep.residual_history)
    if not rep.converged and achieved > 50.0 * solver_cfg.residual_tol:
        raise StepFailure(index, f"inner solver stagnated at residual {achieved:.3e}")
    return tt_round(new, step_tol), rep, rhs


def march(left, right, state0, forcing, n_steps, step_tol=1e-8, solver_cfg=None):
    """Run ``n_steps`` steps.  ``forcing(k)`` returns (bc_k, src_k) for step k
    (1-based); returns (final state, per-step rows (step, max_rank,
    compression, last residual, sweeps))."""
    solver_cfg = solver_cfg or Config(residual_tol=1e-10)
    state = [np.array(c, dtype=float, copy=True) for c in state0]
    rows = []
    for k in range(1, n_steps + 1):
        bc, src = forcing(k)
        state, rep, _ = step(left, right, state, bc, src, step_tol, solver_cfg, index=k)
        rows.append((k, max(ranks_of(state)), compression_ratio(state),
                     rep.residual_history[-1], len(rep.residual_history)))
    return state, rows
