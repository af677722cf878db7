"""Rank-adaptive alternating TT solver on the CUDA engine.

Drop-in for ``ttss.tt_solver.solve`` / ``residual`` (tt_solver.py:80, 445):
same arguments, the reference's own ``SolverConfig`` and ``SolveReport``
dataclasses and exceptions; the sweeps run in ``libt2s2.so``
(csrc/als.cu).  Only the default initial guess's random fallback is drawn
on the host, with numpy's generator seeded exactly like the reference
(tt_solver.py:425-432), because it is input data, not computation.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import ShapeError
from .reference import module as _ref
from .tt import from_device, to_device, tt_norm, tt_rank_one, tt_round, tt_scale

_rsol = _ref("tt_solver")
SolverConfig = _rsol.SolverConfig
SolveReport = _rsol.SolveReport

__all__ = ["SolverConfig", "SolveReport", "solve", "residual", "solve_device", "config_to_c",
           "report_from_c"]

_LOCAL = {"auto": 0, "direct": 1, "iterative": 2}


def config_to_c(cfg):
    """t2s2_solver_config of a SolverConfig (tt_solver.py:39-59).  The
    engine keeps at most T2S2_MAX_SWEEPS entries of history per solve."""
    if cfg.max_sweeps > _native.MAX_SWEEPS:
        raise ValueError(f"max_sweeps > {_native.MAX_SWEEPS} is not supported by the engine's "
                         "report buffers")
    return _native.SolverConfigC(
        max_sweeps=int(cfg.max_sweeps), residual_tol=float(cfg.residual_tol),
        rounding_tol=float(cfg.rounding_tol), enrichment_rank=int(cfg.enrichment_rank),
        max_rank=int(cfg.max_rank), local_solver=_LOCAL[cfg.local_solver],
        local_direct_size=int(cfg.local_direct_size),
        inner_tol_factor=float(cfg.inner_tol_factor),
        stagnation_window=int(cfg.stagnation_window),
        stagnation_drop=float(cfg.stagnation_drop))


def report_from_c(r):
    n = r.n_sweeps
    return SolveReport(residual_history=[float(r.residuals[i]) for i in range(n)],
                       rank_history=[int(r.ranks[i]) for i in range(n)],
                       compression_history=[float(r.compression[i]) for i in range(n)],
                       wall_time=float(r.wall_time), converged=bool(r.converged),
                       stagnated=bool(r.stagnated))


def _default_initial_guess(rhs, cfg, rng):
    """tt_solver.py:425-432 with the rounding and norms on the device."""
    x0 = tt_round(rhs, 0.5, max_rank=1)
    if tt_norm(x0) < 1e-13 * max(tt_norm(rhs), 1.0):
        x0 = tt_rank_one([rng.standard_normal(n) for n in rhs.mode_sizes])
        x0 = tt_scale(x0, tt_norm(rhs) / max(tt_norm(x0), 1e-300))
    return x0


def solve_device(a_h, rhs_h, x0_h, cfg):
    """Solve with device-resident handles; returns (DeviceTrain, SolveReport)."""
    rep = _native.SolveReportC()
    out = _native._P()
    ccfg = config_to_c(cfg)
    _native.check(_native.lib().t2s2_solve(_native.context(), a_h.handle, rhs_h.handle,
                                           x0_h.handle, ctypes.byref(ccfg), ctypes.byref(out),
                                           ctypes.byref(rep)))
    return _native.DeviceTrain(out), report_from_c(rep)


def solve(a, rhs, x0=None, cfg=None):
    """Solve A x = rhs in train format; returns (best iterate, SolveReport)
    (tt_solver.py:445)."""
    cfg = cfg or SolverConfig()
    if a.col_sizes != rhs.mode_sizes or a.row_sizes != rhs.mode_sizes:
        raise ShapeError("operator and right-hand side shapes do not match")
    if tt_norm(rhs) == 0.0:
        raise ValueError("rhs must be nonzero")
    rng = np.random.default_rng(cfg.seed)
    x = x0 if x0 is not None else _default_initial_guess(rhs, cfg, rng)
    if x.mode_sizes != rhs.mode_sizes:
        raise ShapeError("initial guess has wrong mode sizes")
    ha, hb, hx = to_device(a), to_device(rhs), to_device(x)
    try:
        hsol, rep = solve_device(ha, hb, hx, cfg)
        try:
            return from_device(hsol), rep
        finally:
            hsol.free()
    finally:
        ha.free()
        hb.free()
        hx.free()


def residual(a, x, rhs, tol=1e-8):
    """Relative residual ||A x - rhs|| / ||rhs|| (tt_solver.py:80)."""
    ha, hx, hb = to_device(a), to_device(x), to_device(rhs)
    try:
        out = _native._D()
        _native.check(_native.lib().t2s2_residual(_native.context(), ha.handle, hx.handle,
                                                  hb.handle, float(tol), ctypes.byref(out)))
        return float(out.value)
    finally:
        ha.free()
        hx.free()
        hb.free()
