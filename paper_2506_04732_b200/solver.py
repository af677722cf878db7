"""Rank-adaptive alternating TT solver — host API over the CUDA engine.

Same names, arguments and error behaviour as the reference's
``pkg/src/ttss/tt_solver.py``; the sweeps run in ``libt2s2.so``
(csrc/als.cu).  Only the default initial guess's random fallback is drawn
on the host, with numpy's generator seeded exactly like the reference
(tt_solver.py:425-432), because it is input data, not computation.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ShapeError
from .tt import TTVector, from_device, to_device, tt_norm, tt_rank_one, tt_round, tt_scale

__all__ = ["SolverConfig", "SolveReport", "solve", "residual", "solve_device"]

_LOCAL = {"auto": 0, "direct": 1, "iterative": 2}


@dataclass
class SolverConfig:
    max_sweeps: int = 40
    residual_tol: float = 1e-8
    rounding_tol: float = 1e-10
    enrichment_rank: int = 2
    max_rank: int = 64
    local_solver: str = "auto"  # auto | direct | iterative
    local_direct_size: int = 2000
    inner_tol_factor: float = 0.02
    seed: int = 0
    stagnation_window: int = 5
    stagnation_drop: float = 0.01

    def __post_init__(self):
        if self.residual_tol <= 0 or self.rounding_tol <= 0:
            raise ValueError("tolerances must be positive")
        if self.max_rank < 1:
            raise ValueError("max_rank must be at least 1")
        if self.local_solver not in _LOCAL:
            raise ValueError("local_solver must be auto, direct or iterative")

    def to_c(self):
        return _native.SolverConfigC(
            max_sweeps=int(self.max_sweeps), residual_tol=float(self.residual_tol),
            rounding_tol=float(self.rounding_tol), enrichment_rank=int(self.enrichment_rank),
            max_rank=int(self.max_rank), local_solver=_LOCAL[self.local_solver],
            local_direct_size=int(self.local_direct_size),
            inner_tol_factor=float(self.inner_tol_factor),
            stagnation_window=int(self.stagnation_window),
            stagnation_drop=float(self.stagnation_drop))


@dataclass
class SolveReport:
    residual_history: list = field(default_factory=list)
    rank_history: list = field(default_factory=list)
    compression_history: list = field(default_factory=list)
    wall_time: float = 0.0
    converged: bool = False
    stagnated: bool = False

    def to_dict(self):
        return {
            "residuals": list(map(float, self.residual_history)),
            "ranks": list(map(int, self.rank_history)),
            "compression": list(map(float, self.compression_history)),
            "wall_time_s": float(self.wall_time),
            "converged": bool(self.converged),
        }

    @classmethod
    def from_c(cls, r):
        n = r.n_sweeps
        return cls(residual_history=[float(r.residuals[i]) for i in range(n)],
                   rank_history=[int(r.ranks[i]) for i in range(n)],
                   compression_history=[float(r.compression[i]) for i in range(n)],
                   wall_time=float(r.wall_time), converged=bool(r.converged),
                   stagnated=bool(r.stagnated))


def _default_initial_guess(rhs, cfg, rng):
    x0 = tt_round(rhs, 0.5, max_rank=1)
    if tt_norm(x0) < 1e-13 * max(tt_norm(rhs), 1.0):
        x0 = tt_rank_one([rng.standard_normal(n) for n in rhs.mode_sizes])
        x0 = tt_scale(x0, tt_norm(rhs) / max(tt_norm(x0), 1e-300))
    return x0


def solve_device(a_h, rhs_h, x0_h, cfg):
    """Solve with device-resident handles; returns (DeviceTrain, SolveReport)."""
    rep = _native.SolveReportC()
    out = _native._P()
    ccfg = cfg.to_c()
    _native.check(_native.lib().t2s2_solve(_native.context(), a_h.handle, rhs_h.handle,
                                           x0_h.handle, ctypes.byref(ccfg), ctypes.byref(out),
                                           ctypes.byref(rep)))
    return _native.DeviceTrain(out), SolveReport.from_c(rep)


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
