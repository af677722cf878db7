"""Swap the hot path of an unmodified ``ttss`` for the CUDA engine.

``install()`` rebinds, inside the reference's own modules, exactly the
functions the C ABI replaces (include/t2s2.h):

  ttss.tt_solver.solve          (tt_solver.py:445)   -> solver.solve     (t2s2_solve)
  ttss.tt_solver.residual       (tt_solver.py:80)    -> solver.residual  (t2s2_residual)
  ttss.time_integration._march  (time_integration.py:149) -> march._march (t2s2_march)
  ttss.time_integration.solve   (its import of tt_solver.solve, used by
                                 spacetime_solve, time_integration.py:216)

and, with ``arithmetic=True``, the train arithmetic of tensor_train
(tt_round, tt_op_round, tt_norm, tt_dot, tt_add, tt_apply, tt_full) in every
ttss module that imported it.  Public entry points
(``backward_euler_march``, ``crank_nicolson_march``, ``spacetime_solve``,
``solve``) are untouched and reach the engine through these names, so
reference callers need no change.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

from .reference import module as _ref

__all__ = ["install", "uninstall", "installed"]

_saved = []


def _swap(mod, name, new):
    _saved.append((mod, name, getattr(mod, name)))
    setattr(mod, name, new)


def installed():
    return bool(_saved)


def install(arithmetic=False):
    """Route the reference's hot path through libt2s2.so (idempotent)."""
    if _saved:
        return
    from . import march, solver, tt

    sol, ti = _ref("tt_solver"), _ref("time_integration")
    _swap(sol, "solve", solver.solve)
    _swap(sol, "residual", solver.residual)
    _swap(ti, "_march", march._march)
    _swap(ti, "solve", solver.solve)
    if arithmetic:
        names = ("tt_round", "tt_op_round", "tt_norm", "tt_dot", "tt_add", "tt_apply", "tt_full")
        for modname in ("tensor_train", "tt_solver", "time_integration", "operator_assembly"):
            mod = _ref(modname)
            for n in names:
                if hasattr(mod, n):
                    _swap(mod, n, getattr(tt, n))


def uninstall():
    while _saved:
        mod, name, old = _saved.pop()
        setattr(mod, name, old)
