"""Batched parameter sweep (BASELINE config 4): independent steady solves
sharded over ranks.

The solves share nothing, so the multi-GPU path has no data-path
collective: rank k of N takes solves k, k+N, k+2N, ... (round-robin keeps the
seeded eps draws — and with them the cost — spread evenly), runs them on its
own device, and the per-solve results are gathered once at the end
(``gather``; torch.distributed, any backend).  One process per GPU,
``LOCAL_RANK`` selects the device (see _native.context).  Solves run one
after another on a rank's GPU: several engine contexts on one GPU would put
spin-waiting cooperative kernels (Gauss-Jordan hand-offs, Krylov grid
barriers) of different solves side by side, and a kernel whose CTAs are only
partly resident next to another such kernel can wait forever.
"""

from __future__ import annotations

import time

__all__ = ["shard", "run_sweep", "gather"]


def shard(n_items, rank, world):
    """Indices owned by ``rank`` of ``world``."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_items, world))


def _default_solve(a, b, cfg_kwargs):
    from .solver import SolverConfig, solve

    x, rep = solve(a, b, cfg=SolverConfig(**cfg_kwargs))
    return x, rep


def run_sweep(recipes, rank=0, world=1, solve_fn=None, build_fn=None, overrides=None):
    """Solve this rank's share of ``recipes`` (workloads.SteadyRecipe).

    Returns {index: dict(x=cores, residuals, ranks, converged, stagnated,
    wall_s, exact_err)}.  ``solve_fn(a, b, cfg_kwargs)`` and
    ``build_fn(recipe)`` default to the device solver and this package's
    setup; tests substitute CPU stand-ins to exercise the sharding on gloo.
    """
    from . import workloads as wl

    solve_fn = solve_fn or _default_solve
    build_fn = build_fn or wl.steady_problem
    out = {}
    mine = shard(len(recipes), rank, world)

    def one(i):
        r = recipes[i]
        a, b, exact, _ = build_fn(r)
        cfg = dict(r.solver)
        cfg.update(overrides or {})
        t0 = time.perf_counter()
        x, rep = solve_fn(a, b, cfg)
        wall = time.perf_counter() - t0
        out[i] = dict(x=[c.copy() for c in x.cores], residuals=list(rep.residual_history),
                      ranks=list(rep.rank_history), converged=bool(rep.converged),
                      stagnated=bool(rep.stagnated), wall_s=wall, eps=r.eps)

    for i in mine:
        one(i)
    return out


def gather(local, world):
    """Merge every rank's {index: result} on all ranks (no-op for world=1)."""
    if world == 1:
        return dict(local)
    import torch.distributed as dist

    parts = [None] * world
    dist.all_gather_object(parts, local)
    merged = {}
    for p in parts:
        merged.update(p)
    return merged
