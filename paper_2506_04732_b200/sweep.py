"""Batched parameter sweep (BASELINE config 4): independent steady solves
sharded over ranks.

The solves share nothing, so the multi-GPU path has no data-path
collective: rank k of N takes solves k, k+N, k+2N, ... (round-robin keeps the
seeded eps draws — and with them the cost — spread evenly), runs them on its
own device, and the per-solve results are gathered once at the end
(``gather``; torch.distributed, any backend).  One process per GPU,
``LOCAL_RANK`` selects the device (see _native.context).

Within a GPU, ``partitions=P`` runs P solves at a time, one host thread each,
on P disjoint SM partitions (green contexts, csrc/partition.cu): a single
solve leaves most SMs idle through its latency-bound stretches, and the
partitions keep the solves' spin-waiting cooperative kernels (Gauss-Jordan
hand-offs, Krylov grid barriers) on separate SMs — two such kernels sharing
SMs can each be partly resident and wait on each other forever, so plain
concurrent streams are not used.
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


def run_sweep(recipes, rank=0, world=1, solve_fn=None, build_fn=None, overrides=None,
              partitions=1):
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

    if partitions <= 1:
        for i in mine:
            one(i)
        return out
    import threading

    from . import _native

    _native.sm_partitions(partitions)
    queue = list(mine)
    lock = threading.Lock()
    errors = []

    def worker(t):
        _native.use_partition(t)
        while True:
            with lock:
                if not queue or errors:
                    return
                i = queue.pop(0)
            try:
                one(i)
            except Exception as exc:  # surface the first failure
                with lock:
                    errors.append(exc)
                return

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(partitions)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
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
