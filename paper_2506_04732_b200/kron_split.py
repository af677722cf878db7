"""One large operator apply split over GPUs by Kronecker-sum term
(north_star's second sharding; reference: operator_assembly.py:177-226).

The reference's spatial operators are sums over the d dimensions,

    A = sum_l  A_l,   A_l = diag(coef_l) (a0 x ... x block_l x ... x a0),

(`_banded_chain` packs the diffusion terms into one rank-2 chain,
`assemble_convection` adds the d convection terms one by one) and it merges
them by ``tt_op_round`` before anything is applied.  Applied to a train x of
rank r the merged operator of rank R costs 2 r^2 R^2 n^2 flops per core and
gives rank r R; the d separate terms cost d 2 r^2 R_l^2 n^2 and are
independent.  ``sharded_apply`` gives rank k of W the terms k, k + W, ...:

    y_k   = round( sum_{l in shard k} A_l x )        on GPU k (engine)
    y     = round( sum_k y_k )                       after ONE all-gather

A TT sum is a block concatenation of cores, not an element-wise reduction,
so the collective is an all-gather of the partial trains (ranks first, then
one padded payload: two collectives per apply, NCCL over NVLink on GPUs,
gloo in the CPU tests), and every rank ends with the same rounded result.
``sharded_residual`` is tt_solver.residual (tt_solver.py:555-560) on top of
it.  When it pays: DESIGN.md section 7 (the all-gather moves the partial
trains' r_k^2 n d doubles; the step's own operators are rank-1/rank-4 chains
applied in microseconds, so the march never calls this — it is for a single
large apply: high-rank states, unmerged operators with variable coefficients).

The arithmetic is a backend: the device engine (`tt.py`) by default; the
gloo tests inject a CPU stand-in, because the engine has no CPU fallback.
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_terms", "sharded_apply", "sharded_residual", "EngineBackend"]


def shard_terms(n_terms, rank, world):
    """Term indices owned by ``rank`` of ``world`` (round-robin)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_terms, world))


class EngineBackend:
    """TT arithmetic on this rank's GPU (the CUDA engine through tt.py)."""

    def apply(self, op, x):
        from . import tt

        return tt.tt_apply(op, x)

    def add(self, a, b, sa=1.0, sb=1.0):
        from . import tt

        return tt.tt_add(a if sa == 1.0 else tt.tt_scale(a, sa), b if sb == 1.0 else tt.tt_scale(b, sb))

    def round(self, x, tol):
        from . import tt

        return tt.tt_round(x, tol)

    def norm(self, x):
        from . import tt

        return tt.tt_norm(x)

    def vector(self, cores):
        from . import tt

        return tt.TTVector(cores)


def _pack(x):
    """(ranks int64[d+1], payload float64) of a vector train."""
    ranks = np.array([1] + [c.shape[2] for c in x.cores], dtype=np.int64)
    payload = np.concatenate([np.ascontiguousarray(c, dtype=np.float64).ravel() for c in x.cores])
    return ranks, payload


def _unpack(ranks, payload, modes):
    cores, off = [], 0
    for l, n in enumerate(modes):
        size = int(ranks[l]) * n * int(ranks[l + 1])
        cores.append(payload[off:off + size].reshape(int(ranks[l]), n, int(ranks[l + 1])).copy())
        off += size
    return cores


def _all_gather_trains(x, world, device):
    """Every rank's partial train on every rank: ranks first (fixed size),
    then the payloads padded to the largest one."""
    import torch
    import torch.distributed as dist

    modes = [c.shape[1] for c in x.cores]
    ranks, payload = _pack(x)
    t_ranks = torch.from_numpy(ranks).to(device)
    all_ranks = [torch.empty_like(t_ranks) for _ in range(world)]
    dist.all_gather(all_ranks, t_ranks)
    all_ranks = [r.cpu().numpy() for r in all_ranks]
    sizes = [int(sum(int(r[l]) * n * int(r[l + 1]) for l, n in enumerate(modes))) for r in all_ranks]
    buf = torch.zeros(max(sizes), dtype=torch.float64, device=device)
    buf[:payload.size] = torch.from_numpy(payload).to(device)
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    return [_unpack(all_ranks[k], bufs[k].cpu().numpy(), modes) for k in range(world)]


def sharded_apply(terms, x, tol, rank=0, world=1, backend=None, device="cpu"):
    """round(sum_l terms[l] x, tol), the terms split over ``world`` ranks.

    Every rank passes the same ``terms`` and ``x`` and gets the same result.
    The local partial sum is rounded at tol / world (so the partial
    truncations together stay below the final one), the gathered sum at tol.
    ``device``: where the collective's buffers live ("cuda:<k>" for NCCL).
    """
    backend = backend or EngineBackend()
    mine = shard_terms(len(terms), rank, world)
    part = None
    for l in mine:
        y = backend.apply(terms[l], x)
        part = y if part is None else backend.add(part, y)
    if world == 1:
        return backend.round(part, tol)
    if part is None:
        # more ranks than terms: contribute an explicit zero train of rank 1
        part = backend.vector([np.zeros((1, c.shape[1], 1)) for c in x.cores])
    else:
        part = backend.round(part, tol / world)
    total = None
    for cores in _all_gather_trains(part, world, device):
        y = backend.vector(cores)
        total = y if total is None else backend.add(total, y)
    return backend.round(total, tol)


def sharded_residual(terms, x, rhs, tol=1e-12, rank=0, world=1, backend=None, device="cpu"):
    """||sum_l terms[l] x - rhs|| / ||rhs|| (tt_solver.py:555-560) with the
    operator apply split by term."""
    backend = backend or EngineBackend()
    bnorm = backend.norm(rhs)
    if bnorm == 0.0:
        raise ValueError("rhs must be nonzero")
    ax = sharded_apply(terms, x, 0.01 * tol, rank, world, backend, device)
    diff = backend.round(backend.add(ax, rhs, 1.0, -1.0), 0.01 * tol)
    return backend.norm(diff) / bnorm
