"""Comparison helpers shared by the parity tests."""

import numpy as np

from oracle.tt_ops import ranks_of, tt_full

FULL_LIMIT = 2_000_000


def sample_entries(cores, idx):
    out = np.ones((idx.shape[0], 1))
    for l, c in enumerate(cores):
        out = np.einsum("ka,akb->kb", out, c[:, idx[:, l], :])
    return out[:, 0]


def rel_diff(a, b, npoints=100_000, seed=0):
    """Relative difference of two vector trains: on the full grid when it has
    at most FULL_LIMIT entries, else at ``npoints`` seeded sample points."""
    modes = [c.shape[1] for c in b]
    total = int(np.prod([float(m) for m in modes]))
    if total <= FULL_LIMIT:
        fa, fb = tt_full(a), tt_full(b)
    else:
        rng = np.random.default_rng(seed)
        idx = np.column_stack([rng.integers(0, m, npoints) for m in modes])
        fa, fb = sample_entries(a, idx), sample_entries(b, idx)
    return float(np.linalg.norm(fa - fb) / np.linalg.norm(fb))


def op_dense(op):
    from oracle.tt_ops import tt_op_full
    return tt_op_full(op)


def same_ranks(a, b):
    return ranks_of(a) == ranks_of(b)


# Parity protocol: two correct implementations of the
# alternating solver stop at different iterates whose residuals are both
# below residual_tol, and near-ties between the Galerkin and least-squares
# candidates (q_gal == q_old to rounding at repeated visits of the end
# cores) make the raw bond ranks path dependent.  We therefore compare
#   * values: ||x - x_ref|| / ||x_ref|| <= max(1e-10, 10 * (res + res_ref))
#     (error <= cond * residual; north_star's 1e-10 when both converge deeper)
#   * ranks: identical numerical ranks after rounding both at RANK_TOL.
RANK_TOL = 1e-10


def value_tol(res_a, res_b):
    return max(1e-10, 10.0 * (float(res_a) + float(res_b)))


def numerical_ranks(cores, tol=RANK_TOL):
    from oracle.tt_ops import tt_round
    return ranks_of(tt_round(cores, tol))
