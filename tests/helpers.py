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


def bond_spectra(cores):
    """Singular values of every bond unfolding (left-to-right SVD sweep of
    the right-orthonormalised train, i.e. tt_round with tol=0)."""
    from oracle.tt_ops import right_orthonormalize

    work = right_orthonormalize(cores)
    out = []
    for l in range(len(work) - 1):
        r0, n, r1 = work[l].shape
        u, s, vt = np.linalg.svd(work[l].reshape(r0 * n, r1), full_matrices=False)
        out.append(s)
        work[l + 1] = np.einsum("ab,bnc->anc", s[:, None] * vt, work[l + 1])
    return out


def ranks_agree(a, b, tol=RANK_TOL, band=10.0):
    """Numerical bond ranks at ``tol`` (relative, tt_round's per-bond
    threshold) agree, except where a singular value of either train lies
    within a factor ``band`` of the threshold — that tail is the solver's
    noise floor, not structure.  Returns (ok, per-bond (rank_a, rank_b))."""
    d = len(a)
    sa, sb = bond_spectra(a), bond_spectra(b)
    detail, ok = [], True
    for l in range(d - 1):
        ta = tol * np.linalg.norm(sa[l]) / np.sqrt(d - 1)
        tb = tol * np.linalg.norm(sb[l]) / np.sqrt(d - 1)
        ka, kb = int(np.sum(sa[l] > ta)), int(np.sum(sb[l] > tb))
        if ka != kb:
            lo, hi = min(ka, kb), max(ka, kb)
            cand = np.concatenate([sa[l][lo:hi], sb[l][lo:hi]])
            thr = max(ta, tb)
            if not np.all((cand > thr / band) & (cand < thr * band)):
                ok = False
        detail.append((ka, kb))
    return ok, detail
