"""CPU oracle: the rank-adaptive alternating TT linear solver (numpy/scipy).

TEST INFRASTRUCTURE ONLY (see oracle/tt_ops.py for the import rule).

Restates ``pkg/src/ttss/tt_solver.py`` of the reference: one-site alternating
sweeps; per core a guarded choice between the Galerkin-projected solve and
the local least-squares solve through A^T A interfaces, scored by the exact
quadratic ||Ax-b||^2; SVD split of the solved core with residual-gradient
enrichment; Gram-form residual measurement with an exact fallback.

Interface index names (as in the reference):
  pa (x, a, z)        <x| A |x>           tt_solver.py:98-107
  pn (x, a1, a2, z)   <x| A^T A |x>        tt_solver.py:110-124
  pg (x, a, b)        <x| A^T |b>          tt_solver.py:127-139
  pb (x, b)           <x| b>               tt_solver.py:142-151
x is the test-side bond, z the trial-side bond; a are operator bonds and b
right-hand-side bonds.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse.linalg as spla

from .tt_ops import (
    compression_ratio,
    modes_of,
    rank_one,
    ranks_of,
    right_orthonormalize,
    tail_keep,
    tt_add,
    tt_apply,
    tt_norm,
    tt_round,
    tt_scale,
)


@dataclass
class Config:
    """Mirror of SolverConfig (tt_solver.py:39-59)."""

    max_sweeps: int = 40
    residual_tol: float = 1e-8
    rounding_tol: float = 1e-10
    enrichment_rank: int = 2
    max_rank: int = 64
    local_solver: str = "auto"
    local_direct_size: int = 2000
    inner_tol_factor: float = 0.02
    seed: int = 0
    stagnation_window: int = 5
    stagnation_drop: float = 0.01


@dataclass
class Report:
    """Mirror of SolveReport (tt_solver.py:62-76)."""

    residual_history: list = field(default_factory=list)
    rank_history: list = field(default_factory=list)
    compression_history: list = field(default_factory=list)
    wall_time: float = 0.0
    converged: bool = False
    stagnated: bool = False
    # oracle-only bookkeeping: which candidate each core visit kept
    choices: list = field(default_factory=list)


# -- interface recurrences -----------------------------------------------------
# Written as tensordot chains (BLAS-backed) so the oracle's CPU cost is
# representative of the reference when it serves as the CPU baseline.

td = np.tensordot


def step_a_left(phi, xc, ac):
    t = td(phi, xc, ([0], [0]))              # (a, z, m, X)
    t = td(t, ac, ([0, 2], [0, 1]))          # (z, X, n, A)
    return td(t, xc, ([0, 2], [0, 1]))       # (X, A, Z)


def step_a_right(phi, xc, ac):
    t = td(xc, phi, ([2], [0]))              # (x, m, A, Z)
    t = td(ac, t, ([1, 3], [1, 2]))          # (a, n, x, Z)
    return td(t, xc, ([1, 3], [1, 2])).transpose(1, 0, 2)


def step_n_left(phi, xc, ac):
    t = td(phi, xc, ([0], [0]))              # (p, q, z, i, X)
    t = td(t, ac, ([0, 3], [0, 2]))          # (q, z, X, k, P)
    t = td(t, ac, ([0, 3], [0, 1]))          # (z, X, P, j, Q)
    return td(t, xc, ([0, 3], [0, 1]))       # (X, P, Q, Z)


def step_n_right(phi, xc, ac):
    t = td(xc, phi, ([2], [0]))              # (x, i, P, Q, Z)
    t = td(ac, t, ([2, 3], [1, 2]))          # (p, k, x, Q, Z)
    t = td(ac, t, ([1, 3], [1, 3]))          # (q, j, p, x, Z)
    t = td(t, xc, ([1, 4], [1, 2]))          # (q, p, x, z)
    return t.transpose(2, 1, 0, 3)


def step_g_left(phi, xc, ac, bc):
    t = td(phi, xc, ([0], [0]))              # (a, b, n, X)
    t = td(t, ac, ([0, 2], [0, 2]))          # (b, X, k, A)
    return td(t, bc, ([0, 2], [0, 1]))       # (X, A, B)


def step_g_right(phi, xc, ac, bc):
    t = td(xc, phi, ([2], [0]))              # (x, n, A, B)
    t = td(ac, t, ([2, 3], [1, 2]))          # (a, k, x, B)
    return td(t, bc, ([1, 3], [1, 2])).transpose(1, 0, 2)


def step_b_left(phi, xc, bc):
    return td(td(phi, xc, ([0], [0])), bc, ([0, 1], [0, 1]))


def step_b_right(phi, xc, bc):
    return td(td(xc, phi, ([2], [0])), bc, ([1, 2], [1, 2]))


# -- local systems (tt_solver.py:155-246) ----------------------------------------


def galerkin_rhs(pbl, bc, pbr):
    return td(td(pbl, bc, ([1], [0])), pbr, ([2], [1]))


def galerkin_apply(pal, ac, par, u):
    t = td(pal, u, ([2], [0]))               # (x, a, n, w)
    t = td(t, ac, ([1, 2], [0, 2]))          # (x, w, m, b)
    return td(t, par, ([1, 3], [2, 1]))      # (x, m, y)


def galerkin_matrix(pal, ac, par):
    """Rows (x, m, y), columns (X, n, Y): sum_ab L_a (x) A_ab (x) R_b."""
    size = pal.shape[0] * ac.shape[1] * par.shape[0]
    out = np.zeros((size, size))
    for a in range(ac.shape[0]):
        la = pal[:, a, :]
        for b in range(ac.shape[3]):
            out += np.kron(np.kron(la, ac[a, :, :, b]), par[:, b, :])
    return out


def normal_rhs(pgl, ac, bc, pgr):
    t = td(pgl, bc, ([2], [0]))              # (x, a, k, B)
    t = td(t, ac, ([1, 2], [0, 1]))          # (x, B, m, A)
    return td(t, pgr, ([1, 3], [2, 1]))      # (x, m, y)


def normal_apply(pnl, ac, pnr, u):
    t = td(pnl, u, ([3], [0]))               # (x, p, q, n, w)
    t = td(t, ac, ([2, 3], [0, 2]))          # (x, p, w, k, Q)
    t = td(t, ac, ([1, 3], [0, 1]))          # (x, w, Q, m, P)
    return td(t, pnr, ([1, 4, 2], [3, 1, 2]))  # (x, m, y)


def normal_matrix(pnl, ac, pnr):
    gram = td(ac, ac, ([1], [1]))            # (a, m, P, b, n, Q)
    t = td(pnl, gram, ([1, 2], [0, 3]))      # (x, z, m, P, n, Q)
    t = td(t, pnr, ([3, 5], [1, 2]))         # (x, z, m, n, y, w)
    size = pnl.shape[0] * ac.shape[1] * pnr.shape[0]
    return t.transpose(0, 2, 4, 1, 3, 5).reshape(size, size)


def normal_diagonal(pnl, ac, pnr):
    gram = np.einsum("akmP,bkmQ->abmPQ", ac, ac)
    left = np.einsum("xabx->xab", pnl)
    right = np.einsum("yPQy->yPQ", pnr)
    t = td(left, gram, ([1, 2], [0, 1]))     # (x, m, P, Q)
    return td(t, right, ([2, 3], [1, 2])).ravel()


# -- core split with enrichment (tt_solver.py:261-302) -----------------------------


def split_forward(u, grad, tol, enrich, max_rank, d):
    r0, n, _ = u.shape
    uu, ss, vv = np.linalg.svd(u.reshape(r0 * n, -1), full_matrices=False)
    delta = tol * np.linalg.norm(ss) / np.sqrt(max(d - 1, 1))
    keep = min(tail_keep(ss, delta), max_rank)
    basis = uu[:, :keep]
    carry = ss[:keep, None] * vv[:keep]
    extra = 0
    if enrich > 0 and keep < max_rank and grad is not None:
        z = grad.reshape(r0 * n, -1)
        z = z - basis @ (basis.T @ z)
        zu, zs, _ = np.linalg.svd(z, full_matrices=False)
        lead = zs[0] if zs.size else 0.0
        nz = int(np.count_nonzero(zs > 1e-14 * max(lead, 1e-300)))
        extra = min(enrich, max_rank - keep, nz)
        if extra > 0:
            basis = np.hstack([basis, zu[:, :extra]])
    return basis.reshape(r0, n, keep + extra), carry, extra


def split_backward(u, grad, tol, enrich, max_rank, d):
    r0, n, r1 = u.shape
    uu, ss, vv = np.linalg.svd(u.reshape(r0, n * r1), full_matrices=False)
    delta = tol * np.linalg.norm(ss) / np.sqrt(max(d - 1, 1))
    keep = min(tail_keep(ss, delta), max_rank)
    basis = vv[:keep]
    carry = uu[:, :keep] * ss[None, :keep]
    extra = 0
    if enrich > 0 and keep < max_rank and grad is not None:
        z = grad.reshape(-1, n * r1)
        z = z - (z @ basis.T) @ basis
        _, zs, zv = np.linalg.svd(z, full_matrices=False)
        lead = zs[0] if zs.size else 0.0
        nz = int(np.count_nonzero(zs > 1e-14 * max(lead, 1e-300)))
        extra = min(enrich, max_rank - keep, nz)
        if extra > 0:
            basis = np.vstack([basis, zv[:extra]])
    return basis.reshape(keep + extra, n, r1), carry, extra


# -- residual (tt_solver.py:305-329) -----------------------------------------------


def measure_residual(a, x, rhs, bnorm):
    phi = np.ones((1, 1, 1, 1))
    for xc, ac in zip(x, a):
        phi = step_n_left(phi, xc, ac)
    axax = float(phi.ravel()[0])
    psi = np.ones((1, 1, 1))
    for xc, ac, bc in zip(x, a, rhs):
        psi = step_g_left(psi, xc, ac, bc)
    axb = float(psi.ravel()[0])
    est_sq = axax - 2.0 * axb + bnorm * bnorm
    est = np.sqrt(max(est_sq, 0.0)) / bnorm
    if est_sq <= 0 or est < 1e-6:
        diff = tt_add(tt_apply(a, x), tt_scale(rhs, -1.0))
        return tt_norm(diff) / bnorm
    return est


def residual(a, x, rhs, tol=1e-8):
    """Relative residual with a rounded difference (tt_solver.py:80-92)."""
    bnorm = tt_norm(rhs)
    if bnorm == 0.0:
        raise ValueError("rhs must be nonzero")
    diff = tt_round(tt_add(tt_apply(a, x), tt_scale(rhs, -1.0)), 0.01 * tol)
    return tt_norm(diff) / bnorm


# -- guarded core update (tt_solver.py:337-422) --------------------------------------


class _Sweep:
    def __init__(self, a, rhs, cfg, d):
        self.a, self.rhs, self.cfg, self.d = a, rhs, cfg, d
        self.gal_rejects = 0
        self.gal_cap = 2 * d

    def update(self, l, cores, pal, par, pnl, pnr, pgl, pgr, pbl, pbr, current_res):
        cfg = self.cfg
        ac, bc = self.a[l], self.rhs[l]
        u_old = cores[l]
        shape, size = u_old.shape, u_old.size

        c_gal = galerkin_rhs(pbl, bc, pbr)
        c_ls = normal_rhs(pgl, ac, bc, pgr)

        def nmv(u):
            return normal_apply(pnl, ac, pnr, u)

        def score(u):
            return float(np.vdot(u, nmv(u)) - 2.0 * np.vdot(c_ls, u))

        q_old = score(u_old)
        direct = cfg.local_solver == "direct" or (
            cfg.local_solver == "auto" and size <= cfg.local_direct_size
        )
        try_gal = self.gal_rejects < self.gal_cap
        inner_rtol = max(cfg.inner_tol_factor * current_res, 1e-12)

        u_gal = None
        if try_gal:
            if direct:
                mat = galerkin_matrix(pal, ac, par)
                try:
                    u_gal = np.linalg.solve(mat, c_gal.ravel()).reshape(shape)
                except np.linalg.LinAlgError:
                    u_gal = np.linalg.lstsq(mat, c_gal.ravel(), rcond=None)[0].reshape(shape)
            else:
                op = spla.LinearOperator(
                    (size, size),
                    matvec=lambda v: galerkin_apply(pal, ac, par, v.reshape(shape)).ravel(),
                )
                vec, _ = spla.gmres(op, c_gal.ravel(), x0=u_old.ravel(), rtol=inner_rtol,
                                    atol=0.0, restart=40, maxiter=10)
                u_gal = vec.reshape(shape)
        if u_gal is not None and not np.all(np.isfinite(u_gal)):
            u_gal = None

        best, best_q, choice = u_old, q_old, "keep"
        if u_gal is not None:
            q_gal = score(u_gal)
            if q_gal <= best_q:
                best, best_q, choice = u_gal, q_gal, "galerkin"
                self.gal_rejects = 0
            elif try_gal:
                self.gal_rejects += 1

        if choice == "keep":
            if direct:
                mat = normal_matrix(pnl, ac, pnr)
                try:
                    u_ls = np.linalg.solve(mat, c_ls.ravel()).reshape(shape)
                except np.linalg.LinAlgError:
                    u_ls = np.linalg.lstsq(mat, c_ls.ravel(), rcond=None)[0].reshape(shape)
            else:
                op = spla.LinearOperator((size, size), matvec=lambda v: nmv(v.reshape(shape)).ravel())
                dg = normal_diagonal(pnl, ac, pnr)
                dg = np.where(np.abs(dg) > 1e-300, dg, 1.0)
                pre = spla.LinearOperator((size, size), matvec=lambda v: v / dg)
                vec, _ = spla.cg(op, c_ls.ravel(), x0=u_old.ravel(), rtol=inner_rtol,
                                 atol=0.0, maxiter=250, M=pre)
                u_ls = vec.reshape(shape)
            if np.all(np.isfinite(u_ls)):
                q_ls = score(u_ls)
                if q_ls <= best_q:
                    best, best_q, choice = u_ls, q_ls, "lsq"
        grad = nmv(best) - c_ls
        return best, grad, choice


def initial_guess(rhs, cfg, rng):
    """tt_solver.py:425-432: rank-1 compression of rhs, or a random rank-1."""
    x0 = tt_round(rhs, 0.5, max_rank=1)
    if tt_norm(x0) < 1e-13 * max(tt_norm(rhs), 1.0):
        x0 = rank_one([rng.standard_normal(n) for n in modes_of(rhs)])
        x0 = tt_scale(x0, tt_norm(rhs) / max(tt_norm(x0), 1e-300))
    return x0


def solve(a, rhs, x0=None, cfg=None):
    """Alternating solve of A x = rhs (tt_solver.py:445-552).

    ``a`` is a list of operator cores, ``rhs``/``x0`` lists of vector cores.
    Returns (best iterate cores, Report).
    """
    cfg = cfg or Config()
    bnorm = tt_norm(rhs)
    if bnorm == 0.0:
        raise ValueError("rhs must be nonzero")
    rng = np.random.default_rng(cfg.seed)
    t0 = time.perf_counter()
    x = x0 if x0 is not None else initial_guess(rhs, cfg, rng)
    cores = tt_round(x, cfg.rounding_tol, max_rank=cfg.max_rank)
    d = len(cores)
    rep = Report()
    best_res, best_cores = np.inf, [c.copy() for c in cores]
    current_res = 1.0
    sw = _Sweep(a, rhs, cfg, d)
    one3, one4, one2 = np.ones((1, 1, 1)), np.ones((1, 1, 1, 1)), np.ones((1, 1))

    for _ in range(cfg.max_sweeps):
        cores = right_orthonormalize(cores)
        pa = [None] * (d + 1); pn = [None] * (d + 1)
        pg = [None] * (d + 1); pb = [None] * (d + 1)
        pa[d], pn[d], pg[d], pb[d] = one3, one4, one3, one2
        for l in range(d - 1, 0, -1):
            pa[l] = step_a_right(pa[l + 1], cores[l], a[l])
            pn[l] = step_n_right(pn[l + 1], cores[l], a[l])
            pg[l] = step_g_right(pg[l + 1], cores[l], a[l], rhs[l])
            pb[l] = step_b_right(pb[l + 1], cores[l], rhs[l])
        la = [None] * (d + 1); ln = [None] * (d + 1)
        lg = [None] * (d + 1); lb = [None] * (d + 1)
        la[0], ln[0], lg[0], lb[0] = one3, one4, one3, one2

        def visit(l):
            u, grad, choice = sw.update(l, cores, la[l], pa[l + 1], ln[l], pn[l + 1],
                                        lg[l], pg[l + 1], lb[l], pb[l + 1], current_res)
            rep.choices.append(choice)
            return u, grad

        for l in range(d):
            u, grad = visit(l)
            if l == d - 1:
                cores[l] = u
                break
            core, carry, k = split_forward(u, grad, cfg.rounding_tol, cfg.enrichment_rank,
                                           cfg.max_rank, d)
            cores[l] = core
            nxt = np.einsum("ab,bnc->anc", carry, cores[l + 1])
            if k > 0:
                nxt = np.concatenate([nxt, np.zeros((k,) + nxt.shape[1:])], axis=0)
            cores[l + 1] = nxt
            la[l + 1] = step_a_left(la[l], cores[l], a[l])
            ln[l + 1] = step_n_left(ln[l], cores[l], a[l])
            lg[l + 1] = step_g_left(lg[l], cores[l], a[l], rhs[l])
            lb[l + 1] = step_b_left(lb[l], cores[l], rhs[l])

        for l in range(d - 1, -1, -1):
            u, grad = visit(l)
            if l == 0:
                cores[l] = u
                break
            core, carry, k = split_backward(u, grad, cfg.rounding_tol, cfg.enrichment_rank,
                                            cfg.max_rank, d)
            cores[l] = core
            prv = np.einsum("anb,bc->anc", cores[l - 1], carry)
            if k > 0:
                prv = np.concatenate([prv, np.zeros(prv.shape[:2] + (k,))], axis=2)
            cores[l - 1] = prv
            pa[l] = step_a_right(pa[l + 1], cores[l], a[l])
            pn[l] = step_n_right(pn[l + 1], cores[l], a[l])
            pg[l] = step_g_right(pg[l + 1], cores[l], a[l], rhs[l])
            pb[l] = step_b_right(pb[l + 1], cores[l], rhs[l])

        current_res = measure_residual(a, cores, rhs, bnorm)
        rep.residual_history.append(current_res)
        rep.rank_history.append(max(ranks_of(cores)))
        rep.compression_history.append(compression_ratio(cores))
        if current_res < best_res:
            best_res, best_cores = current_res, [c.copy() for c in cores]
        if current_res <= cfg.residual_tol:
            rep.converged = True
            break
        w = cfg.stagnation_window
        hist = rep.residual_history
        if len(hist) > w:
            past, now = min(hist[:-w]), min(hist)
            if past <= 0 or (past - now) / max(past, 1e-300) < cfg.stagnation_drop:
                rep.stagnated = True
                break
    rep.wall_time = time.perf_counter() - t0
    return best_cores, rep
