"""Generate tests/golden/*.npz by running the REFERENCE package.

Run here (where /root/reference is mounted read-only):

    python tools/make_golden.py

It imports ``ttss`` from /root/reference/pkg/src, builds the problems with
the reference's own functions and stores inputs and outputs.  The fixtures
pin (a) this repo's host setup (grids, assembled operators) and (b) the CPU
oracle; the GPU parity tests then compare the CUDA path with both.  Nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from golden_io import put_train  # noqa: E402

import ttss  # noqa: E402,F401
from ttss import spectral1d as rs  # noqa: E402
from ttss import superconsistency as rsc  # noqa: E402
from ttss import tensor_train as rtt  # noqa: E402
from ttss import tt_solver as rsol  # noqa: E402
from ttss import time_integration as rti  # noqa: E402
from ttss.coefficients import constant_coefficient  # noqa: E402
from ttss.operator_assembly import (  # noqa: E402
    ProblemSpec,
    assemble_opset,
    impose_dirichlet,
    rep_axes,
    row_axes,
)

from paper_2506_04732_b200 import workloads as wl  # noqa: E402  (pure-numpy recipes)

OUT = os.path.join(ROOT, "tests", "golden")


def save(name, store):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **store)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def cfg_dict(cfg):
    return {f"cfg_{k}": np.array(v) for k, v in cfg.__dict__.items()}


def grids():
    cases = [(4, 1.0, 0.0), (7, 0.02, 1.0), (7, 1e-12, 1.0), (16, 1e-6, 1.0), (16, 1e-3, -0.5),
             (32, 1e-3, 0.3), (64, 1e-12, 1.0), (65, 1e-2, 2.0)]
    st = {"cases": np.array(cases)}
    for i, (n, e, b) in enumerate(cases):
        g = rsc.sc_grid(n, e, b)
        st[f"{i}_gll"] = rs.gll_nodes(n)
        st[f"{i}_gauss"] = rs.gauss_nodes(n)
        st[f"{i}_bary"] = g.base.bary_w
        st[f"{i}_coll"] = g.coll_nodes
        st[f"{i}_d1"] = g.base.d1
        st[f"{i}_d2"] = g.base.d2
        for k in ("a0", "a1", "a2"):
            st[f"{i}_{k}"] = getattr(g, k)
    save("setup_grids.npz", st)


def spec_of(dims, degree, eps, beta, rho, rhs=1.0, stab="superconsistent"):
    return ProblemSpec(dims=dims, degrees=[degree] * dims,
                       epsilon=constant_coefficient(eps, dims),
                       beta=[constant_coefficient(b, dims) for b in beta],
                       rho=constant_coefficient(rho, dims), rhs=constant_coefficient(rhs, dims),
                       stabilization=stab)


OP_CASES = [
    ("d2", 2, 6, 0.05, [1.0, 3.0], 0.1, "superconsistent"),
    ("d3", 3, 4, 1e-3, [1.0, -0.5, 0.25], 0.0, "superconsistent"),
    ("d2p", 2, 5, 0.2, [0.0, 1.0], 0.3, "plain"),
]


def operators():
    st = {}
    for tag, dims, deg, eps, beta, rho, stab in OP_CASES:
        spec = spec_of(dims, deg, eps, beta, rho, stab=stab)
        op = assemble_opset(spec)
        for k in ("diffusion", "convection", "reaction", "mask_interior", "spatial"):
            put_train(st, f"{tag}_{k}", getattr(op, k).cores)
        a, b = impose_dirichlet(op, spec)
        put_train(st, f"{tag}_rhs", b.cores)
        for scheme in ("backward_euler", "crank_nicolson"):
            mc = rti.MarchConfig(dt=0.01, t_end=0.05, scheme=scheme)
            left, right, _, _ = rti._march_operators(op, spec, mc)
            put_train(st, f"{tag}_{scheme}_left", left.cores)
            put_train(st, f"{tag}_{scheme}_right", right.cores)
    save("setup_ops.npz", st)


def rounding():
    rng = np.random.default_rng(11)
    st = {}
    cases = []
    i = 0
    for modes, rank in [((5, 6, 4), 3), ((4, 4, 4, 4, 4), 5), ((7, 3), 4), ((9,), 1),
                        ((6, 5, 6, 5), 6)]:
        base = rtt.tt_random(modes, rank, rng, norm=2.0)
        # inflate: v + v + small perturbation -> exact low-rank structure at tight tol
        pert = rtt.tt_scale(rtt.tt_random(modes, 2, rng, norm=1.0), 1e-9)
        v = rtt.tt_add(rtt.tt_add(base, base), pert)
        for tol, cap in [(0.0, None), (1e-12, None), (1e-6, None), (1e-2, None), (0.5, 1),
                         (1e-12, 2)]:
            r = rtt.tt_round(v, tol, max_rank=cap)
            put_train(st, f"in{i}", v.cores)
            put_train(st, f"out{i}", r.cores)
            st[f"tol{i}"] = np.array(tol)
            st[f"cap{i}"] = np.array(cap or 0)
            st[f"norm{i}"] = np.array(rtt.tt_norm(v))
            cases.append(i)
            i += 1
    st["count"] = np.array(i)
    save("round.npz", st)


def pde_system(dims, degree, eps=0.05, beta=1.0, rho=0.1):
    spec = spec_of(dims, degree, eps, [beta] * dims, rho)
    return impose_dirichlet(assemble_opset(spec), spec)


SOLVE_CASES = [
    # tag, (dims, degree, eps, beta, rho), cfg kwargs
    ("s1", (1, 9, 0.05, 1.0, 0.1), dict(residual_tol=1e-10, max_rank=40)),
    ("s2", (2, 8, 0.05, 1.0, 0.1), dict(residual_tol=1e-10, max_rank=40)),
    ("s3", (3, 6, 0.05, 1.0, 0.1), dict(residual_tol=1e-10, max_rank=40)),
    ("s4", (2, 8, 1e-3, 1.0, 0.1), dict(residual_tol=1e-12, max_sweeps=10, max_rank=24)),
    ("s5", (3, 6, 0.05, 1.0, 0.1), dict(residual_tol=1e-14, max_sweeps=7, max_rank=5)),
    ("s6", (2, 16, 1e-7, 1.0, 0.0), dict(residual_tol=1e-12, max_rank=2, max_sweeps=30,
                                         enrichment_rank=0)),
    ("s7", (2, 7, 1e-3, 1.0, 0.1), dict(residual_tol=1e-11, seed=42, max_sweeps=8)),
    ("s8", "singular", dict(residual_tol=1e-10, max_sweeps=8)),
]


def singular_system():
    """Diagonal operator with a zero slice: every local solve hits numpy's
    LinAlgError and the reference falls back to lstsq (tt_solver.py:362)."""
    rng = np.random.default_rng(9)
    f = [rng.uniform(1, 2, n) for n in (5, 4, 6)]
    f[0][2] = 0.0
    a = rtt.tt_diag_operator(rtt.tt_from_separable([(1.0, f)]))
    return a, rtt.tt_random((5, 4, 6), 2, rng, norm=1.0)


def solves():
    st = {}
    for tag, sysargs, kw in SOLVE_CASES:
        a, b = singular_system() if sysargs == "singular" else pde_system(*sysargs)
        cfg = rsol.SolverConfig(**kw)
        x0 = rsol._default_initial_guess(b, cfg, np.random.default_rng(cfg.seed))
        t0 = time.time()
        x, rep = rsol.solve(a, b, cfg=cfg)
        put_train(st, f"{tag}_a", a.cores)
        put_train(st, f"{tag}_b", b.cores)
        put_train(st, f"{tag}_x0", x0.cores)
        put_train(st, f"{tag}_x", x.cores)
        st[f"{tag}_res"] = np.array(rep.residual_history)
        st[f"{tag}_ranks"] = np.array(rep.rank_history)
        st[f"{tag}_comp"] = np.array(rep.compression_history)
        st[f"{tag}_conv"] = np.array(rep.converged)
        st[f"{tag}_stag"] = np.array(rep.stagnated)
        for k, v in kw.items():
            st[f"{tag}_cfg_{k}"] = np.array(v)
        print(tag, f"{time.time() - t0:.2f}s", rep.residual_history[-1], x.ranks)
    st["tags"] = np.array([c[0] for c in SOLVE_CASES])
    save("solve_small.npz", st)


def ref_steady(recipe):
    d = recipe.dims
    spec = spec_of(d, recipe.degree, recipe.eps, recipe.beta, 0.0, rhs=0.0)
    op = assemble_opset(spec)
    rows, reps = row_axes(op.grids), rep_axes(op.grids)
    rhs_tt = rtt.tt_from_separable(recipe.rhs_terms(rows))
    g_tt = rtt.tt_rank_one(recipe.exact_factors(reps)) if recipe.has_boundary_data() else None
    a, b = impose_dirichlet(op, spec, rhs_tt=rhs_tt, g_tt=g_tt)
    return a, b, rtt.tt_rank_one(recipe.exact_factors(reps))


def steady_config(index, fname, **over):
    recipe = wl.config(index, **over)
    a, b, exact = ref_steady(recipe)
    cfg = rsol.SolverConfig(**recipe.solver)
    x0 = rsol._default_initial_guess(b, cfg, np.random.default_rng(cfg.seed))
    t0 = time.time()
    x, rep = rsol.solve(a, b, cfg=cfg)
    wall = time.time() - t0
    err = rtt.tt_norm(rtt.tt_add(x, rtt.tt_scale(exact, -1.0))) / rtt.tt_norm(exact)
    st = {}
    put_train(st, "a", a.cores)
    put_train(st, "b", b.cores)
    put_train(st, "x0", x0.cores)
    put_train(st, "x", x.cores)
    st["res"] = np.array(rep.residual_history)
    st["ranks"] = np.array(rep.rank_history)
    st["conv"] = np.array(rep.converged)
    st["exact_err"] = np.array(err)
    st["wall"] = np.array(wall)
    print(fname, f"{wall:.1f}s", "ranks", x.ranks, "res", rep.residual_history[-1], "err", err)
    save(fname, st)


def sweep_small(fname, count=4, sweeps=30):
    """Config 4 scaled: d=3, n=13, four seeded boundary-layer solves, a
    bounded number of sweeps (the full d=6 solves take hours on the CPU)."""
    st = {}
    for i, r in enumerate(wl.sweep_recipes(count=count, dims=3, degree=12)):
        a, b, exact = ref_steady(r)
        cfg = rsol.SolverConfig(**r.solver, max_sweeps=sweeps)
        x0 = rsol._default_initial_guess(b, cfg, np.random.default_rng(cfg.seed))
        x, rep = rsol.solve(a, b, cfg=cfg)
        put_train(st, f"a{i}", a.cores)
        put_train(st, f"b{i}", b.cores)
        put_train(st, f"x{i}", x.cores)
        st[f"res{i}"] = np.array(rep.residual_history)
        st[f"conv{i}"] = np.array(rep.converged)
        st[f"eps{i}"] = np.array(r.eps)
        print(fname, i, f"eps {r.eps:.2e}", x.ranks, rep.residual_history)
    st["count"] = np.array(count)
    st["sweeps"] = np.array(sweeps)
    save(fname, st)


def ref_march(recipe, n_keep, keep_forcing=True, keep_every=1, keep_ops=True):
    d = recipe.dims
    spec = spec_of(d, recipe.degree, recipe.eps, recipe.beta, 0.0, rhs=0.0)
    op = assemble_opset(spec)
    mc = rti.MarchConfig(dt=recipe.dt, t_end=recipe.dt * recipe.n_steps)
    left, right, mask, anti = rti._march_operators(op, spec, mc)
    rows, reps = row_axes(op.grids), rep_axes(op.grids)
    state = rtt.tt_round(rtt.tt_rank_one(recipe.u_factors(reps, 0.0)), 1e-14)
    st = {}
    if keep_ops:
        put_train(st, "left", left.cores)
        put_train(st, "right", right.cores)
    else:  # fingerprints: the tests rebuild the operators with ttss's own setup
        st["left_sums"] = np.array([np.abs(c).sum() for c in left.cores])
        st["right_sums"] = np.array([np.abs(c).sum() for c in right.cores])
    put_train(st, "state0", state.cores)
    cfg = rsol.SolverConfig(**recipe.solver)
    walls = []
    for k in range(1, n_keep + 1):
        t = k * recipe.dt
        bc = rtt.tt_apply(anti, rtt.tt_rank_one(recipe.u_factors(reps, t)))
        src = rtt.tt_scale(rtt.tt_apply(mask, rtt.tt_from_separable(recipe.f_terms(rows, t))),
                           recipe.dt)
        t0 = time.time()
        rhs = rtt.tt_round(rtt.tt_add(rtt.tt_add(rtt.tt_apply(right, state), bc), src),
                           0.01 * recipe.step_tol)
        new, rep = rsol.solve(left, rhs, x0=state, cfg=cfg)
        state = rtt.tt_round(new, recipe.step_tol)
        walls.append(time.time() - t0)
        exact = rtt.tt_rank_one(recipe.u_factors(reps, t))
        err = rtt.tt_norm(rtt.tt_add(state, rtt.tt_scale(exact, -1.0))) / rtt.tt_norm(exact)
        if keep_forcing:
            put_train(st, f"bc{k}", bc.cores)
            put_train(st, f"src{k}", src.cores)
        if k % keep_every == 0 or k == n_keep:
            put_train(st, f"state{k}", state.cores)
        st[f"ranks{k}"] = np.array(state.ranks)
        st[f"res{k}"] = np.array(rep.residual_history)
        st[f"err{k}"] = np.array(err)
        print(f"  step {k}: {walls[-1]:.2f}s ranks {state.ranks} res "
              f"{rep.residual_history[-1]:.3e} err {err:.3e}")
    st["walls"] = np.array(walls)
    st["residual_tol"] = np.array(cfg.residual_tol)
    st["rounding_tol"] = np.array(cfg.rounding_tol)
    st["max_rank"] = np.array(cfg.max_rank)
    st["step_tol"] = np.array(recipe.step_tol)
    return st


def march_config(index, fname, n_keep, **over):
    recipe = wl.config(index, **over)
    print(fname, recipe)
    save(fname, ref_march(recipe, n_keep))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["grids", "ops", "round", "solve", "cfg0", "cfg2", "cfg3s"]
    if "grids" in which:
        grids()
    if "ops" in which:
        operators()
    if "round" in which:
        rounding()
    if "solve" in which:
        solves()
    if "cfg0" in which:
        steady_config(0, "config0.npz")
    if "cfg1s" in which:
        steady_config(1, "config1_small.npz", degree=12)
    if "cfg1" in which:
        steady_config(1, "config1.npz")
    if "cfg4s" in which:
        sweep_small("config4_small.npz")
    if "cfg2" in which:
        march_config(2, "config2_steps.npz", 3)
    if "cfg2s" in which:
        march_config(2, "config2_small.npz", 5, dims=3, degree=12, beta=wl.unit_vector(3, 2))
    if "cfg3s" in which:
        march_config(3, "config3_small.npz", 3, dims=3, beta=wl.unit_vector(3, 3))
