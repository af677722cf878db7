"""The five BASELINE.json configurations as data recipes.

Each recipe only produces numbers (coefficients, sampled separable factors,
solver settings); ``steady_problem`` / ``march_problem`` turn them into
trains with the reference's own setup code (ttss), exactly as
``tools/make_golden.py`` does when it records the reference's outputs.  The manufactured solutions are seeded
synthetic stand-ins for the reference's benchmark problems (there is no
external dataset).

  0  d=2 steady, n=17 nodes, eps=1e-2, b=(1,1), Gaussian bump
  1  d=3 steady, n=33, eps=1e-6, b=(1,.5,.25), separable boundary layer
  2  d=6 + time, n=33, eps=1e-3, translating Gaussian, BE dt=1e-3, 100 steps
  3  d=6 + time, n=65, eps=1e-12, translating Gaussian, dt=5e-4, 200 steps, cap 64
  4  64 independent d=6 steady boundary-layer solves, n=33

"TT tolerance 1e-12" is the solver's SVD rounding tolerance (rounding_tol);
the march keeps the reference's MarchConfig defaults (time_integration.py:
54-60): inner residual_tol=1e-10 and step re-truncation 1e-8.  Tightening
the residual target to 1e-12 is not sustainable over a 100-step march (the
alternating solver stalls at its noise floor after ~60 steps and the bond
ranks grow with every enrichment sweep), and truncating states at 1e-12
with a 1e-10 solve keeps solver noise in the ranks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GAUSS_WIDTH = 0.05      # translating Gaussian exp(-|x - b t|^2 / 0.05)
BUMP_WIDTH = 0.1        # config 0: exp(-sum (x_k - 0.2)^2 / 0.1)
BUMP_CENTER = 0.2


# -- univariate profiles and their derivatives ----------------------------------


def gauss(x, c, w):
    return np.exp(-((x - c) ** 2) / w)


def gauss_d1(x, c, w):
    return -2.0 * (x - c) / w * gauss(x, c, w)


def gauss_d2(x, c, w):
    return (4.0 * (x - c) ** 2 / w ** 2 - 2.0 / w) * gauss(x, c, w)


def layer(s, b, eps):
    """g(s) = (s+1)/2 - (e^{b(s-1)/eps} - e^{-2b/eps}) / (1 - e^{-2b/eps}),
    evaluated without overflow for either sign of b; solves
    -eps g'' + b g' = b/2 with g(-1) = g(1) = 0."""
    s = np.asarray(s, dtype=float)
    if b > 0:
        e = (np.exp(b * (s - 1.0) / eps) - np.exp(-2.0 * b / eps)) / (-np.expm1(-2.0 * b / eps))
    else:
        c = -b
        e = -np.expm1(-c * (s + 1.0) / eps) / (-np.expm1(-2.0 * c / eps))
    return 0.5 * (s + 1.0) - e


@dataclass
class SteadyRecipe:
    name: str
    dims: int
    degree: int
    eps: float
    beta: list
    kind: str                       # "bump" | "layer"
    solver: dict = field(default_factory=dict)

    def rhs_terms(self, axes):
        """Separable terms of f = -eps lap u + beta . grad u on ``axes``."""
        d, eps = self.dims, self.eps
        terms = []
        if self.kind == "bump":
            g = [gauss(ax, BUMP_CENTER, BUMP_WIDTH) for ax in axes]
            for l in range(d):
                lead = (-eps * gauss_d2(axes[l], BUMP_CENTER, BUMP_WIDTH)
                        + self.beta[l] * gauss_d1(axes[l], BUMP_CENTER, BUMP_WIDTH))
                terms.append((1.0, [lead if k == l else g[k] for k in range(d)]))
        else:
            g = [layer(ax, self.beta[k], eps) for k, ax in enumerate(axes)]
            for l in range(d):
                terms.append((0.5 * self.beta[l],
                              [np.ones_like(axes[l]) if k == l else g[k] for k in range(d)]))
        return terms

    def exact_factors(self, axes):
        if self.kind == "bump":
            return [gauss(ax, BUMP_CENTER, BUMP_WIDTH) for ax in axes]
        return [layer(ax, self.beta[k], self.eps) for k, ax in enumerate(axes)]

    def has_boundary_data(self):
        return self.kind == "bump"


@dataclass
class MarchRecipe:
    name: str
    dims: int
    degree: int
    eps: float
    beta: list
    dt: float
    n_steps: int
    step_tol: float = 1e-8
    solver: dict = field(default_factory=dict)

    def u_factors(self, axes, t):
        return [gauss(ax, b * t, GAUSS_WIDTH) for ax, b in zip(axes, self.beta)]

    def f_terms(self, axes, t):
        """u_t + b.grad u = 0 for the translating profile, so f = -eps lap u."""
        g = self.u_factors(axes, t)
        return [(-self.eps, [gauss_d2(ax, b * t, GAUSS_WIDTH) if k == l else g[k]
                             for k, (ax, b) in enumerate(zip(axes, self.beta))])
                for l in range(self.dims)]


def unit_vector(d, seed):
    v = np.random.default_rng(seed).standard_normal(d)
    return list(v / np.linalg.norm(v))


def config(index, **over):
    """Recipe of BASELINE.json configs[index]; keyword overrides for scaled
    test variants (e.g. degree=8)."""
    if index == 0:
        r = SteadyRecipe("d2_steady_bump", 2, 16, 1e-2, [1.0, 1.0], "bump",
                         solver=dict(residual_tol=1e-10, rounding_tol=1e-12))
    elif index == 1:
        r = SteadyRecipe("d3_steady_layer", 3, 32, 1e-6, [1.0, 0.5, 0.25], "layer",
                         solver=dict(residual_tol=1e-10, rounding_tol=1e-12))
    elif index == 2:
        r = MarchRecipe("d6_time_n33", 6, 32, 1e-3, unit_vector(6, 2), 1e-3, 100,
                        solver=dict(residual_tol=1e-10, rounding_tol=1e-12))
    elif index == 3:
        r = MarchRecipe("d6_time_n65", 6, 64, 1e-12, unit_vector(6, 3), 5e-4, 200,
                        solver=dict(residual_tol=1e-10, rounding_tol=1e-12, max_rank=64))
    elif index == 4:
        raise ValueError("config 4 is a batch; use sweep_recipes()")
    else:
        raise ValueError(f"no config {index}")
    for k, v in over.items():
        setattr(r, k, v)
    return r


def sweep_recipes(count=64, seed=4, dims=6, degree=32):
    """Config 4: per solve, eps log-uniform in [1e-12, 1e-1], b a random unit
    vector, separable boundary-layer solution."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        eps = float(10.0 ** rng.uniform(-12.0, -1.0))
        b = rng.standard_normal(dims)
        b = list(b / np.linalg.norm(b))
        out.append(SteadyRecipe(f"sweep_{i}", dims, degree, eps, b, "layer",
                                solver=dict(residual_tol=1e-10, rounding_tol=1e-12)))
    return out


# -- builders: the reference's own problem setup (ttss) ------------------------------


def _spec(recipe):
    """ProblemSpec of a recipe: constant eps and beta, no reaction, zero
    symbolic rhs (the manufactured forcing is supplied as trains)."""
    from .reference import module

    co, asm = module("coefficients"), module("operator_assembly")
    d = recipe.dims
    return asm.ProblemSpec(dims=d, degrees=[recipe.degree] * d,
                           epsilon=co.constant_coefficient(recipe.eps, d),
                           beta=[co.constant_coefficient(b, d) for b in recipe.beta],
                           rho=co.constant_coefficient(0.0, d),
                           rhs=co.constant_coefficient(0.0, d))


def steady_problem(recipe):
    """(A, rhs, exact, opset) for a steady recipe, assembled by ttss
    (operator_assembly.assemble_opset / impose_dirichlet)."""
    from .reference import module

    asm, rtt = module("operator_assembly"), module("tensor_train")
    spec = _spec(recipe)
    opset = asm.assemble_opset(spec)
    rows, reps = asm.row_axes(opset.grids), asm.rep_axes(opset.grids)
    rhs_tt = rtt.tt_from_separable(recipe.rhs_terms(rows))
    g_tt = rtt.tt_rank_one(recipe.exact_factors(reps)) if recipe.has_boundary_data() else None
    a, b = asm.impose_dirichlet(opset, spec, rhs_tt=rhs_tt, g_tt=g_tt)
    return a, b, rtt.tt_rank_one(recipe.exact_factors(reps)), opset


def march_problem(recipe):
    """(left, right, state0, forcing(k) -> (bc_k, src_k), exact(t), opset),
    built by ttss exactly as time_integration._march does
    (time_integration.py:149-163), with the forcing sampled at t_k."""
    from .reference import module

    asm, rtt, rti = (module("operator_assembly"), module("tensor_train"),
                     module("time_integration"))
    spec = _spec(recipe)
    opset = asm.assemble_opset(spec)
    mcfg = rti.MarchConfig(dt=recipe.dt, t_end=recipe.dt * recipe.n_steps)
    left, right, mask, anti = rti._march_operators(opset, spec, mcfg)
    rows, reps = asm.row_axes(opset.grids), asm.rep_axes(opset.grids)
    state0 = rtt.tt_round(rtt.tt_rank_one(recipe.u_factors(reps, 0.0)), 1e-14)

    def forcing(k):
        t = k * recipe.dt
        bc = rtt.tt_apply(anti, rtt.tt_rank_one(recipe.u_factors(reps, t)))
        src = rtt.tt_scale(rtt.tt_apply(mask, rtt.tt_from_separable(recipe.f_terms(rows, t))),
                           recipe.dt)
        return bc, src

    def exact(t):
        return rtt.tt_rank_one(recipe.u_factors(reps, t))

    return left, right, state0, forcing, exact, opset
