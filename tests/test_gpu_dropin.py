"""The drop-in, proven inside the reference itself: an unmodified ``ttss``
(baseline/_ref) has its hot path rebound to the engine by
``paper_2506_04732_b200.dropin.install()`` (the shim INTEGRATION.md
describes), and the reference's own public entry points —
``time_integration.backward_euler_march`` / ``crank_nicolson_march`` /
``spacetime_solve`` and ``tt_solver.solve`` — are called exactly as a ttss
user calls them.  Each result is compared with the same call on the
unpatched ttss (its CPU path), and the engine's launch counters prove the
calls went through libt2s2.so."""

import numpy as np
import pytest

from helpers import rel_diff
from oracle import tt_ops as ot

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def ref():
    from paper_2506_04732_b200 import _native, reference

    _native.context()
    return {m: reference.module(m) for m in ("coefficients", "operator_assembly",
                                             "time_integration", "tt_solver", "tensor_train")}


def _launches():
    from paper_2506_04732_b200 import _native

    return sum(v["launches"] for v in _native.stats_read().values())


def _patched(fn):
    from paper_2506_04732_b200 import _native, dropin

    _native.stats_reset()
    dropin.install()
    try:
        out = fn()
    finally:
        dropin.uninstall()
    assert _launches() > 0, "the patched call did not reach the engine"
    return out


def _spec(ref, dims=3, degree=10, t_end=0.05):
    co, asm = ref["coefficients"], ref["operator_assembly"]
    return asm.ProblemSpec(
        dims=dims, degrees=[degree] * dims, epsilon=co.constant_coefficient(1e-2, dims),
        beta=[co.constant_coefficient(b, dims) for b in (1.0, 0.5, 0.25)[:dims]],
        rho=co.constant_coefficient(0.0, dims), rhs=co.constant_coefficient(1.0, dims),
        initial=co.Coefficient(dims, [(1.0, [co.Bump(0.1 * k, 0.6) for k in range(dims)])]),
        time=asm.TimeSpec(t_end=t_end))


@pytest.mark.parametrize("scheme", ["backward_euler", "crank_nicolson"])
def test_march_through_patched_ttss(ref, scheme):
    asm, ti, sol = ref["operator_assembly"], ref["time_integration"], ref["tt_solver"]
    spec = _spec(ref)
    opset = asm.assemble_opset(spec)
    # the inner target sits where both solvers stop on the same sweep: with
    # 1e-10, backward Euler's first sweeps land near the threshold and the
    # two sides may stop one sweep apart (a cond x 1e-10 = 4e-9 difference);
    # with 1e-12 the reference's own run is unchanged (its residuals are
    # 1e-13..1e-16) and the comparison is at 1e-10.  CN stagnates above
    # 1e-12 in the reference itself, so it keeps 1e-10.
    tol = 1e-12 if scheme == "backward_euler" else 1e-10
    cfg = ti.MarchConfig(dt=0.01, t_end=0.05, scheme=scheme,
                         solver=sol.SolverConfig(residual_tol=tol))
    entry = ti.backward_euler_march if scheme == "backward_euler" else ti.crank_nicolson_march
    want, wdiag = entry(opset, spec, cfg)                       # the reference's CPU path
    got, gdiag = _patched(lambda: entry(opset, spec, cfg))      # same call, engine path
    assert len(got) == len(want) == 6
    rows = []
    for (tg, sg), (tw, sw) in zip(got, want):
        assert tg == tw
        assert type(sg) is type(sw)                              # ttss's own TTVector
        rows.append((tg, sg.ranks, sw.ranks, rel_diff(sg.cores, sw.cores)))
    assert all(r[1] == r[2] for r in rows), rows
    assert all(r[3] <= TOL for r in rows), rows
    assert gdiag.steps == wdiag.steps and gdiag.max_ranks == wdiag.max_ranks
    np.testing.assert_allclose(gdiag.peak_norms, wdiag.peak_norms, rtol=1e-9)
    assert max(gdiag.residuals) <= 1e-10 and max(wdiag.residuals) <= 1e-10


def test_solve_and_residual_through_patched_ttss(ref):
    """A steady PDE system (golden solve case s3's setup) through the patched
    tt_solver.solve / residual.  A steady solve's raw ranks keep the last
    enrichment directions (not re-truncated, unlike march states): ttss
    ends at (1, 7, 7, 1), its numpy restatement at (1, 9, 7, 1) with the
    values equal to 9e-14, so ranks are compared numerically (1e-10)."""
    from helpers import ranks_agree

    asm, sol, co = ref["operator_assembly"], ref["tt_solver"], ref["coefficients"]
    d = 3
    spec = asm.ProblemSpec(dims=d, degrees=[6] * d, epsilon=co.constant_coefficient(0.05, d),
                           beta=[co.constant_coefficient(1.0, d)] * d,
                           rho=co.constant_coefficient(0.1, d),
                           rhs=co.constant_coefficient(1.0, d))
    a, b = asm.impose_dirichlet(asm.assemble_opset(spec), spec)
    cfg = sol.SolverConfig(residual_tol=1e-10, max_rank=40)
    xw, rw = sol.solve(a, b, cfg=cfg)
    xg, rg = _patched(lambda: sol.solve(a, b, cfg=cfg))
    assert type(rg) is type(rw) and rg.converged and rw.converged
    diff = rel_diff(xg.cores, xw.cores)
    ok, detail = ranks_agree(xg.cores, xw.cores)
    assert ok, (detail, xg.ranks, xw.ranks, diff)
    assert diff <= TOL, (diff, rg.residual_history, rw.residual_history)
    res_w = sol.residual(a, xw, b)
    res_g = _patched(lambda: sol.residual(a, xg, b))
    assert res_g <= 1e-10 and abs(res_g - res_w) <= 1e-10


def test_spacetime_through_patched_ttss(ref):
    """One-shot space-time heat solve.  Its alternating iterations are not
    reproducible at the level of raw ranks even between the reference and
    its numpy restatement (the rank-1 start enriches from degenerate
    gradient directions: first-sweep residual 1.2e-7 for ttss, 4.2e-7 for
    the oracle; final ranks 7 and 6, both converged), so the converged
    solutions are compared as functions: values on the full grid and
    numerical ranks at 1e-10."""
    co, asm, ti, sol = (ref["coefficients"], ref["operator_assembly"], ref["time_integration"],
                        ref["tt_solver"])
    from helpers import ranks_agree

    spec = asm.ProblemSpec(dims=1, degrees=[10], epsilon=co.constant_coefficient(0.2, 1),
                           beta=[co.constant_coefficient(0.0, 1)],
                           rho=co.constant_coefficient(0.0, 1),
                           rhs=co.constant_coefficient(0.0, 1),
                           initial=co.Coefficient(1, [(1.0, [co.SinPiK(1)])]),
                           time=asm.TimeSpec(t_end=0.5, degree=12))
    opset = asm.assemble_opset(spec)
    cfg = sol.SolverConfig(residual_tol=1e-11, max_rank=20)
    xw, rw, tw = ti.spacetime_solve(opset, spec, cfg)
    xg, rg, tg = _patched(lambda: ti.spacetime_solve(opset, spec, cfg))
    np.testing.assert_array_equal(tg.base.rep_nodes, tw.base.rep_nodes)
    assert rg.converged and rw.converged
    fw, fg = ot.tt_full(xw.cores), ot.tt_full(xg.cores)
    assert np.linalg.norm(fg - fw) <= 1e-9 * np.linalg.norm(fw)
    ok, detail = ranks_agree(xg.cores, xw.cores)
    assert ok, detail
