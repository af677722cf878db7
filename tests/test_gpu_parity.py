"""Parity of the CUDA path (through the C ABI) with the reference's outputs
(tests/golden) and the CPU oracle.  Protocol: see tests/helpers.py."""

import numpy as np
import pytest

from golden_io import get_train
from helpers import ranks_agree, rel_diff, value_tol
from oracle import tt_ops as ot

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_2506_04732_b200 as pkg
    from paper_2506_04732_b200 import _native, march, solver, tt

    _native.context()  # fail loudly if the engine cannot start
    return pkg, tt, solver, march


def V(tt, cores):
    return tt.TTVector(cores)


def O(tt, cores):
    return tt.TTOperator(cores)


def test_round_matches_reference(golden, pk):
    _, tt, _, _ = pk
    z = golden("round.npz")
    for i in range(int(z["count"])):
        v, want = get_train(z, f"in{i}"), get_train(z, f"out{i}")
        tol, cap = float(z[f"tol{i}"]), int(z[f"cap{i}"]) or None
        got = tt.tt_round(V(tt, v), tol, max_rank=cap).cores
        assert ot.ranks_of(got) == ot.ranks_of(want), (i, ot.ranks_of(got), ot.ranks_of(want))
        assert rel_diff(got, want) <= 1e-12, i
        nrm = tt.tt_norm(V(tt, v))
        assert abs(nrm - float(z[f"norm{i}"])) <= 1e-13 * float(z[f"norm{i}"])


def test_exact_arithmetic_matches_oracle(pk):
    _, tt, _, _ = pk
    rng = np.random.default_rng(5)
    for modes, ra, rb in [((5, 6, 4), 3, 2), ((4, 4, 4, 4), 2, 5), ((7,), 1, 1), ((3, 9), 4, 4)]:
        d = len(modes)
        rka = [1] + [ra] * (d - 1) + [1]
        rkb = [1] + [rb] * (d - 1) + [1]
        a = [rng.standard_normal((rka[l], modes[l], rka[l + 1])) for l in range(d)]
        b = [rng.standard_normal((rkb[l], modes[l], rkb[l + 1])) for l in range(d)]
        op = [rng.standard_normal((2 if l else 1, modes[l], modes[l], 2 if l < d - 1 else 1))
              for l in range(d)]
        assert abs(tt.tt_dot(V(tt, a), V(tt, b)) - ot.tt_dot(a, b)) <= 1e-12 * (
            ot.tt_norm(a) * ot.tt_norm(b))
        s = tt.tt_add(V(tt, a), V(tt, b)).cores
        assert ot.ranks_of(s) == ot.ranks_of(ot.tt_add(a, b))
        np.testing.assert_allclose(tt.tt_full(V(tt, s)), ot.tt_full(a) + ot.tt_full(b),
                                   rtol=1e-12, atol=1e-12 * np.abs(ot.tt_full(a)).max())
        ap = tt.tt_apply(O(tt, op), V(tt, a)).cores
        np.testing.assert_allclose(ot.tt_full(ap), ot.tt_full(ot.tt_apply(op, a)), rtol=1e-11,
                                   atol=1e-11 * np.abs(ot.tt_full(ap)).max())
        np.testing.assert_allclose(tt.tt_op_full(O(tt, op)), ot.tt_op_full(op), rtol=1e-12,
                                   atol=1e-12)


def _cfg(solver, z, tag):
    kw = {k[len(tag) + 5:]: z[k].item() for k in z if k.startswith(f"{tag}_cfg_")}
    return solver.SolverConfig(**kw)


@pytest.mark.parametrize("tag", ["s1", "s2", "s3", "s4", "s5", "s6", "s7", "s8"])
def test_solve_small_matches_reference(golden, pk, tag):
    _, tt, solver, _ = pk
    z = golden("solve_small.npz")
    a, b = O(tt, get_train(z, f"{tag}_a")), V(tt, get_train(z, f"{tag}_b"))
    cfg = _cfg(solver, z, tag)
    x, rep = solver.solve(a, b, cfg=cfg)
    want = get_train(z, f"{tag}_x")
    ref_res = np.array(z[f"{tag}_res"])
    conv = bool(z[f"{tag}_conv"])
    assert max(rep.rank_history) <= cfg.max_rank
    if conv:
        assert rep.converged
        ok, det = ranks_agree(x.cores if hasattr(x, "cores") else x, want)
        assert ok, det
        assert rel_diff(x.cores if hasattr(x, "cores") else x, want) <= value_tol(
            rep.residual_history[-1], ref_res[-1])
    else:
        # Rank-capped, non-converging cases hinge on near-ties between the
        # Galerkin and least-squares candidates (the reference itself varies
        # run to run): require a plateau no worse than the reference's and
        # the same stagnation verdict when the reference stagnated.
        assert rep.residual_history[-1] <= 1.05 * ref_res[-1]
        if bool(z[f"{tag}_stag"]):
            assert rep.stagnated


def test_config0_matches_reference(golden, pk):
    _, tt, solver, _ = pk
    z = golden("config0.npz")
    cfg = solver.SolverConfig(residual_tol=1e-10, rounding_tol=1e-12)
    x, rep = solver.solve(O(tt, get_train(z, "a")), V(tt, get_train(z, "b")),
                          x0=V(tt, get_train(z, "x0")), cfg=cfg)
    want = get_train(z, "x")
    assert rep.converged
    ok, det = ranks_agree(x.cores, want)
    assert ok, det
    assert rel_diff(x.cores, want) <= value_tol(rep.residual_history[-1], z["res"][-1])


@pytest.mark.parametrize("fname,steps", [("config2_small.npz", 5), ("config3_small.npz", 3),
                                         ("config2_steps.npz", 3)])
def test_march_matches_reference(golden, pk, fname, steps):
    _, tt, solver, march = pk
    z = golden(fname)
    left, right = tt.to_device(O(tt, get_train(z, "left"))), tt.to_device(O(tt, get_train(z, "right")))
    state = tt.to_device(V(tt, get_train(z, "state0")))
    bcs = [tt.to_device(V(tt, get_train(z, f"bc{k}"))) for k in range(1, steps + 1)]
    srcs = [tt.to_device(V(tt, get_train(z, f"src{k}"))) for k in range(1, steps + 1)]
    cfg = solver.SolverConfig(residual_tol=float(z["residual_tol"]),
                              rounding_tol=float(z["rounding_tol"]), max_rank=int(z["max_rank"]))
    stored, rows = march.march_device(left, right, state, steps, bcs, srcs, float(z["step_tol"]), cfg,
                                      store_stride=1)
    for k in range(1, steps + 1):
        got = tt.from_device(stored[k]).cores
        want = get_train(z, f"state{k}")
        ok, det = ranks_agree(got, want)
        assert ok, (k, det)
        tol = value_tol(rows[k - 1][3], z[f"res{k}"][-1]) + 2 * float(z["step_tol"])
        assert rel_diff(got, want) <= k * tol, k
    for h in [left, right, state] + bcs + srcs + list(stored.values()):
        h.free()


def test_errors_follow_reference(pk):
    pkg, tt, solver, march = pk
    rng = np.random.default_rng(1)
    eye = tt.tt_identity_operator((3, 3))
    zero = tt.tt_from_separable([(0.0, [np.ones(3), np.ones(3)])])
    with pytest.raises(ValueError):
        solver.solve(eye, zero)
    v = tt.tt_random((3, 4), 2, rng)
    with pytest.raises(pkg.ShapeError):
        solver.solve(tt.tt_identity_operator((3, 5)), v)
    with pytest.raises(ValueError):
        tt.tt_round(v, -1.0)


def test_identity_system_one_sweep(pk):
    _, tt, solver, _ = pk
    rng = np.random.default_rng(0)
    v = tt.tt_random((5, 6, 4), 3, rng, norm=2.0)
    x, rep = solver.solve(tt.tt_identity_operator((5, 6, 4)), v,
                          cfg=solver.SolverConfig(residual_tol=1e-12))
    assert rep.converged and rep.residual_history[-1] <= 1e-12
    assert rel_diff(x.cores, v.cores) <= 1e-12


def test_march_stagnation_raises_with_step(golden, pk):
    pkg, tt, solver, march = pk
    z = golden("config2_small.npz")
    left, right = tt.to_device(O(tt, get_train(z, "left"))), tt.to_device(O(tt, get_train(z, "right")))
    state = tt.to_device(V(tt, get_train(z, "state0")))
    bc, src = tt.to_device(V(tt, get_train(z, "bc1"))), tt.to_device(V(tt, get_train(z, "src1")))
    cfg = solver.SolverConfig(residual_tol=1e-30, max_rank=1, enrichment_rank=0, max_sweeps=8)
    with pytest.raises(pkg.MarchStepError) as err:
        march.march_device(left, right, state, 2, [bc], [src], 1e-12, cfg)
    assert err.value.step == 1


@pytest.mark.parametrize("tag", ["s2", "s3", "s4"])
def test_iterative_local_solver_matches_oracle(golden, pk, tag):
    """Force the Krylov local solves (GMRES for Galerkin, Jacobi-PCG for least
    squares) and compare with the oracle running scipy's solvers."""
    from oracle import als_solver as als

    _, tt, solver, _ = pk
    z = golden("solve_small.npz")
    a, b, x0 = get_train(z, f"{tag}_a"), get_train(z, f"{tag}_b"), get_train(z, f"{tag}_x0")
    kw = {k[len(tag) + 5:]: z[k].item() for k in z if k.startswith(f"{tag}_cfg_")}
    kw["local_solver"] = "iterative"
    x, rep = solver.solve(O(tt, a), V(tt, b), x0=V(tt, x0), cfg=solver.SolverConfig(**kw))
    xo, repo = als.solve(a, b, x0=x0, cfg=als.Config(**kw))
    assert rep.converged == repo.converged
    if repo.converged:
        ok, det = ranks_agree(x.cores, xo)
        assert ok, det
        assert rel_diff(x.cores, xo) <= value_tol(rep.residual_history[-1],
                                                  repo.residual_history[-1])


@pytest.mark.parametrize("n", [1, 7, 33, 165, 500, 825, 1617, 2000, 2112])
def test_dense_local_solve_kernel(pk, n):
    """The fused LU kernel against numpy.linalg.solve (LAPACK getrf/getrs),
    on matrices needing pivoting."""
    from paper_2506_04732_b200 import _native

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    a[np.arange(n), np.arange(n)] *= 1e-3  # small diagonal forces row interchanges
    b = rng.standard_normal(n)
    x = _native.dense_solve(a, b)
    want = np.linalg.solve(a, b)
    cond = np.linalg.cond(a)
    assert np.linalg.norm(x - want) <= 1e-14 * cond * np.linalg.norm(want) + 1e-300
    assert np.linalg.norm(a @ x - b) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(x)


@pytest.mark.parametrize("n", [7, 64, 65, 300, 1000, 1953, 2000, 2500])
def test_dense_local_solve_without_interchanges(pk, n):
    """Column diagonally dominant matrices: partial pivoting makes no
    interchange, so the verified no-pivot kernel alone must solve them, to
    LAPACK's accuracy."""
    from paper_2506_04732_b200 import _native

    rng = np.random.default_rng(100 + n)
    a = rng.standard_normal((n, n))
    a += np.diag(np.abs(a).sum(0))
    b = rng.standard_normal(n)
    _native.stats_reset()
    x = _native.dense_solve(a, b)
    st = _native.stats_read()
    assert st["gj_nopivot"]["launches"] == 1
    assert st.get("lu_fused", {}).get("launches", 0) == 0
    want = np.linalg.solve(a, b)
    assert np.linalg.norm(x - want) <= 1e-14 * np.linalg.cond(a) * np.linalg.norm(want)
    assert np.linalg.norm(a @ x - b) <= 1e-13 * np.linalg.norm(a) * np.linalg.norm(x)


def test_dense_local_solve_late_interchange(pk):
    """Diagonally dominant except one column deep in the matrix: the no-pivot
    kernel runs through several panels, meets a multiplier > 1, declines
    (info -1) and the pivoting kernel solves the original matrix."""
    from paper_2506_04732_b200 import _native

    rng = np.random.default_rng(5)
    n = 300
    a = rng.standard_normal((n, n))
    a += np.diag(np.abs(a).sum(0))
    a[200, 200] *= 1e-6  # column 200 needs a row interchange
    b = rng.standard_normal(n)
    _native.stats_reset()
    x = _native.dense_solve(a, b)
    st = _native.stats_read()
    assert st["gj_nopivot"]["launches"] == 1 and st["lu_fused"]["launches"] == 1
    want = np.linalg.solve(a, b)
    assert np.linalg.norm(x - want) <= 1e-14 * np.linalg.cond(a) * np.linalg.norm(want)


@pytest.mark.parametrize("row", [201, 230, 290])
@pytest.mark.parametrize("mult,pivots", [(3.0, False), (20.0, True)])
def test_dense_local_solve_threshold_pivoting(pk, row, mult, pivots):
    """Threshold partial pivoting of the Gauss-Jordan kernel (|l| <= 8): one
    sub-diagonal entry of column 200 is `mult` times the diagonal, in the same
    32-row diagonal block (row 201), in the next diagonal block's rows (230 —
    checked by a worker's tile task) or further below (290).  A multiplier of 3
    is eliminated without an interchange on the Gauss-Jordan kernel alone, 20
    declines to the pivoting kernel; both to LAPACK's accuracy."""
    from paper_2506_04732_b200 import _native

    rng = np.random.default_rng(11)
    n = 420
    a = rng.standard_normal((n, n))
    a += np.diag(np.abs(a).sum(0))
    a[row, 200] = mult * a[200, 200]
    b = rng.standard_normal(n)
    _native.stats_reset()
    x = _native.dense_solve(a, b)
    st = _native.stats_read()
    assert st["gj_nopivot"]["launches"] == 1
    assert st.get("lu_fused", {}).get("launches", 0) == (1 if pivots else 0)
    want = np.linalg.solve(a, b)
    assert np.linalg.norm(x - want) <= 1e-14 * np.linalg.cond(a) * np.linalg.norm(want)
    assert np.linalg.norm(a @ x - b) <= 1e-13 * np.linalg.norm(a) * np.linalg.norm(x)


@pytest.mark.parametrize("ta,tb,m,n,k", [
    (0, 0, 37, 29, 13), (1, 0, 64, 65, 70), (0, 1, 130, 64, 132), (1, 1, 33, 40, 9),
    (0, 0, 2112, 64, 1024),  # split-K with a reduce stage
    (0, 1, 200, 48, 600),    # split-K, transposed B
    (0, 0, 1024, 2112, 64),  # 64x64 tiles
    (0, 0, 16384, 132, 132),  # 64x136 tiles (the config-4 operator-core stage)
    (1, 0, 9500, 71, 70),     # 64x136 tiles, ragged, transposed A
])
def test_gemm_program_against_torch(pk, ta, tb, m, n, k):
    """The GEMM-program kernel behind every contraction (DMMA tiles, operand
    layouts, split-K) against a plain PyTorch fp64 matmul (cuBLAS)."""
    import torch

    from paper_2506_04732_b200 import _native

    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    a = torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn((n, k) if tb else (k, n), dtype=torch.float64, device="cuda", generator=g)
    c = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    _native.gemm_device(ta, tb, m, n, k, a.data_ptr(), a.shape[1], b.data_ptr(), b.shape[1],
                        c.data_ptr(), n)
    _native.synchronize()
    want = (a.T if ta else a) @ (b.T if tb else b)
    # fp64 rounding of a length-k dot product: well inside 1e-13 relative
    assert torch.isfinite(c).all()
    assert ((c - want).norm() / want.norm()).item() <= 1e-13


def test_dense_local_solve_singular(pk):
    from paper_2506_04732_b200 import _native

    a = np.ones((4, 4))
    with pytest.raises(ValueError):
        _native.dense_solve(a, np.ones(4))


def test_config4_sweep_small_matches_reference(golden, pk):
    """Config 4 scaled (d=3, n=13, four seeded boundary-layer solves) through
    the sweep driver on the device."""
    from paper_2506_04732_b200 import sweep, workloads as wl

    z = golden("config4_small.npz")
    recipes = wl.sweep_recipes(count=int(z["count"]), dims=3, degree=12)
    res = sweep.run_sweep(recipes, overrides={"max_sweeps": int(z["sweeps"])})
    for i in range(int(z["count"])):
        got, ref = res[i], np.array(z[f"res{i}"])
        assert got["converged"] == bool(z[f"conv{i}"])
        want = get_train(z, f"x{i}")
        assert rel_diff(got["x"], want) <= value_tol(got["residuals"][-1], ref[-1])
        ok, det = ranks_agree(got["x"], want)
        assert ok, (i, det)


@pytest.mark.slow
def test_config1_full_matches_reference(golden, pk):
    """Config 1 at full size (d=3, n=33, eps=1e-6): local systems up to
    ~42k unknowns go through the device GMRES/PCG path.  The reference stops
    at max_sweeps without converging (plateau ~1.8e-7), so the run is
    compared by its plateau and its error against the manufactured solution.

    Once a bond reaches full rank (33 = n at the end bonds) the enrichment of
    _split_left/_split_right (tt_solver.py:261-302) appends directions of a
    gradient that is rounding noise after projection, so from there on the
    trajectory depends on the summation order: the reference's own plateau
    is not reproducible across BLAS thread counts, and the step at which the
    residual drops from ~1.2e-4 moves by several sweeps between correct
    implementations (measured: sweep 14 for ttss with default threads, sweep
    3 for ttss on one thread and for the engine's previous CTA-barrier SVD;
    the manufactured-solution error agrees to 6 digits in all of them).
    Bound: same convergence verdict and sweep count, final residual within
    3x of the reference envelope (fixture keys env_*: 1.8e-7 default
    threads, 1.1e-7 one thread), manufactured-solution error equal to the
    envelope's to 1e-4 relative."""
    from oracle import tt_ops as ot
    from paper_2506_04732_b200 import workloads as wl

    _, tt, solver, _ = pk
    z = golden("config1.npz")
    recipe = wl.config(1)
    cfg = solver.SolverConfig(**recipe.solver)
    x, rep = solver.solve(O(tt, get_train(z, "a")), V(tt, get_train(z, "b")),
                          x0=V(tt, get_train(z, "x0")), cfg=cfg)
    assert rep.converged == bool(z["conv"])
    assert len(rep.residual_history) == len(z["res"])
    # envelope of reference runs (default threads: the fixture; 1 thread:
    # leaves the plateau at sweep 3 instead of 14, ends at 1.1e-7 vs 1.8e-7)
    env_res, env_err = float(np.max(z["env_res"])), float(np.max(z["env_err"]))
    assert rep.residual_history[-1] <= 3.0 * env_res, (rep.residual_history[-1], env_res)
    a, b, exact, opset = wl.steady_problem(recipe)
    err = ot.tt_norm(ot.tt_add(x.cores, ot.tt_scale(exact.cores, -1.0))) / ot.tt_norm(exact.cores)
    assert err <= (1 + 1e-4) * env_err, (err, env_err)


def test_singular_local_systems_use_lstsq(golden, pk):
    """Every local system of s8 is exactly singular: numpy raises and the
    reference takes numpy.linalg.lstsq's minimum-norm solution; the engine's
    SVD fallback must land on the same iterate."""
    _, tt, solver, _ = pk
    z = golden("solve_small.npz")
    a, b = O(tt, get_train(z, "s8_a")), V(tt, get_train(z, "s8_b"))
    x, rep = solver.solve(a, b, cfg=_cfg(solver, z, "s8"))
    ref = np.array(z["s8_res"])
    assert rep.stagnated and not rep.converged
    np.testing.assert_allclose(rep.residual_history[-1], ref[-1], rtol=1e-9)
    assert rel_diff(x.cores, get_train(z, "s8_x")) <= 1e-9


def test_config4_sweep_on_sm_partitions(golden, pk):
    """The scaled sweep on two disjoint SM partitions (green contexts), one
    host thread and engine context each: every solve converges to the
    reference's solution, and the engine is deterministic, so a solve's
    result does not depend on the partition (or its SM count) it ran on."""
    from paper_2506_04732_b200 import sweep, workloads as wl

    z = golden("config4_small.npz")
    recipes = wl.sweep_recipes(count=int(z["count"]), dims=3, degree=12)
    ov = {"max_sweeps": int(z["sweeps"])}
    res = sweep.run_sweep(recipes, overrides=ov, partitions=2)
    serial = sweep.run_sweep(recipes[:1], overrides=ov)
    for i in range(int(z["count"])):
        got, ref = res[i], np.array(z[f"res{i}"])
        want = get_train(z, f"x{i}")
        assert got["converged"] == bool(z[f"conv{i}"])
        assert rel_diff(got["x"], want) <= value_tol(got["residuals"][-1], ref[-1])
    assert res[0]["residuals"] == serial[0]["residuals"]
    for c1, c2 in zip(res[0]["x"], serial[0]["x"]):
        np.testing.assert_array_equal(c1, c2)


def test_config3_full_size_steps_match_oracle(pk):
    """Config 3 at full size (d=6, n=65, eps=1e-12, dt=5e-4): the first two
    implicit steps through the device march against the CPU oracle (the
    numpy restatement of time_integration._march / tt_solver.solve) on the
    same operators and forcing.  Ranks identical, states within the
    protocol's tolerance (solve residuals plus the step re-truncation)."""
    from oracle import als_solver as als
    from oracle import march as om
    from paper_2506_04732_b200 import workloads as wl
    from paper_2506_04732_b200.march import march_device

    _, tt, solver, _ = pk
    recipe = wl.config(3)
    left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
    steps = 2
    fs = [forcing(k) for k in range(1, steps + 1)]
    hl, hr, hs = tt.to_device(left), tt.to_device(right), tt.to_device(state0)
    bcs = [tt.to_device(b) for b, _ in fs]
    srcs = [tt.to_device(s) for _, s in fs]
    cfg = solver.SolverConfig(**recipe.solver)
    stored, rows = march_device(hl, hr, hs, steps, bcs, srcs, recipe.step_tol, cfg, store_stride=1)
    state = state0.cores
    for k in range(1, steps + 1):
        state, rep, _ = om.step(left.cores, right.cores, state, fs[k - 1][0].cores,
                                fs[k - 1][1].cores, recipe.step_tol, als.Config(**recipe.solver))
        got = tt.from_device(stored[k]).cores
        ok, det = ranks_agree(got, state)
        assert ok, (k, det)
        tol = value_tol(rows[k - 1][3], rep.residual_history[-1]) + 2 * recipe.step_tol
        assert rel_diff(got, state) <= k * tol, k
    for h in [hl, hr, hs] + bcs + srcs + list(stored.values()):
        h.free()


@pytest.mark.parametrize("index", [0])
def test_config4_full_size_sweeps_within_oracle_spread(pk, index):
    """Config 4 at full size (d=6, n=33): two alternating sweeps of one of
    the 64 seeded boundary-layer solves (index 7: eps = 2.9e-12, the steep
    end of the draw) from the default initial guess.  Far from convergence
    the reference algorithm itself is not reproducible: with the same
    inputs, the oracle's residual after one sweep moves by ~2% between BLAS
    thread counts (0.885 with 1 thread, 0.865 with 8, 0.878 default for
    index 0: tools/c4_check.py), because near-equal candidate scores
    (tt_solver.py:383-387) and enrichment directions depend on the summation
    order.  The device run must reproduce the ranks exactly and its residual
    history must lie within the envelope of five oracle executions (1, 2, 4,
    8 BLAS threads and the default) widened by their own spread.

    The steep seeds (index 7, eps = 2.9e-12) are compared on complete solves
    instead (test_gpu_parity_full.py): after two sweeps their residual moves
    by 25% between the oracle's own thread counts (0.174..0.243) and the
    reference's (0.2018..0.2076, ttss with 1..8 threads), so a two-sweep
    envelope says nothing about them."""
    from threadpoolctl import threadpool_limits

    from oracle import als_solver as als
    from paper_2506_04732_b200 import workloads as wl

    _, tt, solver, _ = pk
    r = wl.sweep_recipes()[index]
    a, b, exact, _ = wl.steady_problem(r)
    kw = dict(r.solver)
    kw["max_sweeps"] = 2
    x, rep = solver.solve(a, b, cfg=solver.SolverConfig(**kw))
    runs = []
    for limit in (1, 2, 4, 8, None):
        with threadpool_limits(limits=limit):
            xo, repo = als.solve(a.cores, b.cores, cfg=als.Config(**kw))
        runs.append((xo, np.array(repo.residual_history)))
        assert ot.ranks_of(x.cores) == ot.ranks_of(xo)
    hist = np.array([h for _, h in runs])
    lo, hi = hist.min(axis=0), hist.max(axis=0)
    spread = np.maximum(hi - lo, 1e-8 * hi)
    got = np.array(rep.residual_history)
    assert np.all(got >= lo - 3 * spread) and np.all(got <= hi + 3 * spread), (got, lo, hi)


@pytest.mark.parametrize("rank", [8, 24, 40, 64])
def test_norm_and_round_wide_cores(pk, rank):
    """TT norm and rounding at the ranks of the residual difference train and
    of config 4 (unfoldings up to 33*64 x 64): the warp-level QR/TSQR leaves
    (one to four columns per warp, multi-leaf trees) and the thin SVD against
    the oracle (numpy Householder QR / LAPACK SVD)."""
    from oracle import tt_ops as ot

    _, tt, _, _ = pk
    rng = np.random.default_rng(rank)
    d, n = 4, 33
    ranks = [1] + [rank] * (d - 1) + [1]
    # graded cores: singular values spread over many orders, a sum of two
    # trains so the unfoldings are rank deficient after the sum
    cores = []
    for l in range(d):
        c = rng.standard_normal((ranks[l], n, ranks[l + 1]))
        c *= np.logspace(0, -12, ranks[l + 1])[None, None, :]
        cores.append(c)
    x = tt.TTVector(cores)
    want = ot.tt_norm(cores)
    got = tt.tt_norm(x)
    assert abs(got - want) <= 1e-13 * want
    s = ot.tt_add(cores, ot.tt_scale(cores, -0.5))  # ranks double, half of them dependent
    got_s = tt.tt_norm(tt.TTVector(s))
    assert abs(got_s - 0.5 * want) <= 1e-12 * want
    r = tt.tt_round(tt.TTVector(s), 1e-10)
    ro = ot.tt_round(s, 1e-10)
    assert r.ranks == list(ot.ranks_of(ro)) or ranks_agree(r.cores, ro)[0]
    full_ok = float(np.prod([float(c.shape[1]) for c in s])) <= 2e6
    if full_ok:
        assert np.linalg.norm(ot.tt_full(r.cores) - ot.tt_full(ro)) <= 1e-9 * np.linalg.norm(ot.tt_full(ro))


@pytest.mark.parametrize("n,budget", [(264, 0), (1601, 0), (1848, 0), (1953, 0), (2000, 0), (1200, 24),
                                      (1952, 64)])
def test_dense_local_solve_deterministic(pk, n, budget):
    """The Gauss-Jordan solve hands panels between CTAs and warps without
    grid barriers (arrival counts, named barriers): repeated solves of one
    system must be bit-identical and accurate (N = 1601: a one-row last
    panel).  Long tile phases — N >= 1953 on 148 CTAs, or fewer CTAs (an SM
    budget) — are the case where CTA 0 finishes a phase ahead of the tile
    workers: its arrival must not stand in for theirs (a shared arrival
    counter did, giving errors of 1e-6 that changed from run to run)."""
    from paper_2506_04732_b200 import _native

    rng = np.random.default_rng(7 + n)
    a = rng.standard_normal((n, n))
    a += np.diag(np.abs(a).sum(0))
    b = rng.standard_normal(n)
    want = np.linalg.solve(a, b)
    _native.set_thread_sm_budget(budget)
    try:
        ref = _native.dense_solve(a, b)
        for _ in range(8):
            assert np.array_equal(_native.dense_solve(a, b), ref)
    finally:
        _native.set_thread_sm_budget(0)
    assert np.linalg.norm(ref - want) <= 1e-13 * np.linalg.norm(want)
