"""Pin the CPU oracle against outputs of the reference itself
(tests/golden/*.npz, produced by tools/make_golden.py)."""

import numpy as np
import pytest

from golden_io import get_train
from helpers import ranks_agree, rel_diff, value_tol
from oracle import als_solver as als
from oracle import march as om
from oracle import tt_ops as ot


def test_round_matches_reference(golden):
    z = golden("round.npz")
    for i in range(int(z["count"])):
        v, want = get_train(z, f"in{i}"), get_train(z, f"out{i}")
        tol, cap = float(z[f"tol{i}"]), int(z[f"cap{i}"]) or None
        got = ot.tt_round(v, tol, max_rank=cap)
        assert ot.ranks_of(got) == ot.ranks_of(want), i
        assert rel_diff(got, want) <= 1e-12, i
        assert abs(ot.tt_norm(v) - float(z[f"norm{i}"])) <= 1e-13 * float(z[f"norm{i}"])


def _cfg(z, tag):
    kw = {k[len(tag) + 5:]: z[k].item() for k in z if k.startswith(f"{tag}_cfg_")}
    return als.Config(**kw)


@pytest.mark.parametrize("tag", ["s1", "s2", "s3", "s4", "s5", "s6", "s7", "s8"])
def test_solve_small_matches_reference(golden, tag):
    z = golden("solve_small.npz")
    a, b, x0 = get_train(z, f"{tag}_a"), get_train(z, f"{tag}_b"), get_train(z, f"{tag}_x0")
    cfg = _cfg(z, tag)
    x, rep = als.solve(a, b, x0=x0, cfg=cfg)
    want = get_train(z, f"{tag}_x")
    conv = bool(z[f"{tag}_conv"])
    ref_res = np.array(z[f"{tag}_res"])
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


def test_initial_guess_matches_reference(golden):
    z = golden("solve_small.npz")
    for tag in ["s1", "s2", "s3"]:
        b = get_train(z, f"{tag}_b")
        x0 = als.initial_guess(b, als.Config(), np.random.default_rng(0))
        assert rel_diff(x0, get_train(z, f"{tag}_x0")) <= 1e-12


def test_config0_matches_reference(golden):
    z = golden("config0.npz")
    cfg = als.Config(residual_tol=1e-10, rounding_tol=1e-12)
    x, rep = als.solve(get_train(z, "a"), get_train(z, "b"), x0=get_train(z, "x0"), cfg=cfg)
    want = get_train(z, "x")
    assert rep.converged
    ok, det = ranks_agree(x, want)
    assert ok, det
    assert rel_diff(x, want) <= value_tol(rep.residual_history[-1], z["res"][-1])


@pytest.mark.parametrize("fname,steps", [("config2_small.npz", 5), ("config3_small.npz", 3),
                                         ("config2_steps.npz", 2)])
def test_march_matches_reference(golden, fname, steps):
    z = golden(fname)
    left, right = get_train(z, "left"), get_train(z, "right")
    state = get_train(z, "state0")
    cfg = als.Config(residual_tol=float(z["residual_tol"]), rounding_tol=float(z["rounding_tol"]),
                     max_rank=int(z["max_rank"]))
    for k in range(1, steps + 1):
        state, rep, _ = om.step(left, right, state, get_train(z, f"bc{k}"),
                                get_train(z, f"src{k}"), float(z["step_tol"]), cfg, index=k)
        want = get_train(z, f"state{k}")
        ok, det = ranks_agree(state, want)
        assert ok, (k, det)
        # solve accuracy plus the step re-truncation, accumulated over steps
        tol = value_tol(rep.residual_history[-1], z[f"res{k}"][-1]) + 2 * float(z["step_tol"])
        assert rel_diff(state, want) <= k * tol, k
