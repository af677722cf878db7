"""Full-length parity of the device march with the REFERENCE (ttss) on the
BASELINE configs at full size: every step of the 100-step config-2 march and
of the 200-step config-3 march, against states recorded by running ttss
(tools/make_golden_full.py -> tests/golden/config{2,3}_full.npz).

For every step the test checks north_star's three criteria:
  * raw TT ranks of the state identical to the reference's;
  * relative difference of the full-grid solution (10^5 seeded sample
    points: the grid has 33^6 / 65^6 entries) within PARITY_TOL;
  * error against the analytic manufactured solution no worse than the
    reference's (to ERR_SLACK relative: both are ~1e-3 backward-Euler time
    errors that agree to many digits).
The achieved numbers of every step are written to
gpurun_out/parity_full_<config>.json (committed under profiles/).

Tolerance: each step re-solves to the reference's residual_tol (1e-10) and
re-truncates at step_tol (1e-8), so two correct implementations differ by
rounding-level amounts amplified by the local solves' conditioning and
accumulated over the steps.  The reference is not reproducible below that
level itself: the same march with 1, 2 or 8 instead of 4 (config 2) / 1
instead of 2 (config 3) OpenBLAS threads differs from the fixture by up to
2.9e-10 / 3.7e-10 (tests/golden/config{2,3}_selfspread.npz: per step the
largest difference over these reference runs; tools/make_golden_full.py
spread).  The bound at step k is therefore max(1e-10, 2 x the reference's
own largest thread-count difference up to step k): north_star's 1e-10
wherever the reference itself holds it, its own noise envelope elsewhere.
"""

import json
import os

import numpy as np
import pytest

from golden_io import get_train, has_train
from helpers import rel_diff
from oracle import tt_ops as ot

pytestmark = pytest.mark.gpu

PARITY_TOL = 1e-10       # north_star: full-grid relative agreement
ERR_SLACK = 1e-6         # relative slack on the manufactured-solution error
PLATEAU_FACTOR = 3.0     # config 4: x the envelope of reference-equivalent plateaus


def _record(name, rows, summary):
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", os.getcwd()), "gpurun_out")
    try:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"parity_full_{name}.json"), "w") as fh:
            json.dump({"summary": summary, "steps": rows}, fh, indent=1)
    except OSError:
        pass


def _march_full(golden, index, fname):
    from paper_2506_04732_b200 import _native, tt, workloads as wl
    from paper_2506_04732_b200.march import march_device
    from paper_2506_04732_b200.solver import SolverConfig

    _native.context()
    z = golden(fname)
    recipe = wl.config(index)
    n = int(z["n_steps"])
    left, right, state0, forcing, exact, _ = wl.march_problem(recipe)
    fs = [forcing(k) for k in range(1, n + 1)]
    hl, hr, hs = tt.to_device(left), tt.to_device(right), tt.to_device(state0)
    bcs = [tt.to_device(b) for b, _ in fs]
    srcs = [tt.to_device(s) for _, s in fs]
    cfg = SolverConfig(**recipe.solver)
    stored, rows = march_device(hl, hr, hs, n, bcs, srcs, recipe.step_tol, cfg, store_stride=1)
    states = {k: tt.from_device(h).cores for k, h in stored.items()}
    for h in [hl, hr, hs] + bcs + srcs + list(stored.values()):
        h.free()
    out, worst = [], {"rel_diff": 0.0, "rank_mismatch": 0, "err_excess": 0.0}
    for k in range(1, n + 1):
        got = states[k]
        ref_ranks = tuple(int(r) for r in z[f"ranks{k}"])
        row = {"step": k, "ranks": list(ot.ranks_of(got)), "ranks_ref": list(ref_ranks),
               "residual": rows[k - 1][3], "residual_ref": float(np.array(z[f"res{k}"])[-1]),
               "sweeps": rows[k - 1][4], "sweeps_ref": int(np.array(z[f"res{k}"]).size)}
        ex = exact(k * recipe.dt).cores
        err = ot.tt_norm(ot.tt_add(got, ot.tt_scale(ex, -1.0))) / ot.tt_norm(ex)
        row["exact_err"], row["exact_err_ref"] = float(err), float(z[f"err{k}"])
        if has_train(z, f"state{k}"):
            row["rel_diff"] = rel_diff(got, get_train(z, f"state{k}"))
            worst["rel_diff"] = max(worst["rel_diff"], row["rel_diff"])
        worst["rank_mismatch"] += int(tuple(row["ranks"]) != ref_ranks)
        worst["err_excess"] = max(worst["err_excess"], err / row["exact_err_ref"] - 1.0)
        out.append(row)
    spread = golden(fname.replace("_full.npz", "_selfspread.npz"))
    summary = dict(worst, config=index, steps=n,
                   reference_self_spread=float(np.max(spread["rel_diff"])),
                   reference_self_spread_threads=[int(t) for t in spread["threads"]],
                   steps_within_1e10=sum(1 for r in out if "rel_diff" in r and r["rel_diff"] <= PARITY_TOL),
                   steps_compared=sum(1 for r in out if "rel_diff" in r), final_exact_err=out[-1]["exact_err"],
                   final_exact_err_ref=out[-1]["exact_err_ref"],
                   sweeps=sum(r["sweeps"] for r in out),
                   sweeps_ref=sum(r["sweeps_ref"] for r in out))
    _record(f"config{index}", out, summary)
    return out, summary


def _bounds(golden, fname):
    """Per-step value bound: max(PARITY_TOL, 2 x running max of the
    reference's own thread-count spread)."""
    z = golden(fname.replace("_full.npz", "_selfspread.npz"))
    steps, diffs = np.array(z["steps"]), np.array(z["rel_diff"])
    run = np.maximum.accumulate(diffs)
    return {int(k): max(PARITY_TOL, 2.0 * float(v)) for k, v in zip(steps, run)}


@pytest.mark.parametrize("index,fname", [(2, "config2_full.npz"), (3, "config3_full.npz")])
def test_march_full_length_matches_reference(golden, index, fname):
    rows, summary = _march_full(golden, index, fname)
    bad_ranks = [(r["step"], r["ranks"], r["ranks_ref"]) for r in rows
                 if r["ranks"] != r["ranks_ref"]]
    assert not bad_ranks, bad_ranks[:5]
    bound = _bounds(golden, fname)
    bad_vals = [(r["step"], r["rel_diff"], bound[r["step"]]) for r in rows
                if "rel_diff" in r and r["rel_diff"] > bound[r["step"]]]
    assert not bad_vals, (summary, bad_vals[:5])
    bad_err = [(r["step"], r["exact_err"], r["exact_err_ref"]) for r in rows
               if r["exact_err"] > r["exact_err_ref"] * (1 + ERR_SLACK)]
    assert not bad_err, bad_err[:5]


# -- config 4: complete steady solves -------------------------------------------------


def _solve_full(golden, index):
    from helpers import sample_entries
    from paper_2506_04732_b200 import _native, solver, tt, workloads as wl

    _native.context()
    z = golden(f"config4_full_{index}.npz")
    r = wl.sweep_recipes()[index]
    a, b, exact, _ = wl.steady_problem(r)
    x0 = tt.TTVector(get_train(z, "x0"))
    x, rep = solver.solve(a, b, x0=x0, cfg=solver.SolverConfig(**r.solver))
    err = ot.tt_norm(ot.tt_add(x.cores, ot.tt_scale(exact.cores, -1.0))) / ot.tt_norm(exact.cores)
    rng = np.random.default_rng(int(z["sample_idx_seed"]))
    idx = np.column_stack([rng.integers(0, n, 10000) for n in x.mode_sizes])
    xs, ref = sample_entries(x.cores, idx), np.array(z["x_samples"])
    out = {
        "index": index, "eps": float(z["eps"]),
        "sweeps": len(rep.residual_history), "sweeps_ref": int(np.array(z["res"]).size),
        "converged": rep.converged, "converged_ref": bool(z["conv"]),
        "stagnated": rep.stagnated, "stagnated_ref": bool(z["stag"]),
        "ranks": list(x.ranks), "ranks_ref": [int(v) for v in z["x_ranks"]],
        "rank_history": rep.rank_history, "rank_history_ref": [int(v) for v in z["ranks"]],
        "residuals": rep.residual_history, "residuals_ref": [float(v) for v in z["res"]],
        "exact_err": float(err), "exact_err_ref": float(z["exact_err"]),
        "sample_rel_diff": float(np.linalg.norm(xs - ref) / np.linalg.norm(ref)),
        "wall_s": rep.wall_time, "wall_s_ref": float(z["wall"]),
    }
    _record(f"config4_{index}", [], out)
    return out


@pytest.mark.parametrize("index", [0, 2, 7])
def test_config4_complete_solve_matches_reference(golden, index):
    """A complete config-4 solve (d=6, n=33, 40 sweeps, rank cap 64) against
    ttss's own complete solve of the same seed.  These solves do not
    converge in the reference either: ranks reach the cap and the residual
    decreases slowly to the sweep limit (a rank-capped plateau), where the
    iterate is path dependent — ttss itself ends seed 0 at residual 2.2e-4
    with 2 OpenBLAS threads and 8.3e-5 with 1 (error 5.1e-4 / 1.9e-4), its
    numpy restatement ends seed 2 at 4.0e-3 against ttss's 1.7e-3 / 2.1e-3.
    Checked exactly: the verdict, the sweep count and the rank history.
    Checked against the envelope of these reference-equivalent runs
    (fixture keys env_*, tools/config4_envelope.py): the final residual and
    the manufactured-solution error no worse than PLATEAU_FACTOR x the
    envelope's largest."""
    o = _solve_full(golden, index)
    z = golden(f"config4_full_{index}.npz")
    env_res, env_err = float(np.max(z["env_res"])), float(np.max(z["env_err"]))
    assert (o["converged"], o["stagnated"]) == (o["converged_ref"], o["stagnated_ref"]), o
    assert o["sweeps"] == o["sweeps_ref"], o
    assert max(o["ranks"]) == max(o["ranks_ref"]) == 64
    assert o["rank_history"] == o["rank_history_ref"], o
    assert o["residuals"][-1] <= PLATEAU_FACTOR * env_res, (o["residuals"][-1], env_res)
    assert o["exact_err"] <= PLATEAU_FACTOR * env_err, (o["exact_err"], env_err)
